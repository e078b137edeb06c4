"""The C-ABI library loads and exports every symbol include/nautilus_b200.h declares."""

import ctypes
import os
import re

from paper_2604_14825_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "nautilus_b200.h")


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(nt_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_library_loads_and_exports_all_symbols():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.nt_abi_version() == 1
    assert L.nt_launch_count() >= 0


def test_struct_layouts_match_header():
    # sizes computed from the header's field order (x86-64 SysV)
    assert ctypes.sizeof(_lib.Tensor4) == 32
    assert ctypes.sizeof(_lib.AttnArgs) == 4 * 32 + 6 * 4 + 4 + 4 + 4 + 4 + 8 + 8 + 4 + 4 + 8 + 8 + 8
    assert ctypes.sizeof(_lib.GemmArgs) == 6 * 8 + 4 * 4
