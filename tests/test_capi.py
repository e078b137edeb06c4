"""The C-ABI library loads and exports every symbol include/nautilus_b200.h declares."""

import ctypes
import os
import re

import pytest

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
    assert L.nt_abi_version() == 4
    assert L.nt_launch_count() >= 0


def test_struct_layouts_match_header():
    # sizes computed from the header's field order (x86-64 SysV)
    assert ctypes.sizeof(_lib.Tensor4) == 32
    # ... + item_rows (int32, ABI 3) + tail padding to 8
    assert ctypes.sizeof(_lib.AttnArgs) == 4 * 32 + 6 * 4 + 4 + 4 + 4 + 4 + 8 + 8 + 4 + 4 + 8 + 8 + 4 + 4 + 3 * 4 + 4 + 8 + 8 + 4 + 4
    assert ctypes.sizeof(_lib.GemmArgs) == 6 * 8 + 4 * 4 + 4 + 4 + 8 + 8


STRUCTS = [("nt_tensor4", "Tensor4"), ("nt_attn_args", "AttnArgs"), ("nt_decode_args", "DecodeArgs"),
           ("nt_decode_paged_args", "DecodePagedArgs"), ("nt_gemm_args", "GemmArgs"),
           ("nt_chain_args", "ChainArgs")]


def test_ctypes_mirrors_match_the_c_compiler(tmp_path):
    """Every ctypes struct has the size and field offsets gcc gives the header's struct."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lines = ['#include <stdio.h>', '#include "nautilus_b200.h"', "int main(void) {"]
    for cname, pyname in STRUCTS:
        lines.append(f'  printf("{pyname} size %zu\\n", sizeof({cname}));')
        for fname, _ in getattr(_lib, pyname)._fields_:
            lines.append(f'  printf("{pyname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.dirname(HDR), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    seen = 0
    for line in filter(None, out):
        pyname, field, val = line.split()
        st = getattr(_lib, pyname)
        got = ctypes.sizeof(st) if field == "size" else getattr(st, field).offset
        assert got == int(val), (pyname, field, got, val)
        seen += 1
    assert seen == sum(1 + len(getattr(_lib, p)._fields_) for _, p in STRUCTS)
