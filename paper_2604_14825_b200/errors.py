"""Error mapping for the device boundary.

The reference raises typed exceptions rooted at ``CompilerError``
(tilecc/errors.py:26-128) and numeric faults ``OutOfBounds`` /
``DivisionByZero`` (tilecc/errors.py, tilecc/numerics.py:61-63, 123-126).
The C ABI returns integer status codes (include/nautilus_b200.h); this module
maps them onto an equivalent hierarchy.  When ``tilecc`` is importable the
classes also derive from the reference's own, so callers that catch
``tilecc.errors.CompilerError`` (e.g. the tuner, tilecc/tuner/tuner.py:180-184)
keep working unchanged.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from .frontdoor import import_tilecc as _import_tilecc

    _import_tilecc()  # sys.path or baseline/_ref
    from tilecc.errors import CompilerError as _RefCompilerError
    from tilecc.errors import OutOfBounds as _RefOutOfBounds
    from tilecc.numerics import DivisionByZero as _RefDivisionByZero
except Exception:  # tilecc absent (e.g. on a GPU box): standalone hierarchy
    class _RefCompilerError(Exception):
        pass

    class _RefOutOfBounds(_RefCompilerError):
        pass

    class _RefDivisionByZero(ArithmeticError):
        pass

from .ma_ir import UnsupportedMA as _UnsupportedMA


class BackendError(_RefCompilerError):
    """Root of the B200 backend's errors (a CompilerError)."""


class UnsupportedMA(BackendError, _UnsupportedMA):
    """The MA program (or this configuration of it) has no sm_100a realisation."""


class InvalidArguments(BackendError):
    pass


class DeviceError(BackendError):
    """CUDA runtime / driver failure."""


class NativeLibraryMissing(BackendError, RuntimeError):
    pass


class OutOfBounds(_RefOutOfBounds):
    pass


class DivisionByZero(_RefDivisionByZero):
    """A softmax denominator was zero on device (every key masked for a row)."""


def raise_for_status(status: int, message: str) -> None:
    if status == 1:
        raise InvalidArguments(message)
    if status == 2:
        raise UnsupportedMA(message)
    raise DeviceError(message)
