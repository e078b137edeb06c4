"""ctypes binding of the C ABI (include/nautilus_b200.h).

The shared library is built in-tree by ``paper_2604_14825_b200.build``.  There
is no fallback: if it is missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NativeLibraryMissing, raise_for_status

LIB_PATH = os.environ.get("NT_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_native", "libnautilus_b200.so")

NT_MASK_NONE, NT_MASK_CAUSAL, NT_MASK_TENSOR, NT_MASK_BITS = 0, 1, 2, 3
NT_DTYPE_BF16, NT_DTYPE_F32, NT_DTYPE_E4M3 = 0, 1, 2

# Every symbol include/nautilus_b200.h declares (checked by tests/test_capi.py).
EXPORTED = (
    "nt_attn_fwd", "nt_attn_workspace_bytes", "nt_attn_prepare", "nt_attn_resident_ctas",
    "nt_attn_plan_create", "nt_attn_plan_launch", "nt_attn_plan_destroy", "nt_attn_decode", "nt_decode_workspace_bytes", "nt_decode_num_splits", "nt_gemm",
    "nt_gemm_chain", "nt_gemm_chain_workspace_bytes", "nt_gemm_k_splits", "nt_gemm_workspace_bytes",
    "nt_cast_f32_to_bf16", "nt_cast_bf16_to_f32", "nt_abi_version", "nt_last_error", "nt_launch_count",
    "nt_module_load", "nt_module_function", "nt_launch", "nt_module_unload", "nt_attn_decode_paged",
    "nt_memcpy2d_async", "nt_mask_to_bits",
)


class Tensor4(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("stride_b", C.c_int64), ("stride_h", C.c_int64),
                ("stride_s", C.c_int64)]


class AttnArgs(C.Structure):
    _fields_ = [("q", Tensor4), ("k", Tensor4), ("v", Tensor4), ("o", Tensor4),
                ("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
                ("seq_q", C.c_int32), ("seq_kv", C.c_int32), ("head_dim", C.c_int32),
                ("scale", C.c_float), ("mask_kind", C.c_int32), ("causal_offset", C.c_int32),
                ("mask", C.c_void_p), ("mask_stride_row", C.c_int64),
                ("out_dtype", C.c_int32), ("err_flag", C.c_void_p), ("work_counter", C.c_void_p),
                ("kv_stages", C.c_int32), ("in_dtype", C.c_int32), ("q_descale", C.c_float),
                ("k_descale", C.c_float), ("v_descale", C.c_float), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_int64), ("item_rows", C.c_int32)]


class DecodeArgs(C.Structure):
    _fields_ = [("q", Tensor4), ("k", Tensor4), ("v", Tensor4), ("o", Tensor4),
                ("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
                ("seq_q", C.c_int32), ("seq_kv", C.c_int32), ("head_dim", C.c_int32),
                ("scale", C.c_float), ("num_splits", C.c_int32), ("out_dtype", C.c_int32),
                ("workspace", C.c_void_p), ("err_flag", C.c_void_p), ("workspace_bytes", C.c_int64),
                ("in_dtype", C.c_int32), ("q_descale", C.c_float), ("k_descale", C.c_float),
                ("v_descale", C.c_float)]


class DecodePagedArgs(C.Structure):
    _fields_ = [("q", Tensor4), ("o", Tensor4), ("k_pages", C.c_void_p), ("v_pages", C.c_void_p),
                ("page_stride", C.c_int64), ("token_stride", C.c_int64), ("head_stride", C.c_int64),
                ("num_pages", C.c_int32), ("page_size", C.c_int32), ("block_table", C.c_void_p),
                ("block_table_stride", C.c_int32), ("seq_lens", C.c_void_p),
                ("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
                ("seq_q", C.c_int32), ("max_seq_kv", C.c_int32), ("head_dim", C.c_int32),
                ("scale", C.c_float), ("num_splits", C.c_int32), ("out_dtype", C.c_int32),
                ("workspace", C.c_void_p), ("err_flag", C.c_void_p), ("workspace_bytes", C.c_int64),
                ("in_dtype", C.c_int32), ("q_descale", C.c_float), ("k_descale", C.c_float),
                ("v_descale", C.c_float)]


class GemmArgs(C.Structure):
    _fields_ = [("a", C.c_void_p), ("lda", C.c_int64), ("b", C.c_void_p), ("ldb", C.c_int64),
                ("c", C.c_void_p), ("ldc", C.c_int64), ("m", C.c_int32), ("n", C.c_int32),
                ("k", C.c_int32), ("out_dtype", C.c_int32), ("k_splits", C.c_int32), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_int64)]


class ChainArgs(C.Structure):
    _fields_ = [("x", C.c_void_p), ("ldx", C.c_int64), ("w1", C.c_void_p), ("ldw1", C.c_int64),
                ("w2", C.c_void_p), ("ldw2", C.c_int64), ("y", C.c_void_p), ("ldy", C.c_int64),
                ("n", C.c_int32), ("k", C.c_int32), ("f", C.c_int32), ("e", C.c_int32),
                ("out_dtype", C.c_int32), ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64)]


_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the native library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} not built: run `python -m paper_2604_14825_b200.build` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            L.nt_attn_fwd.argtypes = [C.POINTER(AttnArgs), C.c_void_p]
            L.nt_attn_prepare.argtypes = [C.POINTER(AttnArgs)]
            L.nt_attn_resident_ctas.argtypes = [C.POINTER(AttnArgs)]
            L.nt_attn_plan_create.argtypes = [C.POINTER(AttnArgs), C.POINTER(C.c_void_p)]
            L.nt_attn_plan_launch.argtypes = [C.c_void_p, C.c_void_p]
            L.nt_attn_plan_destroy.argtypes = [C.c_void_p]
            L.nt_attn_plan_destroy.restype = None
            L.nt_attn_decode.argtypes = [C.POINTER(DecodeArgs), C.c_void_p]
            L.nt_attn_decode_paged.argtypes = [C.POINTER(DecodePagedArgs), C.c_void_p]
            L.nt_decode_workspace_bytes.argtypes = [C.c_int32] * 5
            L.nt_decode_workspace_bytes.restype = C.c_int64
            L.nt_decode_num_splits.argtypes = [C.c_int32] * 4
            L.nt_decode_num_splits.restype = C.c_int
            L.nt_gemm.argtypes = [C.POINTER(GemmArgs), C.c_void_p]
            L.nt_attn_workspace_bytes.argtypes = [C.POINTER(AttnArgs)]
            L.nt_attn_workspace_bytes.restype = C.c_int64
            L.nt_gemm_chain.argtypes = [C.POINTER(ChainArgs), C.c_void_p]
            L.nt_gemm_chain_workspace_bytes.argtypes = [C.c_int32] * 3
            L.nt_gemm_chain_workspace_bytes.restype = C.c_int64
            L.nt_gemm_k_splits.argtypes = [C.c_int32] * 3
            L.nt_gemm_k_splits.restype = C.c_int32
            L.nt_gemm_workspace_bytes.argtypes = [C.c_int32] * 3
            L.nt_gemm_workspace_bytes.restype = C.c_int64
            L.nt_cast_f32_to_bf16.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
            L.nt_cast_bf16_to_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
            L.nt_module_load.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
            L.nt_module_function.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]
            L.nt_launch.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p),
                                    C.c_void_p]
            L.nt_module_unload.argtypes = [C.c_void_p]
            L.nt_memcpy2d_async.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_void_p]
            L.nt_memcpy2d_async.restype = C.c_int
            L.nt_mask_to_bits.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_void_p]
            L.nt_mask_to_bits.restype = C.c_int
            L.nt_last_error.restype = C.c_char_p
            L.nt_launch_count.restype = C.c_int64
            for name in ("nt_attn_fwd", "nt_attn_prepare", "nt_attn_resident_ctas", "nt_attn_plan_create",
                         "nt_attn_plan_launch", "nt_attn_decode", "nt_attn_decode_paged", "nt_gemm", "nt_gemm_chain",
                         "nt_cast_f32_to_bf16", "nt_cast_bf16_to_f32", "nt_abi_version",
                         "nt_module_load", "nt_module_function", "nt_launch", "nt_module_unload"):
                getattr(L, name).restype = C.c_int
            _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().nt_last_error().decode(errors="replace")
        raise_for_status(status, f"{what}: {msg}")


def launch_count() -> int:
    return int(lib().nt_launch_count())


_SMS: dict = {}


def num_sms(device) -> int:
    """SM count of a CUDA device (cached); the C side uses the same attribute."""
    import torch

    idx = torch.device(device).index if torch.device(device).index is not None else torch.cuda.current_device()
    if idx not in _SMS:
        _SMS[idx] = torch.cuda.get_device_properties(idx).multi_processor_count
    return _SMS[idx]
