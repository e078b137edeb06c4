"""Launch plans: a recognised KernelSpec bound to device tensors.

A plan owns the ctypes argument struct for one launch of a C-ABI entry point
(include/nautilus_b200.h) so that hot loops (bench, tuner timing) pay only the
foreign call.  torch is used purely as the device-memory / stream provider.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import _lib
from .errors import DivisionByZero, InvalidArguments
from .recognize import attn_item_rows  # noqa: F401  (the MA t0_i -> K1 item-rows rule)


def _stream_handle(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _as4(t: torch.Tensor) -> torch.Tensor:
    if t.dim() == 2:
        return t.unsqueeze(0).unsqueeze(0)
    if t.dim() == 3:
        return t.unsqueeze(0)
    if t.dim() != 4:
        raise InvalidArguments(f"expected a rank-2/3/4 tensor, got shape {tuple(t.shape)}")
    return t


def _t4(t: torch.Tensor) -> _lib.Tensor4:
    if t.stride(-1) != 1:
        raise InvalidArguments("innermost (head) dimension must be contiguous")
    return _lib.Tensor4(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))


class AttentionPlan:
    """K1 fused attention over a [B, H, N, D] outer grid (bf16 or e4m3 in, bf16/fp32 out).

    e4m3 inputs (``torch.float8_e4m3fn``, head_dim 128, no/causal mask) run the
    tcgen05 kind::f8f6f4 variant -- the paper's FP8 regime,
    beyond the reference's MA precisions -- with per-tensor descales:
    S = (Q K^T) q_descale k_descale scale, O = v_descale softmax(S) V, P rounded
    to e4m3 before P.V.
    """

    def __init__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor,
                 scale: Optional[float], mask_kind: str = "none", mask: Optional[torch.Tensor] = None,
                 causal_offset: int = 0, err_flag: Optional[torch.Tensor] = None, kv_stages: int = 0,
                 q_descale: float = 1.0, k_descale: float = 1.0, v_descale: float = 1.0,
                 work_counter: Optional[torch.Tensor] = None, item_rows: int = 0):
        q, k, v, o = _as4(q), _as4(k), _as4(v), _as4(o)
        e4m3 = q.dtype == torch.float8_e4m3fn
        want = torch.float8_e4m3fn if e4m3 else torch.bfloat16
        for name, t in (("q", q), ("k", k), ("v", v)):
            if t.dtype != want or not t.is_cuda:
                raise InvalidArguments(f"{name} must be a CUDA bf16 tensor (or q, k, v all float8_e4m3fn)")
        if o.dtype not in (torch.bfloat16, torch.float32) or not o.is_cuda:
            raise InvalidArguments("o must be a CUDA bf16/fp32 tensor")
        B, Hq, N, D = q.shape
        Bk, Hkv, M, Dk = k.shape
        if Bk != B or Dk != D or tuple(v.shape) != (B, Hkv, M, D) or tuple(o.shape) != (B, Hq, N, D):
            raise InvalidArguments("q/k/v/o shapes inconsistent")
        self.q, self.k, self.v, self.o, self.mask = q, k, v, o, mask
        self.err = err_flag if err_flag is not None else torch.zeros(1, dtype=torch.int32, device=q.device)
        kind = {"none": _lib.NT_MASK_NONE, "causal": _lib.NT_MASK_CAUSAL, "tensor": _lib.NT_MASK_TENSOR,
                "bits": _lib.NT_MASK_BITS}[mask_kind]
        self.mask_kind = mask_kind
        a = _lib.AttnArgs()
        a.q, a.k, a.v, a.o = _t4(q), _t4(k), _t4(v), _t4(o)
        a.batch, a.heads_q, a.heads_kv, a.seq_q, a.seq_kv, a.head_dim = B, Hq, Hkv, N, M, D
        a.scale = 1.0 if scale is None else float(scale)
        a.mask_kind = kind
        a.causal_offset = int(causal_offset)
        if kind == _lib.NT_MASK_TENSOR:
            if mask is None or mask.dtype != torch.float32 or not mask.is_cuda or mask.stride(-1) != 1:
                raise InvalidArguments("tensor mask must be a CUDA fp32 [N, M] tensor")
            a.mask = mask.data_ptr()
            a.mask_stride_row = mask.stride(0)
        elif kind == _lib.NT_MASK_BITS:
            if mask is None or mask.dtype != torch.int32 or not mask.is_cuda or mask.stride(-1) != 1:
                raise InvalidArguments("bit mask must be a CUDA int32 [N, words] tensor (pack_mask_bits)")
            a.mask = mask.data_ptr()
            a.mask_stride_row = mask.stride(0)
        a.out_dtype = _lib.NT_DTYPE_F32 if o.dtype == torch.float32 else _lib.NT_DTYPE_BF16
        a.err_flag = self.err.data_ptr()
        # dynamic (greedy LPT) item counter of the persistent kernel; reset on device by the
        # last CTA, so plans whose launches are ordered on one stream may share one
        self.work = work_counter if work_counter is not None else torch.zeros(2, dtype=torch.int32,
                                                                              device=q.device)
        a.work_counter = self.work.data_ptr()
        a.kv_stages = int(kv_stages)  # the MA `stages` tunable (0 = scheduler default)
        a.in_dtype = _lib.NT_DTYPE_E4M3 if e4m3 else _lib.NT_DTYPE_BF16
        a.q_descale, a.k_descale, a.v_descale = float(q_descale), float(k_descale), float(v_descale)
        a.item_rows = int(item_rows)  # 0 = library choice, 128 or 256 query rows per work item
        # split-KV workspace (non-zero only for few, long work items)
        ws = int(_lib.lib().nt_attn_workspace_bytes(C.byref(a)))
        # zeroed once per plan: every byte the merge reads is written by K1's TMA stores,
        # which compute-sanitizer's initcheck does not track
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=q.device) if ws else None
        a.workspace = self.ws.data_ptr() if ws else None
        a.workspace_bytes = ws
        from .recognize import attn_effective_rows
        self.item_rows = 256 if e4m3 else attn_effective_rows(int(item_rows), N, B * Hq, _lib.num_sms(q.device),
                                                              d=D, m=M)
        self.kv_slots = attn_kv_slots(64 if e4m3 else D, kv_stages, self.item_rows // 128)  # e4m3: D=64-sized tiles
        self.args = a
        self.shape = (B, Hq, Hkv, N, M, D)
        L = _lib.lib()
        self._ref = C.byref(a)
        # a C-side plan: tensor maps encoded and the kernel loaded once; a launch is
        # one indirect call (nt_attn_plan_launch)
        handle = C.c_void_p()
        _lib.check(L.nt_attn_plan_create(self._ref, C.byref(handle)), "nt_attn_plan_create")
        self._plan = handle
        self._destroy = L.nt_attn_plan_destroy
        self._fn = L.nt_attn_plan_launch
        self.ctas_per_sm = int(L.nt_attn_resident_ctas(self._ref))

    def launch(self, stream=None) -> None:
        st = self._fn(self._plan, _stream_handle(stream))
        if st:
            _lib.check(st, "nt_attn_plan_launch")

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                self._destroy(plan)
            except Exception:  # interpreter shutdown: the library may already be gone
                pass
            self._plan = None

    def flops(self) -> float:
        B, Hq, _, N, M, D = self.shape
        if self.mask_kind == "causal":
            # exact count of unmasked (i, j) pairs for top-left causal (j <= i + off)
            off = int(self.args.causal_offset)
            pairs = _causal_pairs(N, M, off)
            return 4.0 * B * Hq * D * pairs
        return 4.0 * B * Hq * N * M * D

    def check_errors(self) -> None:
        flag = int(self.err.item())
        if flag & 1:
            raise DivisionByZero("tile divide: softmax denominator is zero (row fully masked)")
        if flag >> 8:
            raise RuntimeError(f"device pipeline timeout (wait codes {[c for c in range(16) if flag >> (8 + c) & 1]})")


def pack_mask_bits(mask: torch.Tensor, stream=None):
    """fp32 CUDA Mask [N, M] -> (int32 [N, ceil(M/128)*4] visibility bits, pure) where
    ``pure`` says every value was 0 or -inf (only then may K1 use NT_MASK_BITS)."""
    if mask.dtype != torch.float32 or not mask.is_cuda or mask.dim() != 2 or mask.stride(-1) != 1:
        raise InvalidArguments("mask must be a CUDA fp32 [N, M] tensor with unit column stride")
    n, m = mask.shape
    words = -(-m // 128) * 4
    bits = torch.empty((n, words), dtype=torch.int32, device=mask.device)
    flag = torch.zeros(1, dtype=torch.int32, device=mask.device)
    _lib.check(_lib.lib().nt_mask_to_bits(mask.data_ptr(), n, m, mask.stride(0), bits.data_ptr(), words,
                                          flag.data_ptr(), _stream_handle(stream)), "nt_mask_to_bits")
    return bits, int(flag.item()) == 0


def attn_kv_slots(d: int, ma_stages: int, nq: int = 2) -> int:
    """K/V ring slots K1 uses for an MA `stages` value (csrc/attn_fwd.cuh attn_kv_slots)."""
    st = ma_stages if ma_stages > 0 else 2
    if nq == 1:
        return 2 if d == 128 else (2 if st <= 1 else 4)
    if d == 128:
        return 2 if st <= 1 else 4
    return 4 if st <= 1 else 8


def _causal_pairs(N: int, M: int, off: int) -> int:
    """sum_i clamp(i + off + 1, 0, M): unmasked (query, key) pairs of a causal mask."""
    import numpy as np
    return int(np.clip(np.arange(N, dtype=np.int64) + off + 1, 0, M).sum())


class DecodePlan:
    """K2 split-KV decode over [B, Hq, Nq, 128] queries ((Hq/Hkv) * Nq in {1, 2, 4, 8} rows per kv group).

    An FP8 KV cache: q, k, v all ``torch.float8_e4m3fn`` with per-tensor
    descales, S = (q k^T) q_descale k_descale scale, O = v_descale softmax(S) V
    (the same contract as AttentionPlan's e4m3 inputs; P rounded to e4m3).
    """

    def __init__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor,
                 scale: Optional[float], num_splits: int = 0, err_flag: Optional[torch.Tensor] = None,
                 q_descale: float = 1.0, k_descale: float = 1.0, v_descale: float = 1.0):
        q, k, v, o = _as4(q), _as4(k), _as4(v), _as4(o)
        e4m3 = q.dtype == torch.float8_e4m3fn
        want = torch.float8_e4m3fn if e4m3 else torch.bfloat16
        for name, t in (("q", q), ("k", k), ("v", v)):
            if t.dtype != want or not t.is_cuda:
                raise InvalidArguments(f"{name} must be a CUDA bf16 tensor (or q, k, v all float8_e4m3fn)")
        if o.dtype not in (torch.bfloat16, torch.float32):
            raise InvalidArguments("o must be bf16 or fp32")
        B, Hq, Nq, D = q.shape
        _, Hkv, M, _ = k.shape
        if tuple(v.shape) != (B, Hkv, M, D) or tuple(o.shape) != (B, Hq, Nq, D) or Hq % Hkv:
            raise InvalidArguments("q/k/v/o shapes inconsistent")
        L = _lib.lib()
        splits = int(L.nt_decode_num_splits(B, Hkv, M, int(num_splits)))
        rows = (Hq // Hkv) * Nq
        ws_bytes = int(L.nt_decode_workspace_bytes(B, Hkv, rows, D, splits))
        self.ws = torch.empty(max(ws_bytes // 4, 1), dtype=torch.float32, device=q.device)
        self.err = err_flag if err_flag is not None else torch.zeros(1, dtype=torch.int32, device=q.device)
        a = _lib.DecodeArgs()
        a.q, a.k, a.v, a.o = _t4(q), _t4(k), _t4(v), _t4(o)
        a.batch, a.heads_q, a.heads_kv, a.seq_q, a.seq_kv, a.head_dim = B, Hq, Hkv, Nq, M, D
        a.scale = 1.0 if scale is None else float(scale)
        a.num_splits = splits
        a.out_dtype = _lib.NT_DTYPE_F32 if o.dtype == torch.float32 else _lib.NT_DTYPE_BF16
        a.workspace = self.ws.data_ptr()
        a.workspace_bytes = self.ws.numel() * 4
        a.err_flag = self.err.data_ptr()
        a.in_dtype = _lib.NT_DTYPE_E4M3 if e4m3 else _lib.NT_DTYPE_BF16
        a.q_descale, a.k_descale, a.v_descale = float(q_descale), float(k_descale), float(v_descale)
        self.args, self.splits = a, splits
        self.tensors = (q, k, v, o)
        self.shape = (B, Hq, Hkv, Nq, M, D)
        self.elem_bytes = 1 if e4m3 else 2
        self._fn = L.nt_attn_decode
        self._ref = C.byref(a)
        self.mask_kind = "none"

    def launch(self, stream=None) -> None:
        st = self._fn(self._ref, _stream_handle(stream))
        if st:
            _lib.check(st, "nt_attn_decode")

    def flops(self) -> float:
        B, Hq, _, Nq, M, D = self.shape
        return 4.0 * B * Hq * Nq * M * D

    def kv_bytes(self) -> int:
        B, _, Hkv, _, M, D = self.shape
        return 2 * B * Hkv * M * D * self.elem_bytes

    def check_errors(self) -> None:
        if int(self.err.item()) & 1:
            raise DivisionByZero("tile divide: softmax denominator is zero")


class PagedDecodePlan:
    """K2 split-KV decode over a paged KV cache (nt_attn_decode_paged).

    ``k_pages`` / ``v_pages``: bf16 page pools, ``layout="NHD"`` ->
    [num_pages, page_size, Hkv, 128] or ``"HND"`` -> [num_pages, Hkv, page_size, 128]
    (any strides with the head dim contiguous).  ``block_table``: int32
    [B, max_pages]; ``seq_lens``: int32 [B] keys per sequence.  ``q`` / ``o``:
    [B, Hq, Nq, 128].  The MA program is the dense decode kernel; paging is how
    a serving runtime lays out its K/V buffers.  An FP8 cache: q and both pools
    ``torch.float8_e4m3fn`` with per-tensor descales (DecodePlan's contract), page
    sizes dividing or a multiple of 128.
    """

    def __init__(self, q: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor, block_table: torch.Tensor,
                 seq_lens: torch.Tensor, o: torch.Tensor, scale: Optional[float], layout: str = "NHD",
                 max_seq_kv: Optional[int] = None, num_splits: int = 0, err_flag: Optional[torch.Tensor] = None,
                 q_descale: float = 1.0, k_descale: float = 1.0, v_descale: float = 1.0):
        q, o = _as4(q), _as4(o)
        e4m3 = q.dtype == torch.float8_e4m3fn
        want = torch.float8_e4m3fn if e4m3 else torch.bfloat16
        for name, t in (("q", q), ("k_pages", k_pages), ("v_pages", v_pages)):
            if t.dtype != want or not t.is_cuda:
                raise InvalidArguments(f"{name} must be a CUDA bf16 tensor (or q and both pools float8_e4m3fn)")
        if k_pages.shape != v_pages.shape or k_pages.stride() != v_pages.stride() or k_pages.dim() != 4:
            raise InvalidArguments("k_pages / v_pages must be rank-4 pools of identical shape and strides")
        if block_table.dtype != torch.int32 or seq_lens.dtype != torch.int32:
            raise InvalidArguments("block_table and seq_lens must be int32")
        if layout == "NHD":
            P, ps, Hkv, D = k_pages.shape
            sp, st, sh = k_pages.stride(0), k_pages.stride(1), k_pages.stride(2)
        elif layout == "HND":
            P, Hkv, ps, D = k_pages.shape
            sp, sh, st = k_pages.stride(0), k_pages.stride(1), k_pages.stride(2)
        else:
            raise InvalidArguments("layout must be 'NHD' or 'HND'")
        B, Hq, Nq, Dq = q.shape
        if Dq != D or k_pages.stride(-1) != 1 or tuple(o.shape) != (B, Hq, Nq, D) or Hq % Hkv:
            raise InvalidArguments("q/o/page shapes inconsistent")
        bt = block_table.contiguous()
        if bt.dim() != 2 or bt.shape[0] != B or seq_lens.shape != (B,):
            raise InvalidArguments("block_table must be [B, max_pages] and seq_lens [B]")
        M = int(max_seq_kv) if max_seq_kv is not None else int(bt.shape[1]) * ps
        L = _lib.lib()
        splits = int(L.nt_decode_num_splits(B, Hkv, M, int(num_splits)))
        rows = (Hq // Hkv) * Nq
        ws_bytes = int(L.nt_decode_workspace_bytes(B, Hkv, rows, D, splits))
        self.ws = torch.empty(max(ws_bytes // 4, 1), dtype=torch.float32, device=q.device)
        self.err = err_flag if err_flag is not None else torch.zeros(1, dtype=torch.int32, device=q.device)
        a = _lib.DecodePagedArgs()
        a.q, a.o = _t4(q), _t4(o)
        a.k_pages, a.v_pages = k_pages.data_ptr(), v_pages.data_ptr()
        a.page_stride, a.token_stride, a.head_stride = sp, st, sh
        a.num_pages, a.page_size = P, ps
        a.block_table, a.block_table_stride = bt.data_ptr(), bt.stride(0)
        a.seq_lens = seq_lens.data_ptr()
        a.batch, a.heads_q, a.heads_kv, a.seq_q, a.max_seq_kv, a.head_dim = B, Hq, Hkv, Nq, M, D
        a.scale = 1.0 if scale is None else float(scale)
        a.num_splits = splits
        a.out_dtype = _lib.NT_DTYPE_F32 if o.dtype == torch.float32 else _lib.NT_DTYPE_BF16
        a.workspace = self.ws.data_ptr()
        a.workspace_bytes = self.ws.numel() * 4
        a.err_flag = self.err.data_ptr()
        a.in_dtype = _lib.NT_DTYPE_E4M3 if e4m3 else _lib.NT_DTYPE_BF16
        a.q_descale, a.k_descale, a.v_descale = float(q_descale), float(k_descale), float(v_descale)
        self.elem_bytes = 1 if e4m3 else 2
        self.args, self.splits = a, splits
        self.tensors = (q, k_pages, v_pages, bt, seq_lens, o)
        self.shape = (B, Hq, Hkv, Nq, M, D)
        self._fn = L.nt_attn_decode_paged
        self._ref = C.byref(a)
        self.mask_kind = "none"

    def launch(self, stream=None) -> None:
        st = self._fn(self._ref, _stream_handle(stream))
        if st:
            _lib.check(st, "nt_attn_decode_paged")

    def kv_bytes(self) -> int:
        """K+V bytes the launch streams: every sequence's keys (seq_lens, read on the host)."""
        _, _, Hkv, _, _, D = self.shape
        return int(self.tensors[4].sum().item()) * Hkv * D * 2 * self.elem_bytes

    def check_errors(self) -> None:
        if int(self.err.item()) & 1:
            raise DivisionByZero("tile divide: softmax denominator is zero (empty sequence)")


def decode_eligible(n_rows_per_group: int, d: int, mask_kind: str) -> bool:
    return mask_kind == "none" and d == 128 and n_rows_per_group in (1, 2, 4, 8)
