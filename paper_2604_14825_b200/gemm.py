"""GEMM-chain realisation (config 2): fused K3b when Y fits TMEM, else two K3 GEMMs.

The MA kernel computes per 64-row block
``T = dot(X_rows, W1[:, f-tile])`` then ``Y += dot(T, W2[f-tile, :])`` with Y
read-modify-written in Global every iteration.  On B200:

* E <= 256 and N < 2048: ``nt_gemm_chain`` keeps T and the Y accumulator in
  TMEM (one fused kernel, T rounded to bf16 as the second MMA's operand);
  with N >= 2048 rows the two-GEMM realisation fills the machine better and
  wins despite the T round trip through HBM (B200 A/B, ``tools/chain_ab.py``:
  4096^3 x 128: fused 207 us, two GEMMs 124 us; 1024 x 4096^2 x 128: fused
  49 us, two GEMMs 52 us);
* E > 256 (BASELINE config 2 at E=4096, schedulable only with
  max_tile_elems >= 262144): the 128 x E fp32 accumulator
  cannot live in TMEM, so the same MA is realised as T = X.W1 (bf16) then
  Y = T.W2 -- the sum over j0 of the MA equals the second GEMM's K loop.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import InvalidArguments
from .recognize import GemmChainSpec


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def _mat(t: torch.Tensor, name: str):
    if t.dim() != 2 or t.stride(1) != 1:
        raise InvalidArguments(f"{name} must be a row-major 2-D tensor")
    return t.data_ptr(), t.stride(0)


class GemmPlan:
    """C = A . B with bf16 A [M,K], B [K,N]; C bf16/fp32 [M,N]."""

    def __init__(self, a: torch.Tensor, b: torch.Tensor, c: torch.Tensor):
        if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
            raise InvalidArguments("A and B must be bf16")
        M, K = a.shape
        K2, N = b.shape
        if K2 != K or tuple(c.shape) != (M, N):
            raise InvalidArguments("GEMM shapes inconsistent")
        g = _lib.GemmArgs()
        g.a, g.lda = _mat(a, "A")
        g.b, g.ldb = _mat(b, "B")
        g.c, g.ldc = _mat(c, "C")
        g.m, g.n, g.k = M, N, K
        g.out_dtype = _lib.NT_DTYPE_F32 if c.dtype == torch.float32 else _lib.NT_DTYPE_BF16
        # split K over CTAs for few-tile shapes (fp32 partials + one reduce launch)
        L = _lib.lib()
        g.k_splits = int(L.nt_gemm_k_splits(M, N, K)) if c.is_contiguous() else 1
        ws = int(L.nt_gemm_workspace_bytes(M, N, K)) if g.k_splits > 1 else 0
        self.ws = torch.empty(max(ws // 4, 1), dtype=torch.float32, device=a.device) if ws else None
        g.workspace = self.ws.data_ptr() if ws else None
        g.workspace_bytes = self.ws.numel() * 4 if ws else 0
        if not ws:
            g.k_splits = 1
        self.args, self.tensors = g, (a, b, c)
        self._ref = C.byref(g)
        self._fn = _lib.lib().nt_gemm
        self.flops = 2.0 * M * N * K

    def launch(self, stream=None):
        st = self._fn(self._ref, _stream(stream))
        if st:
            _lib.check(st, "nt_gemm")


FUSED_MAX_ROWS = 2048


class ChainPlan:
    """Y = (X . W1) . W2 -- fused (E <= 256) or as two GEMMs."""

    def __init__(self, x: torch.Tensor, w1: torch.Tensor, w2: torch.Tensor, y: torch.Tensor,
                 force_two_gemms: bool = False):
        N, K = x.shape
        K2, F = w1.shape
        F2, E = w2.shape
        if K2 != K or F2 != F or tuple(y.shape) != (N, E):
            raise InvalidArguments("GEMM chain shapes inconsistent")
        self.flops = 2.0 * N * K * F + 2.0 * N * F * E
        self.fused = E <= 256 and N < FUSED_MAX_ROWS and not force_two_gemms
        self.tensors = (x, w1, w2, y)
        if self.fused:
            c = _lib.ChainArgs()
            c.x, c.ldx = _mat(x, "X")
            c.w1, c.ldw1 = _mat(w1, "W1")
            c.w2, c.ldw2 = _mat(w2, "W2")
            c.y, c.ldy = _mat(y, "Y")
            c.n, c.k, c.f, c.e = N, K, F, E
            c.out_dtype = _lib.NT_DTYPE_F32 if y.dtype == torch.float32 else _lib.NT_DTYPE_BF16
            ws = int(_lib.lib().nt_gemm_chain_workspace_bytes(N, F, E))
            self.ws = torch.empty(max(ws // 4, 1), dtype=torch.float32, device=x.device)
            c.workspace = self.ws.data_ptr() if ws else None
            c.workspace_bytes = self.ws.numel() * 4
            self.args = c
            self._ref = C.byref(c)
            self._fn = _lib.lib().nt_gemm_chain
        else:
            self.t = torch.empty((N, F), dtype=torch.bfloat16, device=x.device)
            self.g1 = GemmPlan(x, w1, self.t)
            self.g2 = GemmPlan(self.t, w2, y)

    @property
    def realisation(self) -> str:
        return "chain_fused" if self.fused else "gemm x2"

    def launch(self, stream=None):
        if self.fused:
            st = self._fn(self._ref, _stream(stream))
            if st:
                _lib.check(st, "nt_gemm_chain")
        else:
            self.g1.launch(stream)
            self.g2.launch(stream)


def run_gemm_chain(spec: GemmChainSpec, inputs: dict, dev, out_dtype=None):
    from .executor import _to_device, to_bf16

    x = to_bf16(_to_device(inputs[spec.x], dev, spec.x))
    w1 = to_bf16(_to_device(inputs[spec.w1], dev, spec.w1))
    w2 = to_bf16(_to_device(inputs[spec.w2], dev, spec.w2))
    for nm, t, shp in ((spec.x, x, (spec.n, spec.k)), (spec.w1, w1, (spec.k, spec.f)),
                       (spec.w2, w2, (spec.f, spec.e))):
        if tuple(t.shape) != shp:
            from .errors import OutOfBounds
            raise OutOfBounds(f"input {nm!r}: wrong shape {tuple(t.shape)}")
    odt = torch.float32 if out_dtype in (None, "fp32", torch.float32) else torch.bfloat16
    y = torch.empty((spec.n, spec.e), dtype=odt, device=dev)
    plan = ChainPlan(x, w1, w2, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.launch()
    e1.record()
    e1.synchronize()
    info = {"kernel": plan.realisation, "ma_tile": (spec.block_m, spec.block_f), "gpu_tile": (128, 128)}
    return y, e0.elapsed_time(e1), plan.flops, info
