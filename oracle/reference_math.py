"""CPU oracle: fp64 math references for the configuration programs.

TEST INFRASTRUCTURE ONLY (see oracle/ma_interp.py header).

Restates, in vectorised numpy fp64, what ``oracle_eval``
(tilecc/frontend/oracle.py:25-63) computes for the SURVEY Appendix A
programs (naive-loop fp64 evaluation of every def):

* attention (A.1/A.2/A.3): S = Q (K c)^T [+ Mask]; m = rowmax; P = exp(S - m);
  l = rowsum P; O = (P V) / l  -- the defs at tests/conftest.py:16-26 with the
  scale inside the dot operand and the Mask inside max/exp (A.3);
* GEMM chain (A.4): Y = (X W1) W2.

Summation order differs from the naive loops only at fp64 rounding level;
``tests/test_oracle.py`` pins this against the reference's own oracle_eval
output (golden fixtures) with atol 1e-12, the tolerance of the reference's
test_oracle_matches_numpy_attention (tests/test_frontend.py:123-130).
"""

from __future__ import annotations

import numpy as np


def attention_fp64(q, k, v, scale=None, mask=None, causal=False) -> np.ndarray:
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    kk = k * scale if scale is not None else k
    s = q @ kk.T
    if mask is not None:
        s = s + np.asarray(mask, dtype=np.float64)
    if causal:
        n, m = s.shape
        s = np.where(np.arange(m)[None, :] <= np.arange(n)[:, None], s, -np.inf)
    mx = s.max(axis=1, keepdims=True)
    p = np.exp(s - mx)
    return (p @ v) / p.sum(axis=1, keepdims=True)


def attention_batched_fp64(q, k, v, scale=None, causal=False) -> np.ndarray:
    """[B, Hq, N, D] x [B, Hkv, M, D] with GQA head mapping hkv = hq // (Hq/Hkv)."""
    q = np.asarray(q, dtype=np.float64)
    B, Hq, N, D = q.shape
    Hkv = k.shape[1]
    out = np.empty((B, Hq, N, v.shape[-1]), dtype=np.float64)
    g = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            out[b, h] = attention_fp64(q[b, h], k[b, h // g], v[b, h // g], scale, None, causal)
    return out


def gemm_chain_fp64(x, w1, w2) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return (x @ np.asarray(w1, dtype=np.float64)) @ np.asarray(w2, dtype=np.float64)
