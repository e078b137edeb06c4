"""Operator specs (`.te` text) for the BASELINE configurations.

These are the reference-schedulable spellings:

* ``attention`` -- tests/conftest.py:16-26 (config 1);
* ``scaled_0p125`` / ``llama`` -- A.2: the scale sits inside the dot operand
  (``sum(..) * c`` and a separate ``Qs = Q*c`` def crash the reference
  scheduler with IterationMismatch);
* ``llama_causal`` -- A.3: the Mask is added inside ``max`` and ``exp``
  (conftest CAUSAL_SRC yields no seeds);
* ``gemm2`` -- A.4, the two-GEMM chain (config 2).

Batch, heads and GQA are not expressible at realistic sizes in the reference
(SURVEY.md 0.5), so the compiled unit is the 2-D single-head program and the
runtime adds the batch x head (x GQA) outer grid.
"""

ATTENTION = """\
tensor Q[fp32](N, D)
tensor K[fp32](M, D)
tensor V[fp32](M, D)
S(i, j) = sum(k, Q(i, k) * K(j, k))
m(i) = max(j, S(i, j))
P(i, j) = exp(S(i, j) - m(i))
l(i) = sum(j, P(i, j))
O(i, d) = sum(j, P(i, j) * V(j, d)) / l(i)
output O
"""


def scaled_attention(c: float) -> str:
    return f"""\
tensor Q[fp32](N, D)
tensor K[fp32](M, D)
tensor V[fp32](M, D)
S(i, j) = sum(k, Q(i, k) * (K(j, k) * {c!r}))
m(i) = max(j, S(i, j))
P(i, j) = exp(S(i, j) - m(i))
l(i) = sum(j, P(i, j))
O(i, d) = sum(j, P(i, j) * V(j, d)) / l(i)
output O
"""


def masked_attention(c: float) -> str:
    return f"""\
tensor Q[fp32](N, D)
tensor K[fp32](M, D)
tensor V[fp32](M, D)
tensor Mask[fp32](N, M)
S(i, j) = sum(k, Q(i, k) * (K(j, k) * {c!r}))
m(i) = max(j, S(i, j) + Mask(i, j))
P(i, j) = exp(S(i, j) + Mask(i, j) - m(i))
l(i) = sum(j, P(i, j))
O(i, d) = sum(j, P(i, j) * V(j, d)) / l(i)
output O
"""


GEMM2 = """\
tensor X[fp32](N, K)
tensor W1[fp32](K, F)
tensor W2[fp32](F, E)
T(i, j) = sum(k, X(i, k) * W1(k, j))
Y(i, n) = sum(j, T(i, j) * W2(j, n))
output Y
"""

LLAMA_SCALE = 0.08838834764831845  # 1/sqrt(128), exactly as SURVEY.md A.3 writes it

# Natural spellings the reference scheduler cannot fuse without upstream.apply()
# (scale / mask applied after the sum): the reference's own
# CAUSAL_SRC (tests/conftest.py:28-39) and the post-sum scale.
CAUSAL_NATURAL = """\
tensor Q[fp32](N, D)
tensor K[fp32](M, D)
tensor V[fp32](M, D)
tensor Mask[fp32](N, M)
S(i, j) = sum(k, Q(i, k) * K(j, k)) + Mask(i, j)
m(i) = max(j, S(i, j))
P(i, j) = exp(S(i, j) - m(i))
l(i) = sum(j, P(i, j))
O(i, d) = sum(j, P(i, j) * V(j, d)) / l(i)
output O
"""


def scaled_post(c: float, masked: bool = False) -> str:
    mask_decl = "tensor Mask[fp32](N, M)\n" if masked else ""
    mask_add = " + Mask(i, j)" if masked else ""
    return f"""\
tensor Q[fp32](N, D)
tensor K[fp32](M, D)
tensor V[fp32](M, D)
{mask_decl}S(i, j) = sum(k, Q(i, k) * K(j, k)) * {c!r}{mask_add}
m(i) = max(j, S(i, j))
P(i, j) = exp(S(i, j) - m(i))
l(i) = sum(j, P(i, j))
O(i, d) = sum(j, P(i, j) * V(j, d)) / l(i)
output O
"""

PROGRAMS = {
    "attention": ATTENTION,
    "scaled_0p125": scaled_attention(0.125),
    "llama": scaled_attention(LLAMA_SCALE),
    "llama_causal": masked_attention(LLAMA_SCALE),
    "gemm2": GEMM2,
    "causal_natural": CAUSAL_NATURAL,
    "scaled_post_0p125": scaled_post(0.125),
    "llama_causal_natural": scaled_post(LLAMA_SCALE, masked=True),
}
