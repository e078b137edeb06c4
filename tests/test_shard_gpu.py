"""Simulated ranks on one GPU: every rank's shard runs through the real launch plan.

Each rank's ``plan_shard`` / ``plan_row_shard`` slice is launched as its own
AttentionPlan / DecodePlan / ChainPlan (exactly what that rank executes under
torchrun), the per-rank outputs are reassembled with the gather's own
``assemble`` / ``assemble_rows``, and the result is compared with the
unsharded launch: bitwise where neither side splits KV (the per-(b, h) item
math is then identical), else within the BASELINE tolerance against the
unsharded output and the fp64 oracle.
"""

import numpy as np
import pytest
import torch

from oracle import reference_math

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2


def _rnd(shape, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.randn(shape, generator=g, device="cuda").bfloat16()


def _err(a, b):
    a, b = a.double().cpu().numpy(), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b))), float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("B,Hq,Hkv,N,D,causal,world", [
    (1, 32, 8, 2048, 128, True, 8),     # Llama GQA, one kv-group per rank (split-KV units on the shards)
    (1, 32, 8, 1024, 128, True, 2),
    (4, 12, 12, 512, 64, False, 4),     # BERT-like batch split
    (2, 8, 2, 768, 128, False, 2),
])
def test_attention_shards_equal_unsharded(B, Hq, Hkv, N, D, causal, world):
    from paper_2604_14825_b200.runtime import AttentionPlan
    from paper_2604_14825_b200.shard import assemble, plan_shard

    q, k, v = _rnd((B, Hq, N, D), 1), _rnd((B, Hkv, N, D), 2), _rnd((B, Hkv, N, D), 3)
    kind = "causal" if causal else "none"
    scale = 1 / D ** 0.5
    full = torch.empty((B, Hq, N, D), dtype=torch.float32, device="cuda")
    pf = AttentionPlan(q, k, v, full, scale, kind)
    pf.launch()
    g = Hq // Hkv
    parts, split_any = [], pf.ws is not None
    for r in range(world):
        sh = plan_shard(B, Hkv, world, r)
        q0, q1 = sh.q_heads(g)
        o = torch.empty((sh.b1 - sh.b0, q1 - q0, N, D), dtype=torch.float32, device="cuda")
        p = AttentionPlan(q[sh.b0:sh.b1, q0:q1], k[sh.b0:sh.b1, sh.h0:sh.h1], v[sh.b0:sh.b1, sh.h0:sh.h1],
                          o, scale, kind)
        p.launch()
        p.check_errors()
        split_any |= p.ws is not None
        parts.append(o)
    torch.cuda.synchronize()
    pf.check_errors()
    got = assemble(torch.stack(parts, 0), plan_shard(B, Hkv, world, 0).axis)
    assert got.shape == full.shape
    if not split_any:
        assert torch.equal(got, full)
    ref = reference_math.attention_batched_fp64(q.double().cpu().numpy(), k.double().cpu().numpy(),
                                                v.double().cpu().numpy(), scale, causal)
    for t in (got, full):
        e, r = _err(t, ref)
        assert e <= MAX_ABS and r <= REL_L2, (e, r)
    e, r = _err(got, full.double().cpu().numpy())
    assert e <= MAX_ABS and r <= REL_L2, (e, r)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_decode_shards_equal_unsharded(world):
    from paper_2604_14825_b200.runtime import DecodePlan
    from paper_2604_14825_b200.shard import assemble, plan_shard

    B, Hkv, g, M, D = 8, 8, 4, 4096, 128
    q, k, v = _rnd((B, Hkv, g, D), 4), _rnd((B, Hkv, M, D), 5), _rnd((B, Hkv, M, D), 6)
    full = torch.empty((B, Hkv, g, D), dtype=torch.float32, device="cuda")
    DecodePlan(q, k, v, full, 1 / D ** 0.5).launch()
    parts = []
    for r in range(world):
        sh = plan_shard(B, Hkv, world, r)
        o = torch.empty((sh.b1 - sh.b0, sh.h1 - sh.h0, g, D), dtype=torch.float32, device="cuda")
        DecodePlan(q[sh.b0:sh.b1, sh.h0:sh.h1], k[sh.b0:sh.b1, sh.h0:sh.h1], v[sh.b0:sh.b1, sh.h0:sh.h1], o,
                   1 / D ** 0.5).launch()
        parts.append(o)
    torch.cuda.synchronize()
    got = assemble(torch.stack(parts, 0), plan_shard(B, Hkv, world, 0).axis)
    ref = reference_math.attention_batched_fp64(q.double().cpu().numpy(), k.double().cpu().numpy(),
                                                v.double().cpu().numpy(), 1 / D ** 0.5, False)
    for t in (got, full):
        e, r = _err(t, ref)
        assert e <= MAX_ABS and r <= REL_L2, (e, r)


@pytest.mark.parametrize("rows,E,world", [(1024, 128, 2), (1000, 128, 4), (2048, 512, 2)])
def test_chain_row_shards_equal_unsharded(rows, E, world):
    from paper_2604_14825_b200.gemm import ChainPlan
    from paper_2604_14825_b200.shard import assemble_rows, plan_row_shard

    K = F = 512
    x = _rnd((rows, K), 7)
    w1 = (_rnd((K, F), 8).float() / K ** 0.5).bfloat16()
    w2 = (_rnd((F, E), 9).float() / F ** 0.5).bfloat16()
    full = torch.empty((rows, E), dtype=torch.float32, device="cuda")
    ChainPlan(x, w1, w2, full).launch()
    parts = []
    for r in range(world):
        s = plan_row_shard(rows, world, r)
        y = torch.empty((s.r1 - s.r0, E), dtype=torch.float32, device="cuda")
        ChainPlan(x[s.r0:s.r1], w1, w2, y).launch()
        parts.append(y)
    torch.cuda.synchronize()
    got = assemble_rows(parts, rows)
    # fp64 of the realised arithmetic: T = X.W1 rounded to bf16, then T.W2
    t = (x.double() @ w1.double()).bfloat16().double()
    ref = (t @ w2.double()).cpu().numpy()
    for y in (got, full):
        e, r = _err(y, ref)
        assert e <= MAX_ABS and r <= REL_L2, (e, r)
    e, r = _err(got, full.double().cpu().numpy())
    assert e <= MAX_ABS and r <= REL_L2, (e, r)
