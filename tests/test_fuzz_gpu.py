"""Seeded random shapes through K1 and K2b against the float64 oracle (GPU).

Each case draws batch / heads / GQA ratio / lengths (ragged, tiny, N != M) / head dim /
mask kind / output dtype / item rows / ring depth (K1) or rows per group / splits /
dense or paged cache / page size / layout (K2b) from a fixed seed, so failures
reproduce; the bound is the BASELINE tolerance.
"""

import numpy as np
import pytest
import torch

from oracle import reference_math
from oracle.ma_interp import round_bf16

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2


def _check(got, ref):
    got = np.asarray(got, np.float64)
    assert np.all(np.isfinite(got))
    mx = float(np.max(np.abs(got - ref)))
    rl = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    assert mx <= MAX_ABS and rl <= REL_L2, (mx, rl)


def _k1_case(seed):
    g = np.random.default_rng(1000 + seed)
    D = int(g.choice([64, 128]))
    hkv = int(g.choice([1, 2, 3]))
    Hq = hkv * int(g.choice([1, 2, 4]))
    B = int(g.integers(1, 3))
    N = int(g.choice([1, 7, 100, 128, 255, 256, 300, 513, 1000, 1500]))
    M = N if g.random() < 0.5 else int(g.choice([1, 64, 129, 384, 700, 1300]))
    kind = str(g.choice(["none", "causal", "tensor", "bits"]))
    if kind == "causal":
        M = max(M, N)  # top-left causal: every row keeps key 0
    f32 = bool(g.random() < 0.5)
    rows = int(g.choice([0, 128, 256]))
    stages = int(g.choice([1, 2, 4]))
    return B, Hq, hkv, N, M, D, kind, f32, rows, stages


@pytest.mark.parametrize("seed", range(64))
def test_k1_random_shapes_vs_fp64(seed):
    from paper_2604_14825_b200.runtime import AttentionPlan, pack_mask_bits

    B, Hq, Hkv, N, M, D, kind, f32, rows, stages = _k1_case(seed)
    g = np.random.default_rng(seed)
    q = round_bf16(g.standard_normal((B, Hq, N, D)))
    k = round_bf16(g.standard_normal((B, Hkv, M, D)))
    v = round_bf16(g.standard_normal((B, Hkv, M, D)))
    dev = torch.device("cuda")
    mask_np = mt = None
    if kind in ("tensor", "bits"):
        mask_np = np.where(g.random((N, M)) < 0.4, -np.inf, 0.0).astype(np.float32)
        mask_np[:, 0] = 0.0
        mt = torch.from_numpy(mask_np).to(dev)
        if kind == "bits":
            mt = pack_mask_bits(mt)[0]
    o = torch.full((B, Hq, N, D), float("nan"), dtype=torch.float32 if f32 else torch.bfloat16, device=dev)
    plan = AttentionPlan(*(torch.from_numpy(x).to(dev).bfloat16() for x in (q, k, v)), o, D ** -0.5, kind, mt,
                         kv_stages=stages, item_rows=rows)
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    if mask_np is not None:
        ref = np.stack([np.stack([reference_math.attention_fp64(q[b, h], k[b, h // (Hq // Hkv)],
                                                                v[b, h // (Hq // Hkv)], D ** -0.5, mask_np)
                                  for h in range(Hq)]) for b in range(B)])
    else:
        ref = reference_math.attention_batched_fp64(q, k, v, D ** -0.5, kind == "causal")
    _check(o.float().cpu().numpy(), ref)


@pytest.mark.parametrize("seed", range(48))
def test_k2b_random_decode_vs_fp64(seed):
    from paper_2604_14825_b200.runtime import DecodePlan, PagedDecodePlan

    g = np.random.default_rng(2000 + seed)
    D = 128
    Hkv = int(g.choice([1, 2, 4]))
    gq = int(g.choice([1, 2, 4, 8]))
    Nq = int(g.choice([1, 2])) if gq <= 4 else 1
    Hq = Hkv * gq
    B = int(g.integers(1, 4))
    M = int(g.choice([1, 63, 128, 500, 1024, 3000, 5000]))
    splits = int(g.choice([0, 1, 3, 7]))
    paged = bool(g.random() < 0.5)
    q = round_bf16(g.standard_normal((B, Hq, Nq, D)))
    k = round_bf16(g.standard_normal((B, Hkv, M, D)))
    v = round_bf16(g.standard_normal((B, Hkv, M, D)))
    dev = torch.device("cuda")
    o = torch.full((B, Hq, Nq, D), float("nan"), device=dev)
    tq = torch.from_numpy(q).to(dev).bfloat16()
    if not paged:
        plan = DecodePlan(tq, torch.from_numpy(k).to(dev).bfloat16(), torch.from_numpy(v).to(dev).bfloat16(), o,
                          D ** -0.5, num_splits=splits)
        lens = [M] * B
    else:
        ps = int(g.choice([8, 16, 32, 64, 128, 256]))
        layout = str(g.choice(["NHD", "HND"]))
        lens = [int(x) for x in g.integers(1, M + 1, B)]
        npp = -(-M // ps)
        P = B * npp + 3
        perm = g.permutation(P)[: B * npp].reshape(B, npp)
        shape = (P, ps, Hkv, D) if layout == "NHD" else (P, Hkv, ps, D)
        kp = np.zeros(shape, np.float32)
        vp = np.zeros(shape, np.float32)
        for b in range(B):
            for j in range(npp):
                lo, hi = j * ps, min(M, (j + 1) * ps)
                if layout == "NHD":
                    kp[perm[b, j], : hi - lo] = k[b, :, lo:hi].transpose(1, 0, 2)
                    vp[perm[b, j], : hi - lo] = v[b, :, lo:hi].transpose(1, 0, 2)
                else:
                    kp[perm[b, j], :, : hi - lo] = k[b, :, lo:hi]
                    vp[perm[b, j], :, : hi - lo] = v[b, :, lo:hi]
        plan = PagedDecodePlan(tq, torch.from_numpy(kp).to(dev).bfloat16(), torch.from_numpy(vp).to(dev).bfloat16(),
                               torch.from_numpy(perm.astype(np.int32)).to(dev),
                               torch.tensor(lens, dtype=torch.int32, device=dev), o, D ** -0.5, layout=layout,
                               max_seq_kv=M, num_splits=splits)
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    got = o.cpu().numpy()
    for b in range(B):
        ref = reference_math.attention_batched_fp64(q[b:b + 1], k[b:b + 1, :, :lens[b]], v[b:b + 1, :, :lens[b]],
                                                    D ** -0.5, False)
        _check(got[b:b + 1], ref)
