"""K2 split-KV decode on the B200 vs the CPU oracle (need a GPU)."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import reference_math
from oracle.ma_interp import round_bf16

pytestmark = pytest.mark.gpu


def _check(got, ref, max_abs=2e-2, rel=1e-2):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert np.all(np.isfinite(got))
    mx = float(np.max(np.abs(got - ref)))
    rl = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert mx <= max_abs and rl <= rel, (mx, rl)


@pytest.mark.parametrize("case", ["decode4", "decode1", "b200_decode4"])
def test_execute_ma_decode_matches_reference(case):
    from paper_2604_14825_b200 import execute_ma

    mod, inputs, interp32, ref64 = load_golden(case)
    bufs, rep = execute_ma(mod, inputs)
    assert rep.realisation[0]["kernel"] == "attn_decode_splitkv"
    _check(bufs[mod.output], interp32)
    _check(bufs[mod.output], ref64)


@pytest.mark.parametrize("B,Hq,Hkv,Nq,M,splits", [(2, 8, 2, 1, 4096, 0), (3, 4, 4, 2, 3000, 0),
                                                  (1, 16, 2, 1, 20000, 7), (2, 4, 1, 1, 777, 3),
                                                  (1, 2, 2, 1, 64, 0)])
def test_decode_vs_fp64(B, Hq, Hkv, Nq, M, splits):
    from paper_2604_14825_b200.runtime import DecodePlan

    D = 128
    g = np.random.default_rng(B * 1000 + M)
    q = round_bf16(g.standard_normal((B, Hq, Nq, D)))
    k = round_bf16(g.standard_normal((B, Hkv, M, D)))
    v = round_bf16(g.standard_normal((B, Hkv, M, D)))
    tq, tk, tv = (torch.from_numpy(x).cuda().bfloat16() for x in (q, k, v))
    o = torch.empty((B, Hq, Nq, D), dtype=torch.float32, device="cuda")
    plan = DecodePlan(tq, tk, tv, o, 1 / np.sqrt(D), num_splits=splits)
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    ref = reference_math.attention_batched_fp64(q, k, v, 1 / np.sqrt(D), False)
    _check(o.cpu().numpy(), ref)


def _paged_cache(k, v, page_size, layout, seed):
    """Scatter dense [B, Hkv, M, D] K/V into shuffled page pools + block table."""
    B, Hkv, M, D = k.shape
    npp = -(-M // page_size)
    P = B * npp + 3  # a few spare pages
    perm = np.random.default_rng(seed).permutation(P)[: B * npp].reshape(B, npp)
    shape = (P, page_size, Hkv, D) if layout == "NHD" else (P, Hkv, page_size, D)
    kp = np.zeros(shape, np.float32)
    vp = np.zeros(shape, np.float32)
    for b in range(B):
        for i in range(npp):
            lo, hi = i * page_size, min(M, (i + 1) * page_size)
            ks = k[b, :, lo:hi]  # [Hkv, n, D]
            vs = v[b, :, lo:hi]
            if layout == "NHD":
                kp[perm[b, i], : hi - lo] = ks.transpose(1, 0, 2)
                vp[perm[b, i], : hi - lo] = vs.transpose(1, 0, 2)
            else:
                kp[perm[b, i], :, : hi - lo] = ks
                vp[perm[b, i], :, : hi - lo] = vs
    return kp, vp, perm.astype(np.int32)


@pytest.mark.parametrize("page_size,layout", [(16, "NHD"), (64, "HND"), (128, "NHD"), (8, "HND")])
def test_paged_decode_vs_fp64(page_size, layout):
    """Paged KV cache (block table, ragged seq_lens) == dense attention over each sequence's prefix."""
    from paper_2604_14825_b200.runtime import PagedDecodePlan

    B, Hq, Hkv, Nq, M, D = 4, 16, 4, 1, 2304, 128
    g = np.random.default_rng(page_size)
    q = round_bf16(g.standard_normal((B, Hq, Nq, D)))
    k = round_bf16(g.standard_normal((B, Hkv, M, D)))
    v = round_bf16(g.standard_normal((B, Hkv, M, D)))
    lens = np.array([M, 1, 777, 1500], dtype=np.int32)
    kp, vp, bt = _paged_cache(k, v, page_size, layout, seed=7)
    tq = torch.from_numpy(q).cuda().bfloat16()
    tkp = torch.from_numpy(kp).cuda().bfloat16()
    tvp = torch.from_numpy(vp).cuda().bfloat16()
    o = torch.empty((B, Hq, Nq, D), dtype=torch.float32, device="cuda")
    plan = PagedDecodePlan(tq, tkp, tvp, torch.from_numpy(bt).cuda(), torch.from_numpy(lens).cuda(), o,
                           1 / np.sqrt(D), layout=layout, max_seq_kv=M)
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    got = o.cpu().numpy()
    for b in range(B):
        n = int(lens[b])
        ref = reference_math.attention_batched_fp64(q[b:b + 1], k[b:b + 1, :, :n], v[b:b + 1, :, :n],
                                                    1 / np.sqrt(D), False)
        _check(got[b:b + 1], ref)


def test_paged_decode_matches_dense_kernel_when_splits_match():
    """Same splits, same keys: paged K2 (FMA-pipe dots, fp32 P) and dense K2b (tcgen05,
    P rounded to bf16) agree to the P rounding, and both match fp64."""
    from paper_2604_14825_b200.runtime import DecodePlan, PagedDecodePlan

    B, Hq, Hkv, Nq, M, D = 2, 8, 2, 1, 4096, 128
    g = np.random.default_rng(5)
    q = torch.from_numpy(round_bf16(g.standard_normal((B, Hq, Nq, D)))).cuda().bfloat16()
    k = round_bf16(g.standard_normal((B, Hkv, M, D)))
    v = round_bf16(g.standard_normal((B, Hkv, M, D)))
    kp, vp, bt = _paged_cache(k, v, 64, "NHD", seed=3)
    o1 = torch.empty((B, Hq, Nq, D), dtype=torch.float32, device="cuda")
    o2 = torch.empty_like(o1)
    DecodePlan(q, torch.from_numpy(k).cuda().bfloat16(), torch.from_numpy(v).cuda().bfloat16(), o1,
               0.088, num_splits=6).launch()
    PagedDecodePlan(q, torch.from_numpy(kp).cuda().bfloat16(), torch.from_numpy(vp).cuda().bfloat16(),
                    torch.from_numpy(bt).cuda(), torch.full((B,), M, dtype=torch.int32, device="cuda"), o2,
                    0.088, max_seq_kv=M, num_splits=6).launch()
    torch.cuda.synchronize()
    assert float((o1 - o2).abs().max()) < 5e-3
    ref = reference_math.attention_batched_fp64(q.float().cpu().numpy(), k, v, 0.088, False)
    _check(o1.cpu().numpy(), ref)
    _check(o2.cpu().numpy(), ref)


@pytest.mark.parametrize("Hq,Hkv,Nq,page_size", [(8, 8, 1, 32), (16, 2, 1, 16), (4, 4, 2, 128), (8, 4, 1, 8)])
def test_paged_decode_row_packings(Hq, Hkv, Nq, page_size):
    """R = (Hq/Hkv)*Nq rows per kv group of 1, 8, 2, 2 over paged caches of several page sizes."""
    from paper_2604_14825_b200.runtime import PagedDecodePlan

    B, M, D = 3, 1300, 128
    g = np.random.default_rng(Hq * 100 + page_size)
    q = round_bf16(g.standard_normal((B, Hq, Nq, D)))
    k = round_bf16(g.standard_normal((B, Hkv, M, D)))
    v = round_bf16(g.standard_normal((B, Hkv, M, D)))
    lens = np.array([M, 700, 65], dtype=np.int32)
    kp, vp, bt = _paged_cache(k, v, page_size, "NHD", seed=page_size)
    o = torch.empty((B, Hq, Nq, D), dtype=torch.float32, device="cuda")
    plan = PagedDecodePlan(torch.from_numpy(q).cuda().bfloat16(), torch.from_numpy(kp).cuda().bfloat16(),
                           torch.from_numpy(vp).cuda().bfloat16(), torch.from_numpy(bt).cuda(),
                           torch.from_numpy(lens).cuda(), o, 1 / np.sqrt(D), max_seq_kv=M)
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    got = o.cpu().numpy()
    for b in range(B):
        n = int(lens[b])
        ref = reference_math.attention_batched_fp64(q[b:b + 1], k[b:b + 1, :, :n], v[b:b + 1, :, :n],
                                                    1 / np.sqrt(D), False)
        _check(got[b:b + 1], ref)


def test_paged_decode_empty_sequence_raises():
    """A sequence with no keys has a zero softmax denominator (tilecc/numerics.py:123-126)."""
    from paper_2604_14825_b200.errors import DivisionByZero
    from paper_2604_14825_b200.runtime import PagedDecodePlan

    B, Hq, Hkv, M, D, ps = 2, 4, 1, 256, 128, 64
    g = np.random.default_rng(0)
    q = torch.from_numpy(round_bf16(g.standard_normal((B, Hq, 1, D)))).cuda().bfloat16()
    pool = torch.from_numpy(round_bf16(g.standard_normal((8, ps, Hkv, D)))).cuda().bfloat16()
    bt = torch.arange(8, dtype=torch.int32, device="cuda").reshape(2, 4)
    lens = torch.tensor([256, 0], dtype=torch.int32, device="cuda")
    o = torch.empty((B, Hq, 1, D), dtype=torch.float32, device="cuda")
    plan = PagedDecodePlan(q, pool, pool, bt, lens, o, 0.088, max_seq_kv=M)
    plan.launch()
    torch.cuda.synchronize()
    with pytest.raises(DivisionByZero):
        plan.check_errors()


def test_workspace_smaller_than_required_is_rejected():
    """ABI v2: a workspace_bytes below what the splits need is NT_ERR_INVALID, not an OOB write."""
    from paper_2604_14825_b200.errors import InvalidArguments
    from paper_2604_14825_b200.gemm import GemmPlan
    from paper_2604_14825_b200.runtime import DecodePlan

    D = 128
    q = torch.zeros((1, 4, 1, D), dtype=torch.bfloat16, device="cuda")
    k = torch.zeros((1, 1, 4096, D), dtype=torch.bfloat16, device="cuda")
    o = torch.empty((1, 4, 1, D), dtype=torch.float32, device="cuda")
    plan = DecodePlan(q, k, k, o, 0.1, num_splits=8)
    plan.args.workspace_bytes = 64
    with pytest.raises(InvalidArguments):
        plan.launch()
    # split-K GEMM: k_splits is clamped to what the workspace holds (here: none -> unsplit, still correct)
    a = torch.randn((256, 4096), device="cuda").bfloat16()
    b = (torch.randn((4096, 128), device="cuda") / 64).bfloat16()
    c = torch.empty((256, 128), dtype=torch.float32, device="cuda")
    g = GemmPlan(a, b, c)
    assert g.args.k_splits > 1
    g.args.workspace_bytes = 0
    g.launch()
    torch.cuda.synchronize()
    ref = a.float() @ b.float()
    assert float((c - ref).abs().max()) < 2e-2


# ------------------------------------------------------------ e4m3 (FP8) KV cache
# K2b with kind::f8f6f4: q, k, v in e4m3 with per-tensor descales, P rounded to
# e4m3 before P.V.  Checked, like K1's e4m3 path (test_attention_gpu.py), against
# the fp64 attention of the DEQUANTISED inputs: the bound covers P's 3-bit
# mantissa and fp32 accumulation only.
E4M3_MAX_ABS = 8e-2
E4M3_REL_L2 = 4e-2


def _quant_e4m3(x, amax_target=448.0):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    descale = float(t.abs().max()) / amax_target
    q = (t / descale).to(torch.float8_e4m3fn)
    return q, descale, (q.float() * descale).double().numpy()


@pytest.mark.parametrize("B,Hq,Hkv,Nq,M,splits,out_dtype", [
    (2, 8, 2, 1, 4096, 0, torch.float32),
    (3, 4, 4, 2, 3000, 0, torch.bfloat16),   # ragged tail tile
    (1, 16, 2, 1, 20000, 7, torch.float32),  # 8 rows per group, explicit splits
    (2, 4, 1, 1, 777, 3, torch.float32),
    (1, 2, 2, 1, 64, 0, torch.float32),      # one partial tile
])
def test_e4m3_decode_vs_fp64_of_dequantised_inputs(B, Hq, Hkv, Nq, M, splits, out_dtype):
    from paper_2604_14825_b200.runtime import DecodePlan

    D = 128
    g = np.random.default_rng(7 * B + M)
    q8, qd, qf = _quant_e4m3(g.standard_normal((B, Hq, Nq, D)) * 1.5)
    k8, kd, kf = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    v8, vd, vf = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    o = torch.empty((B, Hq, Nq, D), dtype=out_dtype, device="cuda")
    plan = DecodePlan(q8.cuda(), k8.cuda(), v8.cuda(), o, 1 / np.sqrt(D), num_splits=splits,
                      q_descale=qd, k_descale=kd, v_descale=vd)
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    ref = reference_math.attention_batched_fp64(qf, kf, vf, 1 / np.sqrt(D), False)
    _check(o.float().cpu().numpy(), ref, max_abs=E4M3_MAX_ABS, rel=E4M3_REL_L2)


def test_e4m3_decode_128k_single_sequence():
    """One long sequence: every split holds ~1K keys, the combine merges ~128 partials."""
    from paper_2604_14825_b200.runtime import DecodePlan

    B, Hq, Hkv, M, D = 1, 8, 1, 131072, 128
    g = np.random.default_rng(11)
    q8, qd, qf = _quant_e4m3(g.standard_normal((B, Hq, 1, D)))
    k8, kd, kf = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    v8, vd, vf = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    o = torch.empty((B, Hq, 1, D), dtype=torch.float32, device="cuda")
    plan = DecodePlan(q8.cuda(), k8.cuda(), v8.cuda(), o, 1 / np.sqrt(D), q_descale=qd, k_descale=kd,
                      v_descale=vd)
    assert plan.kv_bytes() == 2 * M * D
    plan.launch()
    torch.cuda.synchronize()
    ref = reference_math.attention_batched_fp64(qf, kf, vf, 1 / np.sqrt(D), False)
    _check(o.cpu().numpy(), ref, max_abs=E4M3_MAX_ABS, rel=E4M3_REL_L2)


def test_e4m3_decode_rejects_mixed_dtypes():
    from paper_2604_14825_b200.errors import InvalidArguments
    from paper_2604_14825_b200.runtime import DecodePlan

    q = torch.zeros((1, 2, 1, 128), dtype=torch.float8_e4m3fn, device="cuda")
    k = torch.zeros((1, 2, 256, 128), dtype=torch.bfloat16, device="cuda")
    o = torch.empty((1, 2, 1, 128), dtype=torch.float32, device="cuda")
    with pytest.raises(InvalidArguments):
        DecodePlan(q, k, k, o, 0.1)


def _paged_e4m3(k8, v8, page_size, layout, seed):
    """e4m3 page pools (as uint8 bytes through the fp32 scatter, then reinterpreted)."""
    kp, vp, bt = _paged_cache(k8.view(torch.uint8).numpy().astype(np.float32),
                              v8.view(torch.uint8).numpy().astype(np.float32), page_size, layout, seed)
    as8 = lambda x: torch.from_numpy(x.astype(np.uint8)).view(torch.float8_e4m3fn).cuda()  # noqa: E731
    return as8(kp), as8(vp), torch.from_numpy(bt).cuda()


@pytest.mark.parametrize("page_size,layout", [(16, "NHD"), (64, "HND"), (128, "NHD"), (256, "HND"), (8, "NHD"),
                                              (32, "HND")])
def test_e4m3_paged_decode_vs_fp64(page_size, layout):
    """FP8 paged cache, ragged sequence lengths, vs fp64 of the dequantised inputs."""
    from paper_2604_14825_b200.runtime import PagedDecodePlan

    B, Hq, Hkv, Nq, M, D = 4, 16, 4, 1, 2304, 128
    g = np.random.default_rng(100 + page_size)
    q8, qd, qf = _quant_e4m3(g.standard_normal((B, Hq, Nq, D)))
    k8, kd, kf = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    v8, vd, vf = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    lens = np.array([M, 1, 777, 1500], dtype=np.int32)
    kp, vp, bt = _paged_e4m3(k8, v8, page_size, layout, seed=9)
    o = torch.empty((B, Hq, Nq, D), dtype=torch.float32, device="cuda")
    plan = PagedDecodePlan(q8.cuda(), kp, vp, bt, torch.from_numpy(lens).cuda(), o, 1 / np.sqrt(D), layout=layout,
                           max_seq_kv=M, q_descale=qd, k_descale=kd, v_descale=vd)
    assert plan.kv_bytes() == int(lens.sum()) * Hkv * D * 2
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    got = o.cpu().numpy()
    for b in range(B):
        n = int(lens[b])
        ref = reference_math.attention_batched_fp64(qf[b:b + 1], kf[b:b + 1, :, :n], vf[b:b + 1, :, :n],
                                                    1 / np.sqrt(D), False)
        _check(got[b:b + 1], ref, max_abs=E4M3_MAX_ABS, rel=E4M3_REL_L2)


def test_e4m3_paged_decode_is_bitwise_the_dense_decode():
    """Same splits, same keys: the page gathers build the dense kernel's shared-memory tiles."""
    from paper_2604_14825_b200.runtime import DecodePlan, PagedDecodePlan

    B, Hq, Hkv, Nq, M, D = 2, 8, 2, 1, 4096, 128
    g = np.random.default_rng(6)
    q8, qd, _ = _quant_e4m3(g.standard_normal((B, Hq, Nq, D)))
    k8, kd, _ = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    v8, vd, _ = _quant_e4m3(g.standard_normal((B, Hkv, M, D)))
    kp, vp, bt = _paged_e4m3(k8, v8, 32, "NHD", seed=4)
    o1 = torch.empty((B, Hq, Nq, D), dtype=torch.float32, device="cuda")
    o2 = torch.empty_like(o1)
    kw = dict(q_descale=qd, k_descale=kd, v_descale=vd)
    DecodePlan(q8.cuda(), k8.cuda(), v8.cuda(), o1, 0.088, num_splits=6, **kw).launch()
    PagedDecodePlan(q8.cuda(), kp, vp, bt, torch.full((B,), M, dtype=torch.int32, device="cuda"), o2, 0.088,
                    max_seq_kv=M, num_splits=6, **kw).launch()
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("e4m3", [False, True])
def test_decode_with_an_empty_split(e4m3):
    """129 keys over 3 splits of 128-key ranges: the third split has no keys (its four
    quarter partials merge to weight 0) and the second holds one key."""
    from paper_2604_14825_b200.runtime import DecodePlan

    B, Hq, Hkv, M, D = 2, 8, 2, 129, 128
    g = np.random.default_rng(129)
    if e4m3:
        (q, qd, qf), (k, kd, kf), (v, vd, vf) = (_quant_e4m3(g.standard_normal(s))
                                                 for s in ((B, Hq, 1, D), (B, Hkv, M, D), (B, Hkv, M, D)))
        kw, tol = dict(q_descale=qd, k_descale=kd, v_descale=vd), dict(max_abs=E4M3_MAX_ABS, rel=E4M3_REL_L2)
    else:
        qf, kf, vf = (round_bf16(g.standard_normal(s)) for s in ((B, Hq, 1, D), (B, Hkv, M, D), (B, Hkv, M, D)))
        q, k, v = (torch.from_numpy(x).bfloat16() for x in (qf, kf, vf))
        kw, tol = {}, {}
    o = torch.empty((B, Hq, 1, D), dtype=torch.float32, device="cuda")
    plan = DecodePlan(q.cuda(), k.cuda(), v.cuda(), o, 1 / np.sqrt(D), num_splits=3, **kw)
    assert plan.splits == 3
    plan.launch()
    torch.cuda.synchronize()
    plan.check_errors()
    ref = reference_math.attention_batched_fp64(qf, kf, vf, 1 / np.sqrt(D), False)
    _check(o.cpu().numpy(), ref, **tol)
