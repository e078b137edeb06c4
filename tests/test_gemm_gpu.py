"""K3 GEMM / K3b fused chain on the B200 vs the CPU oracle (need a GPU)."""

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


@pytest.mark.parametrize("case", ["gemm_v6", "gemm_v5", "b200_gemm_v6", "b200_gemm_e512"])
def test_execute_ma_gemm_chain_matches_reference(case):
    from paper_2604_14825_b200 import execute_ma

    mod, inputs, interp32, ref64 = load_golden(case)
    bufs, rep = execute_ma(mod, inputs)
    _check(bufs[mod.output], interp32)
    _check(bufs[mod.output], ref64)
    e = inputs[rep.specs[0].w2].shape[1]
    assert rep.realisation[0]["kernel"] == ("chain_fused" if e <= 256 else "gemm x2")


@pytest.mark.parametrize("M,N,K,f32", [(128, 128, 64, True), (256, 512, 512, True), (300, 264, 136, True),
                                       (1024, 768, 1024, False), (4096, 4096, 4096, False)])
def test_gemm_vs_fp64(M, N, K, f32):
    from paper_2604_14825_b200.gemm import GemmPlan

    g = np.random.default_rng(M + N + K)
    a = round_bf16(g.standard_normal((M, K)))
    b = round_bf16(g.standard_normal((K, N)) / np.sqrt(K))
    ta = torch.from_numpy(a).cuda().bfloat16()
    tb = torch.from_numpy(b).cuda().bfloat16()
    c = torch.empty((M, N), dtype=torch.float32 if f32 else torch.bfloat16, device="cuda")
    GemmPlan(ta, tb, c).launch()
    torch.cuda.synchronize()
    ref = a.astype(np.float64) @ b.astype(np.float64)
    _check(c.float().cpu().numpy(), ref, max_abs=3e-2 if not f32 else 2e-2)


@pytest.mark.parametrize("N,K,F,E", [(256, 256, 512, 128), (512, 1024, 1024, 64), (384, 512, 768, 256),
                                     (130, 136, 200, 72)])
def test_fused_chain_vs_fp64(N, K, F, E):
    from paper_2604_14825_b200.gemm import ChainPlan

    g = np.random.default_rng(N + K + F + E)
    x = round_bf16(g.standard_normal((N, K)))
    w1 = round_bf16(g.standard_normal((K, F)) / np.sqrt(K))
    w2 = round_bf16(g.standard_normal((F, E)) / np.sqrt(F))
    tx, t1, t2 = (torch.from_numpy(v).cuda().bfloat16() for v in (x, w1, w2))
    y = torch.empty((N, E), dtype=torch.float32, device="cuda")
    plan = ChainPlan(tx, t1, t2, y)
    assert plan.fused
    plan.launch()
    torch.cuda.synchronize()
    _check(y.cpu().numpy(), reference_math.gemm_chain_fp64(x, w1, w2))


def test_two_gemm_chain_realisation_e4096_shape():
    from paper_2604_14825_b200.gemm import ChainPlan

    N, K, F, E = 512, 1024, 1024, 4096
    g = np.random.default_rng(5)
    x = round_bf16(g.standard_normal((N, K)))
    w1 = round_bf16(g.standard_normal((K, F)) / np.sqrt(K))
    w2 = round_bf16(g.standard_normal((F, E)) / np.sqrt(F))
    tx, t1, t2 = (torch.from_numpy(v).cuda().bfloat16() for v in (x, w1, w2))
    y = torch.empty((N, E), dtype=torch.float32, device="cuda")
    plan = ChainPlan(tx, t1, t2, y)
    assert not plan.fused
    plan.launch()
    torch.cuda.synchronize()
    _check(y.cpu().numpy(), reference_math.gemm_chain_fp64(x, w1, w2))


def test_many_rows_small_e_uses_two_gemms():
    """N >= 2048: the two-GEMM realisation is chosen (faster on B200) and matches fp64."""
    from paper_2604_14825_b200.gemm import FUSED_MAX_ROWS, ChainPlan

    N, K, F, E = FUSED_MAX_ROWS, 256, 384, 128
    g = np.random.default_rng(11)
    x = round_bf16(g.standard_normal((N, K)))
    w1 = round_bf16(g.standard_normal((K, F)) / np.sqrt(K))
    w2 = round_bf16(g.standard_normal((F, E)) / np.sqrt(F))
    tx, t1, t2 = (torch.from_numpy(v).cuda().bfloat16() for v in (x, w1, w2))
    y = torch.empty((N, E), dtype=torch.float32, device="cuda")
    plan = ChainPlan(tx, t1, t2, y)
    assert not plan.fused and plan.realisation == "gemm x2"
    plan.launch()
    torch.cuda.synchronize()
    _check(y.cpu().numpy(), reference_math.gemm_chain_fp64(x, w1, w2))


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 512), (2304, 2816, 320), (4100, 4104, 136)])
def test_cta_pair_gemm_vs_fp64(M, N, K):
    """Shapes with >= 74 tiles of 256x256 take the cta_group::2 kernel (incl. ragged M/N edges)."""
    from paper_2604_14825_b200.gemm import GemmPlan

    g = np.random.default_rng(M + N + K)
    a = round_bf16(g.standard_normal((M, K)))
    b = round_bf16(g.standard_normal((K, N)) / np.sqrt(K))
    ta = torch.from_numpy(a).cuda().bfloat16()
    tb = torch.from_numpy(b).cuda().bfloat16()
    c = torch.empty((M, N), dtype=torch.float32, device="cuda")
    GemmPlan(ta, tb, c).launch()
    torch.cuda.synchronize()
    ref = torch.from_numpy(a).double().cuda() @ torch.from_numpy(b).double().cuda()
    err = (c.double() - ref).abs()
    assert float(err.max()) <= 2e-2 and float(err.norm() / ref.norm()) <= 1e-2


@pytest.mark.parametrize("M,N,K,f32", [(4096, 128, 4096, False), (4096, 128, 4096, True), (1000, 64, 8192, True),
                                       (256, 128, 2048, False), (4100, 120, 1000, True)])
def test_split_k_gemm_vs_fp64(M, N, K, f32):
    """Few-tile shapes split K over CTAs (fp32 partials + reduce): the chain's T.W2 at E=128."""
    from paper_2604_14825_b200 import _lib
    from paper_2604_14825_b200.gemm import GemmPlan

    g = np.random.default_rng(M + 3 * N + K)
    a = round_bf16(g.standard_normal((M, K)))
    b = round_bf16(g.standard_normal((K, N)) / np.sqrt(K))
    ta = torch.from_numpy(a).cuda().bfloat16()
    tb = torch.from_numpy(b).cuda().bfloat16()
    c = torch.empty((M, N), dtype=torch.float32 if f32 else torch.bfloat16, device="cuda")
    plan = GemmPlan(ta, tb, c)
    expect = int(_lib.lib().nt_gemm_k_splits(M, N, K))
    assert plan.args.k_splits == expect
    if (M, N, K) == (4096, 128, 4096):
        assert expect > 1
    for _ in range(2):  # the workspace is reused across launches
        plan.launch()
    torch.cuda.synchronize()
    ref = a.astype(np.float64) @ b.astype(np.float64)
    _check(c.float().cpu().numpy(), ref, max_abs=3e-2 if not f32 else 2e-2)
