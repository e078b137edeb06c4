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


@pytest.mark.parametrize("case", ["decode4", "decode1"])
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
