"""Generic MA -> CUDA SIMT lowering (paper_2604_14825_b200/simt.py).

Corpus: tests/golden/simt_corpus.{json,npz}, generated from the reference's own
program corpus and selftest programs by tests/golden/gen_simt_corpus.py (the
real tilecc pipeline and interpret_ma).

CPU tests: the numpy oracle equals the reference interpret_ma bit for bit on
every corpus case (fp32 and fp64), every case lowers in both precisions, the
block-level analyses are as expected, and a sample compiles with nvcc for
sm_100a.  GPU tests: every case runs through execute_ma on the device and
matches the reference -- bit for bit where the program has no exp / exp2 /
log2 (the lowering keeps interpret_ma's operation order and rounding), within
the stated tolerances where CUDA's transcendental functions differ from
numpy's in the last ulps.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ma_interp
from paper_2604_14825_b200 import ma_ir, simt

# tolerances for programs with exp / exp2 / log2 (CUDA <= 2 ulp vs numpy):
FP32_RTOL, FP32_ATOL = 2e-5, 1e-6
FP64_RTOL, FP64_ATOL = 1e-12, 1e-14
SELFTEST_TOL = 1e-9  # tilecc selftest gate (tilecc/cli.py:293): fp64 vs oracle_eval


def _load():
    with open(os.path.join(GOLDEN, "simt_corpus.json")) as f:
        cases = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "simt_corpus.npz"))
    return cases, arrays


CASES, ARR = _load()
IDS = [f"{c['case']}-{c['name']}-s{c['seed']}" for c in CASES]


def _module(case):
    return ma_ir.from_json(json.dumps(case["ma"]))


def _inputs(case):
    """The generator's inputs (tests/golden/gen_simt_corpus.py make_inputs), in input order."""
    rng = np.random.default_rng(case["program"] + 1)
    return {n: rng.standard_normal(tuple(case["shapes"][n])) for n in case["inputs"]}


def _transcendental(mod) -> bool:
    for k in mod.kernels:
        for st in simt._statements(k.body):
            if isinstance(st, ma_ir.Compute):
                for n in st.expr.walk():
                    if isinstance(n, ma_ir.Un) and n.op in ("exp", "exp2", "log2"):
                        return True
    return False


def test_corpus_covers_every_family():
    names = {c["name"] for c in CASES}
    srcs = "\n".join(c["src"] for c in CASES)
    assert {"selftest_copy", "selftest_matmul-bias", "selftest_softmax", "attention64"} <= names
    for token in ("sum(k", "max(j", "exp(", "T(r: R"):
        assert token in srcs, token
    assert len(CASES) >= 100


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_matches_reference_on_corpus(case):
    """The numpy restatement is pinned on the corpus too (fp32 and fp64, bit for bit)."""
    mod = _module(case)
    ins = _inputs(case)
    o32, _ = ma_interp.interpret_ma(mod, ins, "fp32", account=False)
    o64, _ = ma_interp.interpret_ma(mod, ins, "fp64", account=False)
    np.testing.assert_array_equal(o32[case["output"]], ARR[f"{case['case']}_ref32"])
    np.testing.assert_array_equal(o64[case["output"]], ARR[f"{case['case']}_ref64"])


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_lowering_builds(case):
    mod = _module(case)
    for prec in ("fp32", "fp64"):
        prog = simt.lower(mod, prec)
        assert len(prog.launches) == len(mod.kernels)
        assert prog.source.count("__global__") == len(mod.kernels)
        for ln in prog.launches:
            assert ln.grid >= 1 and (ln.grid == 1 or not ln.sequential)


def test_rational_precision_is_unsupported():
    from paper_2604_14825_b200.errors import UnsupportedMA

    with pytest.raises(UnsupportedMA):
        simt.lower(_module(CASES[0]), "rational")


def test_block_analyses():
    # matmul64: independent output tiles -> parallel grid over every block point
    mm = [c for c in CASES if c["name"] == "matmul64"][0]
    prog = simt.lower(_module(mm))
    assert not prog.carried and not any(ln.sequential for ln in prog.launches)
    assert prog.launches[0].grid == prog.launches[0].points == 4


def test_global_conflict_forces_sequential_blocks():
    """Two block points accumulating into the same Global row must run in order."""
    A = ma_ir.Affine.make
    sl = lambda off, n: ma_ir.Slice(off, n)  # noqa: E731
    # Y[0:4] = Y[0:4] + X[4*b : 4*b+4]  over blocks b in [0, 3)
    y_ref = ma_ir.Ref((4,), "Y", (sl(A({}), 4),))
    x_ref = ma_ir.Ref((4,), "X", (sl(A({"b": 4}), 4),))
    body = (ma_ir.Compute("Y", (sl(A({}), 4),), ma_ir.Bin((4,), "add", y_ref, x_ref)),)
    k = ma_ir.Kernel("k0", (("b", "blockIdx.x", 3),), body)
    mod = ma_ir.Module((ma_ir.Buffer("X", (12,), is_input=True), ma_ir.Buffer("Y", (4,), is_output=True)),
                       (k,), "Y")
    prog = simt.lower(mod)
    assert prog.launches[0].sequential and prog.launches[0].grid == 1


def test_carried_private_buffer_forces_reference_order():
    """A Register buffer read before it is written in a block keeps the CPU executor's order."""
    A = ma_ir.Affine.make
    sl = lambda off, n: ma_ir.Slice(off, n)  # noqa: E731
    acc = ma_ir.Ref((4,), "acc", (sl(A({}), 4),))
    x_ref = ma_ir.Ref((4,), "X", (sl(A({"b": 4}), 4),))
    body = (ma_ir.Compute("acc", (sl(A({}), 4),), ma_ir.Bin((4,), "add", acc, x_ref)),
            ma_ir.Compute("Y", (sl(A({"b": 4}), 4),), acc))
    k = ma_ir.Kernel("k0", (("b", "blockIdx.x", 3),), body)
    mod = ma_ir.Module((ma_ir.Buffer("X", (12,), is_input=True), ma_ir.Buffer("Y", (12,), is_output=True),
                        ma_ir.Buffer("acc", (4,), scope="Register")), (k,), "Y")
    prog = simt.lower(mod)
    assert prog.carried and prog.launches[0].grid == 1


SAMPLE = [c for c in CASES if c["seed"] == 0][::6]


@pytest.mark.parametrize("case", SAMPLE, ids=[f"{c['case']}-{c['name']}" for c in SAMPLE])
def test_nvcc_compiles_for_sm100a(case):
    prog = simt.lower(_module(case), "fp32")
    path = simt.compile_cubin(prog)
    assert os.path.getsize(path) > 0


# ---------------------------------------------------------------- GPU parity


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_simt_fp32_matches_reference_interp(case):
    from paper_2604_14825_b200 import execute_ma

    mod = _module(case)
    bufs, rep = execute_ma(mod, _inputs(case), None, "fp32", backend="simt")
    got = np.asarray(bufs[case["output"]])
    ref = ARR[f"{case['case']}_ref32"]
    assert got.dtype == np.float32 and got.shape == ref.shape
    assert rep.launches == len(mod.kernels) and rep.realisation[0]["kernel"] == "simt"
    if _transcendental(mod):
        np.testing.assert_allclose(got, ref, rtol=FP32_RTOL, atol=FP32_ATOL)
    else:
        np.testing.assert_array_equal(got, ref)  # same operation order and rounding


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_simt_fp64_matches_reference_interp_and_oracle(case):
    from paper_2604_14825_b200 import execute_ma

    mod = _module(case)
    bufs, _ = execute_ma(mod, _inputs(case), None, "fp64")  # auto: fp64 -> SIMT
    got = np.asarray(bufs[case["output"]])
    ref = ARR[f"{case['case']}_ref64"]
    assert got.dtype == np.float64
    if _transcendental(mod):
        np.testing.assert_allclose(got, ref, rtol=FP64_RTOL, atol=FP64_ATOL)
    else:
        np.testing.assert_array_equal(got, ref)
    assert float(np.max(np.abs(got - ARR[f"p{case['program']}_oracle"]))) < SELFTEST_TOL


@pytest.mark.gpu
def test_auto_backend_routes_unrecognised_programs_to_simt():
    from paper_2604_14825_b200 import execute_ma

    case = [c for c in CASES if c["name"] == "selftest_softmax"][0]
    bufs, rep = execute_ma(_module(case), _inputs(case))
    assert rep.realisation[0]["kernel"] == "simt"
    np.testing.assert_allclose(bufs[case["output"]], ARR[f"{case['case']}_ref32"], rtol=FP32_RTOL,
                               atol=FP32_ATOL)


@pytest.mark.gpu
def test_simt_division_by_zero_raises():
    from paper_2604_14825_b200 import execute_ma
    from paper_2604_14825_b200.errors import DivisionByZero

    # Y = X / Z: numpy's tile divide raises on any zero denominator (tilecc/numerics.py:123-126)
    A = ma_ir.Affine.make
    sl = lambda off, n: ma_ir.Slice(off, n)  # noqa: E731
    body = (ma_ir.Compute("Y", (sl(A({}), 4),), ma_ir.Bin((4,), "div", ma_ir.Ref((4,), "X", (sl(A({}), 4),)),
                                                         ma_ir.Ref((4,), "Z", (sl(A({}), 4),)))),)
    m = ma_ir.Module((ma_ir.Buffer("X", (4,), is_input=True), ma_ir.Buffer("Z", (4,), is_input=True),
                      ma_ir.Buffer("Y", (4,), is_output=True)), (ma_ir.Kernel("k0", (), body),), "Y")
    x = np.ones(4)
    with pytest.raises(DivisionByZero):
        execute_ma(m, {"X": x, "Z": np.array([1.0, 2.0, 0.0, 4.0])}, backend="simt")
    bufs, _ = execute_ma(m, {"X": x, "Z": np.array([1.0, 2.0, 4.0, 8.0])}, backend="simt")
    np.testing.assert_array_equal(bufs["Y"], np.float32([1, 0.5, 0.25, 0.125]))


@pytest.mark.gpu
@pytest.mark.parametrize("case", __import__("conftest").io_cases())
def test_simt_runs_the_baseline_families_exactly(case):
    """The attention / decode / GEMM-chain goldens through the SIMT lowering in fp32:
    interpret_ma's own arithmetic on the device (the tcgen05 kernels compute in bf16)."""
    from conftest import load_golden
    from paper_2604_14825_b200 import execute_ma

    mod, inputs, interp32, oracle64 = load_golden(case)
    bufs, rep = execute_ma(mod, inputs, None, "fp32", backend="simt")
    got = np.asarray(bufs[mod.output])
    np.testing.assert_allclose(got, interp32, rtol=FP32_RTOL, atol=FP32_ATOL)
    assert float(np.max(np.abs(got - oracle64))) < 1e-4


def test_unrealisable_family_members_are_reported():
    """An attention MA with head dim 32 is recognised but has no tcgen05 kernel (auto -> SIMT)."""
    from paper_2604_14825_b200.executor import tcgen05_unsupported
    from paper_2604_14825_b200.recognize import recognize

    case = [c for c in CASES if c["name"] == "attention64"][0]
    specs = recognize(_module(case))
    assert "head dim 32" in tcgen05_unsupported(specs[0])


@pytest.mark.gpu
def test_auto_backend_falls_back_to_simt_for_unsupported_head_dim():
    from paper_2604_14825_b200 import execute_ma

    case = [c for c in CASES if c["name"] == "attention64"][0]
    bufs, rep = execute_ma(_module(case), _inputs(case))
    assert rep.realisation[0]["kernel"] == "simt"
    np.testing.assert_allclose(bufs[case["output"]], ARR[f"{case['case']}_ref32"], rtol=FP32_RTOL, atol=FP32_ATOL)
