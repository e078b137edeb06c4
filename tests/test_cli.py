"""Device CLI gates (paper_2604_14825_b200/cli.py) mirroring tilecc/cli.py selftest / check / tune."""

import json

import pytest

from paper_2604_14825_b200 import cli
from paper_2604_14825_b200.programs import PROGRAMS

SOFTMAX = """
tensor X[fp32](N, M)
m(i) = max(j, X(i, j))
E(i, j) = exp(X(i, j) - m(i))
s(i) = sum(j, E(i, j))
Y(i, j) = E(i, j) / s(i)
output Y
"""
MATMUL = """
tensor A[fp32](N, K)
tensor B[fp32](K, M)
T(i, j) = sum(k, A(i, k) * B(k, j))
output T
"""


def test_argparser_mirrors_reference_subcommands():
    ap = cli.build_argparser()
    a = ap.parse_args(["check", "p.te", "--bind", "N=8,M=8", "--trials", "2"])
    assert a.command == "check" and a.trials == 2 and cli._parse_bind(a.bind) == {"N": 8, "M": 8}
    assert ap.parse_args(["selftest"]).command == "selftest"
    assert ap.parse_args(["tune", "p.te", "--gpus", "8"]).gpus == 8


@pytest.mark.gpu
def test_selftest_passes_on_device(capsys):
    assert cli.main(["selftest"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert [ln.split()[1] for ln in out] == ["copy", "matmul-bias", "softmax"]
    assert all(ln.split()[2] == "ok" for ln in out)


@pytest.mark.gpu
@pytest.mark.parametrize("src,exact", [(MATMUL, "True"), (SOFTMAX, "n/a")])
def test_check_gate_on_device(tmp_path, capsys, src, exact):
    p = tmp_path / "prog.te"
    p.write_text(src)
    assert cli.main(["check", str(p), "--bind", "N=32,M=24,K=16", "--trials", "2"]) == 0
    rows = capsys.readouterr().out.splitlines()[1:]
    assert rows and all(r.split()[1] == exact and r.split()[-1] == "ok" for r in rows)


@pytest.mark.gpu
def test_run_attention_on_tensor_cores(tmp_path, capsys):
    p = tmp_path / "attn.te"
    p.write_text(PROGRAMS["attention"])
    assert cli.main(["run", str(p), "--bind", "N=256,M=256,D=64", "--backend", "auto"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert rec["shape"] == [256, 64] and "attn_fwd" in rec["realisation"][0]


@pytest.mark.gpu
def test_tune_simt_program_on_device(tmp_path, capsys):
    p = tmp_path / "mm.te"
    p.write_text(MATMUL)
    out = tmp_path / "out"
    assert cli.main(["tune", str(p), "--bind", "N=128,M=128,K=64", "--tune-budget", "12",
                     "--out", str(out)]) == 0
    lines = (out / "tuning.jsonl").read_text().strip().splitlines()
    assert len(lines) == 12
    costs = [json.loads(ln)["cost"] for ln in lines]
    assert any(isinstance(c, (int, float)) and c < 1e9 for c in costs)  # device-timed, finite
