"""Generate the committed golden fixtures by running the REAL reference.

Run here (the dev container, where /root/reference exists):

    python tests/golden/gen_golden.py

For every case it runs the reference pipeline
  parse_program -> bind_dims -> elaborate -> classify_loops
  (tilecc/pipeline.py:37-43) -> run_autoscheduler (tilecc/autosched/scheduler.py:73)
  -> lower_seed (tilecc/pipeline.py:46-55)
and writes
  <case>.seed<k>.ma.json   MA module (paper_2604_14825_b200.ma_ir JSON)
  <case>.seed<k>.ma.txt    emit_tile_text(ma, "generic") (tilecc/ma/emit.py:32)
  <case>.seed<k>.schedule.jsonl  serialize_schedule (tilecc/schedule/steps.py:87)
  <case>.seed<k>.cost.json cost_model(ma).to_json() (tilecc/ma/cost.py:66)
and, for cases with `io`, the bf16-representable inputs (as bf16 bits), the
reference interpret_ma fp32 output (tilecc/ma/interp.py:102) and the fp64
oracle_eval output (tilecc/frontend/oracle.py:25) plus the dynamic CostReport.

Inputs follow tests/conftest.py:65-67 (`gaussian_inputs`: default_rng(seed)
standard_normal per input in input order), optionally scaled, then rounded
to bf16 so the GPU sees identical values (BASELINE.md parity protocol).
"""

from __future__ import annotations

import json
import math
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from tilecc.autosched.scheduler import SchedulerOptions, run_autoscheduler  # noqa: E402
from tilecc.frontend.oracle import oracle_eval  # noqa: E402
from tilecc.ma.device import DEFAULT_DEVICE  # noqa: E402
from tilecc.ma.emit import emit_tile_text  # noqa: E402
from tilecc.ma.interp import interpret_ma  # noqa: E402
from tilecc.pipeline import frontend, lower_seed  # noqa: E402
from tilecc.schedule.steps import serialize_schedule  # noqa: E402

from oracle.ma_interp import bf16_bits, causal_mask, round_bf16  # noqa: E402
from paper_2604_14825_b200 import ma_ir  # noqa: E402
from paper_2604_14825_b200.programs import PROGRAMS  # noqa: E402


def write(path, text):
    with open(path, "w") as f:
        f.write(text)


def make_inputs(bound, seed, scales, mask):
    rng = np.random.default_rng(seed)
    out = {}
    for name in bound.input_names():
        shape = bound.shapes[name]
        if name == "Mask":
            out[name] = causal_mask(*shape) if mask == "causal" else np.zeros(shape, np.float32)
            rng.standard_normal(shape)  # keep the stream aligned with conftest
            continue
        x = rng.standard_normal(shape) * scales.get(name, 1.0)
        out[name] = round_bf16(x)
    return out


CASES = [
    # name, program, binding, seeds exported, io, extra
    dict(name="attn256", prog="attention", bind=dict(N=256, M=256, D=64), seeds="all", io=True),
    dict(name="bert512", prog="scaled_0p125", bind=dict(N=512, M=512, D=64), seeds=[0, 1], io=True),
    dict(name="causal512", prog="llama_causal", bind=dict(N=512, M=512, D=128), seeds=[0, 1], io=True,
         mask="causal"),
    dict(name="llama2k", prog="llama", bind=dict(N=2048, M=2048, D=128), seeds=[0], io=False),
    dict(name="causal2k", prog="llama_causal", bind=dict(N=2048, M=2048, D=128), seeds=[0], io=False),
    dict(name="causal4k", prog="llama_causal", bind=dict(N=4096, M=4096, D=128), seeds=[0], io=False),
    dict(name="causal8k", prog="llama_causal", bind=dict(N=8192, M=8192, D=128), seeds=[0], io=False),
    dict(name="causal16k", prog="llama_causal", bind=dict(N=16384, M=16384, D=128), seeds=[0], io=False),
    dict(name="decode4", prog="llama", bind=dict(N=4, M=2048, D=128), seeds=[0], io=True),
    dict(name="decode1", prog="llama", bind=dict(N=1, M=1024, D=128), seeds=[0], io=True),
    dict(name="decode4_32k", prog="llama", bind=dict(N=4, M=32768, D=128), seeds=[0], io=False),
    dict(name="decode4_64k", prog="llama", bind=dict(N=4, M=65536, D=128), seeds=[0], io=False),
    dict(name="decode4_128k", prog="llama", bind=dict(N=4, M=131072, D=128), seeds=[0], io=False),
    dict(name="gemm_v6", prog="gemm2", bind=dict(N=256, K=256, F=512, E=128), seeds=[0], io=True,
         scales={"W1": 1 / 16.0, "W2": 1 / math.sqrt(512)}),
    dict(name="gemm_v5", prog="gemm2", bind=dict(N=128, K=1024, F=256, E=128), seeds=[0], io=True,
         scales={"W1": 1 / 32.0, "W2": 1 / math.sqrt(512)}),
    dict(name="gemm4k_e128", prog="gemm2", bind=dict(N=4096, K=4096, F=4096, E=128), seeds=[0], io=False),
    dict(name="gemm4k_e4096", prog="gemm2", bind=dict(N=4096, K=4096, F=4096, E=4096), seeds=[0],
         io=False, device=dict(max_tile_elems=1000000)),
    # tile-assignment variants of the config-1 kernel (same structure, other tiles)
    dict(name="attn256_t128x128", prog="attention", bind=dict(N=256, M=256, D=64), seeds=[0], io=True,
         assign=dict(t0_i=128, t0_j=128)),
    dict(name="attn256_t32x64", prog="attention", bind=dict(N=256, M=256, D=64), seeds=[0], io=True,
         assign=dict(t0_i=32, t0_j=64)),
    dict(name="causal512_t128x64", prog="llama_causal", bind=dict(N=512, M=512, D=128), seeds=[0],
         io=True, mask="causal", assign=dict(t0_i=128, t0_j=64)),
    # the same programs scheduled for the B200 profile (paper_2604_14825_b200/b200.device,
    # SchedulerOptions(backends=("sm100a",))): config 2 at E=4096 schedules without overrides
    dict(name="b200_attn256", prog="attention", bind=dict(N=256, M=256, D=64), seeds="all", io=True,
         profile="b200"),
    dict(name="b200_bert512", prog="scaled_0p125", bind=dict(N=512, M=512, D=64), seeds=[0], io=True,
         profile="b200"),
    dict(name="b200_causal512", prog="llama_causal", bind=dict(N=512, M=512, D=128), seeds=[0], io=True,
         mask="causal", profile="b200"),
    dict(name="b200_decode4", prog="llama", bind=dict(N=4, M=2048, D=128), seeds=[0], io=True, profile="b200"),
    dict(name="b200_gemm_v6", prog="gemm2", bind=dict(N=256, K=256, F=512, E=128), seeds=[0], io=True,
         scales={"W1": 1 / 16.0, "W2": 1 / math.sqrt(512)}, profile="b200"),
    dict(name="b200_gemm_e512", prog="gemm2", bind=dict(N=256, K=256, F=256, E=512), seeds=[0], io=True,
         scales={"W1": 1 / 16.0, "W2": 1 / 16.0}, profile="b200"),
    dict(name="b200_gemm4k_e4096", prog="gemm2", bind=dict(N=4096, K=4096, F=4096, E=4096), seeds=[0],
         io=False, profile="b200"),
    dict(name="b200_causal8k", prog="llama_causal", bind=dict(N=8192, M=8192, D=128), seeds=[0], io=False,
         profile="b200"),
    # natural spellings (mask / scale after the sum) scheduled with the upstream fix
    # (paper_2604_14825_b200/upstream.py; the unfixed scheduler raises IterationMismatch)
    dict(name="fix_causal_natural256", prog="causal_natural", bind=dict(N=256, M=256, D=64), seeds=[0], io=True,
         mask="causal", fixes=True),
    dict(name="fix_scaled_post512", prog="scaled_post_0p125", bind=dict(N=512, M=512, D=64), seeds=[0], io=True,
         fixes=True),
    dict(name="fix_llama_causal_natural512", prog="llama_causal_natural", bind=dict(N=512, M=512, D=128), seeds=[0],
         io=True, mask="causal", fixes=True),
]


def b200_context():
    from tilecc.ma.device import load_device
    return (load_device(os.path.join(REPO, "paper_2604_14825_b200", "b200.device")),
            SchedulerOptions(backends=("sm100a",)))


def main():
    # `gen_golden.py NAME ...` regenerates only those cases (merged into the manifest)
    only = set(sys.argv[1:])
    mpath = os.path.join(HERE, "manifest.json")
    manifest = json.load(open(mpath)) if only and os.path.exists(mpath) else {}
    for case in CASES:
        if only and case["name"] not in only:
            continue
        name = case["name"]
        src = PROGRAMS[case["prog"]]
        device, opts = DEFAULT_DEVICE, SchedulerOptions()
        if case.get("profile") == "b200":
            device, opts = b200_context()
        if case.get("device"):
            device = replace(device, **case["device"])
        bound, base = frontend(src, case["bind"])
        if case.get("fixes"):
            from paper_2604_14825_b200 import upstream
            upstream.apply()
        try:
            seeds = run_autoscheduler(base, device, opts)
        finally:
            if case.get("fixes"):
                upstream.restore()
        which = range(len(seeds)) if case["seeds"] == "all" else case["seeds"]
        entry = {"program": case["prog"], "binding": case["bind"], "n_seeds": len(seeds),
                 "seeds": list(which), "assignment": case.get("assign"),
                 "device": case.get("device"), "io": case["io"], "mask": case.get("mask")}
        if case.get("profile"):
            entry["profile"] = case["profile"]
        if case.get("fixes"):
            entry["upstream_fixes"] = True
        for k in which:
            sd = seeds[k]
            assignment = None
            if case.get("assign"):
                assignment = {t.name: t.default for t in sd.schedule.tunables}
                assignment.update(case["assign"])
            lw = lower_seed(base, sd.schedule, device, assignment)
            stem = os.path.join(HERE, f"{name}.seed{k}")
            mod = ma_ir.from_tilecc(lw.ma)
            write(stem + ".ma.json", ma_ir.to_json(mod) + "\n")
            write(stem + ".ma.txt", emit_tile_text(lw.ma))
            write(stem + ".schedule.jsonl", serialize_schedule(sd.schedule))
            write(stem + ".cost.json", lw.static_cost.to_json())
            if case["io"] and k == list(which)[0]:
                inputs = make_inputs(bound, 0, case.get("scales", {}), case.get("mask"))
                outs, rep = interpret_ma(lw.ma, inputs, device, "fp32")
                ref64 = oracle_eval(bound, inputs, "fp64")
                arrays = {}
                for n, v in inputs.items():
                    if n == "Mask":
                        continue
                    arrays["in_" + n] = bf16_bits(v)
                arrays["interp_fp32"] = np.asarray(outs[lw.ma.output], dtype=np.float32)
                arrays["oracle_fp64"] = np.asarray(ref64[lw.ma.output], dtype=np.float64)
                np.savez_compressed(stem + ".io.npz", **arrays)
                write(stem + ".interp_cost.json", rep.to_json())
        manifest[name] = entry
        print(name, "seeds", len(seeds), "exported", list(which))
    write(os.path.join(HERE, "manifest.json"), json.dumps(manifest, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
