"""Reference outputs at the BASELINE sizes, and on raw (non-bf16) fp32 inputs.

Run here (the dev container, where /root/reference exists):

    python tests/golden/gen_golden_full.py [case ...]

Companion of gen_golden.py (same pipeline, same seeds, same input recipe).
The inputs at these sizes are tens of MB, so they are NOT committed: the tests
regenerate them from the seed with the same recipe (`make_inputs` below,
numpy default_rng -- deterministic across machines) and check them against the
SHA-256 of their bytes recorded here.  What is committed is the REAL
reference `interpret_ma` fp32 output (tilecc/ma/interp.py:102), or a row
sample of it when the full output is large.

Cases
  causal8k_slice  one (b, h) slice of config 4 at N = M = 8192 (A.3 program,
                  seed-0 schedule, causal Mask): the full interpret_ma run
                  (~70 s); rows sampled (first/last 256, every 16th)
  decode4_32k     config 5's per-group program: N = 4 query rows (the 4 q-heads
                  of one kv group), M = 32768 keys; full output
  gemm4k_e128     config 2 parity shape 4096^3 x 128: the first BLOCKS row
                  blocks of the reference MA (kernel block extent shrunk to
                  BLOCKS -- blocks are independent, so those rows equal the full
                  run's); rows [0, 64*BLOCKS)
  gemm4k_e4096    config 2 at E = 4096 (max_tile_elems = 10^6), same
                  block prefix, every 8th row of it
  raw_*           config 1/3/4/5/2 parity programs fed raw N(0,1) fp32 inputs
                  (NOT rounded to bf16): the drop-in contract is fp32 numpy in,
                  exactly like interpret_ma; full output

Each case writes <case>.full.npz with
  interp_fp32   the reference output rows (float32)
  rows          the row indices they are (int64)
and a manifest entry (full_manifest.json) with the program, binding, seed,
schedule seed, block prefix, input recipe and per-input SHA-256.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from tilecc.autosched.scheduler import SchedulerOptions, run_autoscheduler  # noqa: E402
from tilecc.ma.device import DEFAULT_DEVICE  # noqa: E402
from tilecc.ma.interp import interpret_ma  # noqa: E402
from tilecc.pipeline import frontend, lower_seed  # noqa: E402

from oracle.ma_interp import causal_mask, round_bf16  # noqa: E402
from paper_2604_14825_b200 import ma_ir  # noqa: E402
from paper_2604_14825_b200.programs import PROGRAMS  # noqa: E402

MANIFEST = os.path.join(HERE, "full_manifest.json")


def make_inputs(input_names, shapes, seed, scales, mask, raw):
    """gen_golden.make_inputs, optionally without the bf16 rounding (raw fp32).

    tests/conftest.py:65-67 recipe: default_rng(seed).standard_normal per input
    in input order (the Mask consumes its draw too), times the input's scale."""
    rng = np.random.default_rng(seed)
    out = {}
    for name in input_names:
        shape = tuple(shapes[name])
        if name == "Mask":
            out[name] = causal_mask(*shape) if mask == "causal" else np.zeros(shape, np.float32)
            rng.standard_normal(shape)
            continue
        x = rng.standard_normal(shape) * scales.get(name, 1.0)
        out[name] = x.astype(np.float32) if raw else round_bf16(x)
    return out


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_rows(n):
    if n <= 1024:
        return np.arange(n)
    rows = set(range(256)) | set(range(n - 256, n)) | set(range(0, n, 16))
    return np.array(sorted(rows))


S4K = 1 / 64.0  # 1/sqrt(4096): keeps T and Y ~ N(0, 1)
CASES = {
    "causal8k_slice": dict(prog="llama_causal", bind=dict(N=8192, M=8192, D=128), mask="causal"),
    "decode4_32k": dict(prog="llama", bind=dict(N=4, M=32768, D=128)),
    "gemm4k_e128": dict(prog="gemm2", bind=dict(N=4096, K=4096, F=4096, E=128), blocks=8,
                        scales={"W1": S4K, "W2": S4K}),
    "gemm4k_e4096": dict(prog="gemm2", bind=dict(N=4096, K=4096, F=4096, E=4096), blocks=8,
                         scales={"W1": S4K, "W2": S4K}, device=dict(max_tile_elems=1000000)),
    "raw_attn256": dict(prog="attention", bind=dict(N=256, M=256, D=64), raw=True),
    "raw_bert512": dict(prog="scaled_0p125", bind=dict(N=512, M=512, D=64), raw=True),
    "raw_causal512": dict(prog="llama_causal", bind=dict(N=512, M=512, D=128), mask="causal", raw=True),
    "raw_decode4": dict(prog="llama", bind=dict(N=4, M=2048, D=128), raw=True),
    "raw_gemm_v6": dict(prog="gemm2", bind=dict(N=256, K=256, F=512, E=128), raw=True,
                        scales={"W1": 1 / 16.0, "W2": 1 / math.sqrt(512)}),
}


def run_case(name, case):
    src = PROGRAMS[case["prog"]]
    device = DEFAULT_DEVICE
    if case.get("device"):
        device = replace(DEFAULT_DEVICE, **case["device"])
    bound, base = frontend(src, case["bind"])
    seeds = run_autoscheduler(base, device, SchedulerOptions())
    lw = lower_seed(base, seeds[0].schedule, device, None)
    ma = lw.ma
    nblk = case.get("blocks")
    if nblk is not None:
        k0 = ma.kernels[0]
        assert len(ma.kernels) == 1 and len(k0.blocks) == 1, "block prefix needs a 1-D grid"
        var, axis, ext = k0.blocks[0]
        assert nblk <= ext
        ma = replace(ma, kernels=(replace(k0, blocks=((var, axis, nblk),)),))
    names = bound.input_names()
    shapes = {n: tuple(bound.shapes[n]) for n in names}
    inputs = make_inputs(names, shapes, 0, case.get("scales", {}), case.get("mask"), case.get("raw", False))
    t0 = time.time()
    outs, _ = interpret_ma(ma, inputs, device, "fp32")
    dt = time.time() - t0
    out = np.asarray(outs[ma.output], dtype=np.float32)
    if nblk is not None:
        # rows covered by the prefix: the block variable's output slice is t*var
        rows_per = out.shape[0] // ext
        rows = np.arange(nblk * rows_per)
        if out.shape[1] > 1024:  # E = 4096: every 8th row of the prefix keeps the fixture ~1 MB
            rows = rows[::8]
    else:
        rows = sample_rows(out.shape[0])
    np.savez_compressed(os.path.join(HERE, f"{name}.full.npz"), interp_fp32=out[rows], rows=rows)
    # the MA (full grid) the test executes on the device
    full_mod = ma_ir.from_tilecc(lw.ma)
    with open(os.path.join(HERE, f"{name}.full_ma.json"), "w") as f:
        f.write(ma_ir.to_json(full_mod) + "\n")
    entry = {"program": case["prog"], "binding": case["bind"], "seed": 0, "schedule_seed": 0,
             "scales": case.get("scales", {}), "mask": case.get("mask"), "raw": case.get("raw", False),
             "device": case.get("device"), "block_prefix": nblk, "input_order": list(names),
             "shapes": {n: list(s) for n, s in shapes.items()},
             "sha256": {n: sha(v) for n, v in inputs.items() if n != "Mask"},
             "interp_seconds": round(dt, 2), "output": ma.output}
    print(f"{name}: interpret_ma {dt:.1f} s, rows {len(rows)}", flush=True)
    return entry


def main():
    want = sys.argv[1:] or list(CASES)
    man = {}
    if os.path.exists(MANIFEST):
        with open(MANIFEST) as f:
            man = json.load(f)
    for name in want:
        man[name] = run_case(name, CASES[name])
        with open(MANIFEST, "w") as f:
            f.write(json.dumps(man, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
