import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def golden_stem(case, seed=None):
    man = golden_manifest()[case]
    seed = man["seeds"][0] if seed is None else seed
    return os.path.join(GOLDEN, f"{case}.seed{seed}")


def load_golden(case, seed=None):
    """(Module, inputs dict fp32 (bf16-representable), interp_fp32, oracle_fp64)."""
    from oracle.ma_interp import causal_mask, from_bf16_bits
    from paper_2604_14825_b200 import ma_ir

    stem = golden_stem(case, seed)
    with open(stem + ".ma.json") as f:
        mod = ma_ir.from_json(f.read())
    io = np.load(stem + ".io.npz")
    inputs = {}
    for b in mod.inputs():
        if b.name == "Mask":
            inputs["Mask"] = causal_mask(*b.shape)
        else:
            inputs[b.name] = from_bf16_bits(io["in_" + b.name]).reshape(b.shape)
    return mod, inputs, io["interp_fp32"], io["oracle_fp64"]


def io_cases():
    return [k for k, v in golden_manifest().items() if v["io"]]


def all_ma_files():
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".ma.json"))
