"""Time DecodePlan launches (CUDA events, L2 flushed) -- A/B of decode library variants via NT_LIB_PATH.

    python tools/decode_time.py [--e4m3] [--b 64] [--hkv 8] [--g 4] [--m 32768] [--splits 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_14825_b200.runtime import DecodePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--e4m3", action="store_true")
ap.add_argument("--b", type=int, default=64)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--g", type=int, default=4)
ap.add_argument("--m", type=int, default=32768)
ap.add_argument("--splits", type=int, default=0)
a = ap.parse_args()
dt = torch.float8_e4m3fn if a.e4m3 else torch.bfloat16
q = torch.randn(a.b, a.hkv, a.g, 128, device="cuda").to(dt)
k = torch.randn(a.b, a.hkv, a.m, 128, device="cuda").to(dt)
v = torch.randn(a.b, a.hkv, a.m, 128, device="cuda").to(dt)
o = torch.empty(a.b, a.hkv, a.g, 128, device="cuda", dtype=torch.bfloat16)
plan = DecodePlan(q, k, v, o, 0.088, num_splits=a.splits)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    plan.launch()
ts = []
for _ in range(10):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.launch()
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
kv = 2 * a.b * a.hkv * a.m * 128 * (1 if a.e4m3 else 2)
print(f"{'e4m3' if a.e4m3 else 'bf16'} B={a.b} Hkv={a.hkv} g={a.g} M={a.m} splits={plan.splits}: "
      f"{ms * 1e3:.1f} us, {kv / (ms * 1e-3) / 1e9:.0f} GB/s")
