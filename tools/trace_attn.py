"""Dump the NT_TRACE pipeline timeline of one attention CTA (debug tool).

    NT_LIB_PATH=.../libnt_trace.so python tools/trace_attn.py [--cta 0] [--n 8192]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_14825_b200 import _lib  # noqa: E402
from paper_2604_14825_b200.runtime import AttentionPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cta", type=int, default=0)
ap.add_argument("--item", type=int, default=0, help="which of the CTA's work items to stamp")
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--causal", type=int, default=1)
ap.add_argument("--out", default="gpurun_out/trace.json")
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--b", type=int, default=1)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--scale", type=float, default=0.0883883)
ap.add_argument("--e4m3", action="store_true", help="e4m3 Q/K/V (the kind::f8f6f4 variant)")
a = ap.parse_args()
L = _lib.lib()
L.nt_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
buf = torch.zeros(4 * 64 * 8, dtype=torch.int64, device="cuda")
N, D = a.n, a.d
q = torch.randn(a.b, a.hq, N, D, device="cuda").bfloat16()
k = torch.randn(a.b, a.hkv, N, D, device="cuda").bfloat16()
v = torch.randn(a.b, a.hkv, N, D, device="cuda").bfloat16()
o = torch.empty(a.b, a.hq, N, D, device="cuda").bfloat16()
if a.e4m3:
    q, k, v = (t.float().to(torch.float8_e4m3fn) for t in (q, k, v))
plan = AttentionPlan(q, k, v, o, a.scale, "causal" if a.causal else "none")
for _ in range(3):
    plan.launch()
torch.cuda.synchronize()
L.nt_debug_set_trace(buf.data_ptr(), a.cta, a.item)
plan.launch()
torch.cuda.synchronize()
L.nt_debug_set_trace(None, a.cta, 0)
t = buf.view(4, 64, 8).cpu().numpy()
base = t[t > 0].min()
res = {}
for role, name in enumerate(["mma", "softmax0", "softmax1", "producer"]):
    rows = []
    for it in range(64):
        r = t[role, it]
        if (r > 0).any():
            rows.append([int(x - base) if x > 0 else None for x in r])
    res[name] = rows
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump(res, open(a.out, "w"))
print("kernel entry", int(t[3, 63, 7] - base) if t[3, 63, 7] > 0 else None)
# per item (role 3 rows 32+li / 48+li): last tile done, epilogue prepared, store_o entry,
# O complete, item start, item end; producer reach/publish, MMA has Q, softmax ask/get
for li in range(8):
    r32, r48 = t[3, 32 + li], t[3, 48 + li]
    f = lambda x: int(x - base) if x > 0 else None
    print(f"item {li}: start {f(r32[6])} last-tile {f(r32[0])} prepared {f(r32[1])} store_o {f(r32[2])} "
          f"O-complete {f(r48[6])} end {f(r32[7])} | ask {f(r48[4])} got {f(r48[5])} mma-Q {f(r48[3])}")
print("items (start, end) of tile 0:", [(int(t[3, 32 + i, 6] - base), int(t[3, 32 + i, 7] - base))
                                       for i in range(16) if t[3, 32 + i, 6] > 0])
print("per item [producer reaches, published, -, Q landed, softmax asks, softmax gets, O complete]:")
for i in range(15):
    r = t[3, 48 + i, :7]
    if (r > 0).any():
        print(i, [int(x - base) if x > 0 else None for x in r])
for name in ("mma", "softmax0", "softmax1", "producer"):
    print(name)
    for i, r in enumerate(res[name][:12]):
        print(i, r)
