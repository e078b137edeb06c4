"""K2b per-tile timeline of one CTA (NT_TRACE build; add -DNT_DTC_COMPUTEONLY for the consumers alone).

    NT_LIB_PATH=.../lib_trace.so python tools/trace_decode.py [--e4m3] [--cta 0]
Prints, per tile, clock64 deltas: MMA S issued / P seen / PV issued; softmax S seen /
S loaded / exps done / PV(t-1) seen / P stored; producer K / V issued.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_14825_b200 import _lib  # noqa: E402
from paper_2604_14825_b200.runtime import DecodePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--e4m3", action="store_true")
ap.add_argument("--cta", type=int, default=0)
ap.add_argument("--m", type=int, default=32768)
a = ap.parse_args()
L = _lib.lib()
L.nt_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
dt = torch.float8_e4m3fn if a.e4m3 else torch.bfloat16
B, Hkv, g = 64, 8, 4
q = torch.randn(B, Hkv, g, 128, device="cuda").to(dt)
k = torch.randn(B, Hkv, a.m, 128, device="cuda").to(dt)
v = torch.randn(B, Hkv, a.m, 128, device="cuda").to(dt)
o = torch.empty(B, Hkv, g, 128, device="cuda", dtype=torch.bfloat16)
plan = DecodePlan(q, k, v, o, 0.088)
for _ in range(3):
    plan.launch()
torch.cuda.synchronize()
buf = torch.zeros(4 * 64 * 8, dtype=torch.int64, device="cuda")
L.nt_debug_set_trace(buf.data_ptr(), a.cta, 0)
plan.launch()
torch.cuda.synchronize()
L.nt_debug_set_trace(None, a.cta, 0)
t = buf.view(4, 64, 8).cpu().numpy()
base = t[t > 0].min()
print("tile | MMA: S_iss P_seen PV_iss Sfull Ssf Smma PVfull PVmma | SMX: S_seen S_ld exps PVw P_st | PROD: K V")
for i in range(0, 64):
    m, sm, pr = t[0, i], t[1, i], t[3, i]
    if not (m > 0).any():
        continue
    f = lambda r, n: " ".join(f"{int(x - base):7d}" if x > 0 else "      -" for x in r[:n])  # noqa: E731
    print(f"{i:4d} | {f(m, 8)} | {f(sm, 5)} | {f(pr, 2)}")
per = [int(t[1, i + 1, 4] - t[1, i, 4]) for i in range(8, 40) if t[1, i, 4] > 0 and t[1, i + 1, 4] > 0]
if per:
    print("softmax P-store period (tiles 8-40): median", sorted(per)[len(per) // 2], "clk")
