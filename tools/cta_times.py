"""Per-CTA entry/exit times of one K1 launch (NT_TRACE build): load balance and start-up cost."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_14825_b200 import _lib
from paper_2604_14825_b200.runtime import AttentionPlan
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048); ap.add_argument("--causal", type=int, default=1)
ap.add_argument("--d", type=int, default=128); ap.add_argument("--b", type=int, default=1)
ap.add_argument("--hq", type=int, default=32); ap.add_argument("--hkv", type=int, default=8)
a = ap.parse_args()
L = _lib.lib(); L.nt_debug_set_cta_times.argtypes = [ctypes.c_void_p]
buf = torch.zeros(2 * 148 * 3, dtype=torch.int64, device="cuda")  # [cta][entry, exit, units << 32 | steps]
q = torch.randn(a.b, a.hq, a.n, a.d, device="cuda").bfloat16(); k = torch.randn(a.b, a.hkv, a.n, a.d, device="cuda").bfloat16()
v = torch.randn(a.b, a.hkv, a.n, a.d, device="cuda").bfloat16(); o = torch.empty(a.b, a.hq, a.n, a.d, device="cuda").bfloat16()
plan = AttentionPlan(q, k, v, o, a.d ** -0.5, "causal" if a.causal else "none")
for _ in range(3): plan.launch()
torch.cuda.synchronize()
L.nt_debug_set_cta_times(buf.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan.launch(); e1.record(); e1.synchronize()
L.nt_debug_set_cta_times(None)
t = buf.view(2 * 148, 3).cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
start = (t[:, 0] - t0) / 1e3; end = (t[:, 1] - t0) / 1e3
print(f"event {e0.elapsed_time(e1)*1e3:.1f} us; CTAs {len(t)}; start spread {start.max():.1f} us; "
      f"end: min {end.min():.1f} median {sorted(end)[len(end)//2]:.1f} max {end.max():.1f} us")
import numpy as np
e = np.sort(end)
print("end-time deciles (us):", " ".join(f"{x:.1f}" for x in np.percentile(e, [0, 10, 25, 50, 75, 90, 100])))
units = t[:, 2] >> 32
steps = t[:, 2] & 0xffffffff
dur = (t[:, 1] - t[:, 0]) / 1e3
ok = steps > 0
print(f"units per CTA: min {units.min()} max {units.max()} total {units.sum()}; steps per CTA: min {steps.min()} "
      f"median {int(np.median(steps))} max {steps.max()} total {steps.sum()}")
print(f"us per step (CTA duration / steps): median {np.median(dur[ok] / steps[ok]):.3f} "
      f"min {np.min(dur[ok] / steps[ok]):.3f} max {np.max(dur[ok] / steps[ok]):.3f}; "
      f"fixed cost fit (dur = a + b*steps): ", end="")
A = np.vstack([np.ones(ok.sum()), steps[ok], units[ok]]).T
coef = np.linalg.lstsq(A, dur[ok], rcond=None)[0]
print(f"a {coef[0]:.2f} us, b {coef[1]:.3f} us/step, c {coef[2]:.2f} us/unit")
