"""Stress one K1 configuration: many launches with L2 flushes between them (debug tool).

    python tools/k1_stress.py B H N D causal f32 reps [e4m3]
Checks for pipeline timeouts and that every launch reproduces the first one bit for bit.
"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan
B, H, N, D, causal, f32, reps = (int(x) for x in sys.argv[1:8])
e4m3 = len(sys.argv) > 8 and sys.argv[8] == "1"
q = torch.randn(B, H, N, D, device="cuda").bfloat16()
k = torch.randn(B, H, N, D, device="cuda").bfloat16()
v = torch.randn(B, H, N, D, device="cuda").bfloat16()
if e4m3:
    q, k, v = (t.float().to(torch.float8_e4m3fn) for t in (q, k, v))
o = torch.empty(B, H, N, D, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
err = torch.zeros(1, dtype=torch.int32).pin_memory()  # host-mapped: readable after a device trap
p = AttentionPlan(q, k, v, o, D ** -0.5, "causal" if causal else "none", err_flag=err)
try:
    p.launch()
    torch.cuda.synchronize()
    first = o.clone()
    mismatches = 0
    for i in range(reps):
        flush.zero_()
        p.launch()
        if i % 25 == 0:
            torch.cuda.synchronize()
            mismatches += int(not torch.equal(o, first))
    torch.cuda.synchronize()
    mismatches += int(not torch.equal(o, first))
    print("done", sys.argv[1:], "err", int(err[0]), "mismatching checks", mismatches, flush=True)
except Exception as e:
    import time
    time.sleep(1)
    f = int(err[0]); print("FAIL", sys.argv[1:], "timed-out waits", [c for c in range(16) if f >> (8 + c) & 1], str(e).splitlines()[0])
