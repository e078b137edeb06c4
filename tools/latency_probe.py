"""Config-1 latency: one 256x256x64 attention launch, event-timed alone, back-to-back, and in a CUDA graph."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan
dev = torch.device("cuda")
q, k, v = (torch.randn(1, 1, 256, 64, device=dev).bfloat16() for _ in range(3))
o = torch.empty(1, 1, 256, 64, device=dev, dtype=torch.float32)
plan = AttentionPlan(q, k, v, o, None, "none")
for _ in range(10): plan.launch()
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)
# single launches
ts = []
for _ in range(50):
    a, b = E(), E(); a.record(); plan.launch(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
print(f"single launch (events around it): median {sorted(ts)[25]:.2f} us, min {min(ts):.2f} us")
# back-to-back
a, b = E(), E(); a.record()
for _ in range(200): plan.launch()
b.record(); b.synchronize()
print(f"back-to-back: {a.elapsed_time(b) * 1e3 / 200:.2f} us per launch")
# CUDA graph of 20 launches
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    plan.launch(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20): plan.launch(s)
torch.cuda.synchronize()
a, b = E(), E(); a.record()
for _ in range(10): g.replay()
b.record(); b.synchronize()
print(f"graph replay: {a.elapsed_time(b) * 1e3 / 200:.2f} us per launch")
