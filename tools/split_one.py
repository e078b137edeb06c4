"""One split-KV launch pair (Hq=4, 8K causal) for an ncu launch list."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan
q = torch.randn(1, 4, 8192, 128, device="cuda").bfloat16()
k = torch.randn(1, 1, 8192, 128, device="cuda").bfloat16()
v = torch.randn(1, 1, 8192, 128, device="cuda").bfloat16()
o = torch.empty_like(q)
p = AttentionPlan(q, k, v, o, 0.088, "causal")
for _ in range(4):
    p.launch()
torch.cuda.synchronize()
