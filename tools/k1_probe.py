"""Run one K1 configuration in a fresh process; print ok / the failure (debug tool)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan
B, H, N, D, causal = (int(x) for x in sys.argv[1:6])
q = torch.randn(B, H, N, D, device="cuda").bfloat16()
k = torch.randn(B, H, N, D, device="cuda").bfloat16()
v = torch.randn(B, H, N, D, device="cuda").bfloat16()
o = torch.empty(B, H, N, D, device="cuda", dtype=torch.float32)
p = AttentionPlan(q, k, v, o, D ** -0.5, "causal" if causal else "none")
try:
    for _ in range(3):
        p.launch()
    torch.cuda.synchronize()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), is_causal=bool(causal))
    print("ok", sys.argv[1:6], float((o - ref).abs().max()))
except Exception as e:
    print("FAIL", sys.argv[1:6], str(e).splitlines()[0])
