"""K1 timing vs the MA `stages` tunable (K/V ring depth)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan
for (B, Hq, Hkv, N, D, causal) in [(1, 32, 8, 8192, 128, True), (32, 12, 12, 512, 64, False), (1, 32, 8, 2048, 128, True)]:
    q = torch.randn(B, Hq, N, D, device="cuda").bfloat16(); k = torch.randn(B, Hkv, N, D, device="cuda").bfloat16()
    v = torch.randn(B, Hkv, N, D, device="cuda").bfloat16(); o = torch.empty(B, Hq, N, D, device="cuda").bfloat16()
    res = []
    for st in (1, 2):
        p = AttentionPlan(q, k, v, o, D ** -0.5, "causal" if causal else "none", kv_stages=st)
        for _ in range(3): p.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): p.launch()
        e1.record(); e1.synchronize()
        res.append(f"stages={st} ({p.kv_slots} slots): {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
    print((B, Hq, N, D, causal), "; ".join(res))
