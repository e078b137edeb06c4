"""K1 (256-row items) vs K1w (512-row items, four softmax warpgroups) at D=64, no mask."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan
for (B, H, N) in [(32, 12, 512), (1, 48, 4096), (4, 37, 2048), (1, 16, 16384)]:
    q = torch.randn(B, H, N, 64, device="cuda").bfloat16()
    k = torch.randn(B, H, N, 64, device="cuda").bfloat16()
    v = torch.randn(B, H, N, 64, device="cuda").bfloat16()
    o = torch.empty_like(q)
    res = []
    for rows in (256, 512):
        p = AttentionPlan(q, k, v, o, 0.125, "none", item_rows=rows)
        for _ in range(3):
            p.launch()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); p.launch(); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = sorted(ts)[5]
        res.append(f"rows {rows}: {ms*1e3:8.1f} us {p.flops()/ms/1e9:7.1f} TF")
    print(f"B={B} H={H} N={N}: " + " | ".join(res))
