"""Split-KV units vs one unit per item on few-item shapes (per-GPU load at 2/4/8 GPUs)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan

for (Hq, Hkv, N, causal) in [(4, 1, 8192, True), (8, 2, 8192, True), (16, 4, 8192, True), (32, 8, 8192, True),
                             (2, 2, 4096, False)]:
    q = torch.randn(1, Hq, N, 128, device="cuda").bfloat16()
    k = torch.randn(1, Hkv, N, 128, device="cuda").bfloat16()
    v = torch.randn(1, Hkv, N, 128, device="cuda").bfloat16()
    o = torch.empty_like(q)
    res = []
    for split in (True, False):
        p = AttentionPlan(q, k, v, o, 0.088, "causal" if causal else "none")
        if not split:
            p.args.workspace = None
        flush = torch.empty(64 * 1024 * 1024, device="cuda")
        for _ in range(3):
            p.launch()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); p.launch(); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[5]
        res.append((split and p.ws is not None, ms, p.flops() / ms / 1e9))
    print(f"Hq={Hq} Hkv={Hkv} N={N} causal={causal}: " +
          "  ".join(f"{'split' if s else 'whole'} {ms*1e3:.1f} us {tf:.0f} TFLOP/s" for s, ms, tf in res))
