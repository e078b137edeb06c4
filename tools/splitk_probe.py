"""Time the GEMM chain's second GEMM (T.W2, 4096 x E x 4096) with and without split K."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200 import _lib
from paper_2604_14825_b200.gemm import GemmPlan

for (M, N, K) in [(4096, 128, 4096), (4096, 64, 4096), (4096, 4096, 4096)]:
    a = torch.randn(M, K, device="cuda").bfloat16()
    b = (torch.randn(K, N, device="cuda") / K ** 0.5).bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for force in (None, 1, 2, 4, 6, 8):
        if M == 4096 and N == 4096 and force not in (None, 1):
            continue
        p = GemmPlan(a, b, c)
        if force:
            p.args.k_splits = min(force, p.args.k_splits) if force > 1 else 1
        for _ in range(3):
            p.launch()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            p.launch()
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{M}x{N}x{K} splits={p.args.k_splits}: {ms*1e3:.1f} us")
