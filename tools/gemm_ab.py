"""K3 GEMM timing at the chain shapes (run twice: default and NT_GEMM_1SM=1)."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.gemm import GemmPlan
tag = "1sm" if os.environ.get("NT_GEMM_1SM") else "2sm"
for (M, N, K) in [(4096, 4096, 4096), (8192, 8192, 8192), (4096, 1024, 4096), (512, 4096, 1024)]:
    a = torch.randn(M, K, device="cuda").bfloat16(); b = (torch.randn(K, N, device="cuda") / K ** 0.5).bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    p = GemmPlan(a, b, c)
    for _ in range(3): p.launch()
    torch.cuda.synchronize()
    ref = (a.float() @ b.float())
    err = float((c.float() - ref).abs().max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): p.launch()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{tag} {M}x{N}x{K}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.0f} TFLOP/s  max-abs err {err:.3e}")
