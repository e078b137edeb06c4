"""cuBLAS (torch.matmul) bf16 at the GEMM-chain shapes, for context next to K3."""
import torch
for (M, N, K) in [(4096, 4096, 4096), (4096, 128, 4096), (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(K, N, device="cuda").bfloat16()
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): c = a @ b
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cuBLAS {M}x{N}x{K}: {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.0f} TFLOP/s")
