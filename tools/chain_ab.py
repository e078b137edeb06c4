"""A/B: fused chain kernel vs two K3 GEMMs for the GEMM-chain MA at several shapes."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.gemm import ChainPlan
for (N, K, F, E) in [(4096, 4096, 4096, 128), (4096, 4096, 4096, 256), (128, 1024, 256, 128), (256, 256, 512, 128),
                     (1024, 4096, 4096, 128), (4096, 1024, 1024, 128), (8192, 4096, 4096, 128)]:
    x = torch.randn(N, K, device="cuda").bfloat16()
    w1 = (torch.randn(K, F, device="cuda") / K ** 0.5).bfloat16()
    w2 = (torch.randn(F, E, device="cuda") / F ** 0.5).bfloat16()
    res = {}
    for force in (False, True):
        y = torch.empty(N, E, device="cuda", dtype=torch.float32)
        p = ChainPlan(x, w1, w2, y, force_two_gemms=force)
        for _ in range(3):
            p.launch()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(20):
            p.launch()
        ev[1].record()
        ev[1].synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 20
        res[p.realisation] = (ms, p.flops / ms / 1e9)
    print(N, K, F, E, {k: (round(v[0] * 1e3, 1), round(v[1], 1)) for k, v in res.items()})
