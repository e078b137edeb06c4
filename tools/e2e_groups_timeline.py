"""Timeline of the streamed execute_ma over (batch, kv-head) group chunks (Llama 8K, B=1):
per-chunk H2D-landed / kernel-done / D2H-done event times, to see what the e2e step waits on."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200.runtime import AttentionPlan

B, Hq, Hkv, N, D = 1, 32, 8, 8192, 128
g = Hq // Hkv
gen = torch.Generator().manual_seed(0)
qh = torch.randn(B, Hq, N, D, generator=gen).to(torch.bfloat16).pin_memory()
kh = torch.randn(B, Hkv, N, D, generator=gen).to(torch.bfloat16).pin_memory()
vh = torch.randn(B, Hkv, N, D, generator=gen).to(torch.bfloat16).pin_memory()
oh = torch.empty(B, Hq, N, D, dtype=torch.bfloat16).pin_memory()
qd, kd, vd, od = (torch.empty_like(t, device="cuda") for t in (qh, kh, vh, oh))
comp = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for n in (4, 8, 2):
    plans = []
    for c in range(n):
        h0, h1 = Hkv * c // n, Hkv * (c + 1) // n
        plans.append(AttentionPlan(qd[:, h0 * g:h1 * g], kd[:, h0:h1], vd[:, h0:h1], od[:, h0 * g:h1 * g], 0.088,
                                   "causal"))
    for rep in range(3):
        t0 = E(); t0.record(comp)
        s_in.wait_stream(comp)
        landed, kdone, odone = [], [], []
        with torch.cuda.stream(s_in):
            for c in range(n):
                h0, h1 = Hkv * c // n, Hkv * (c + 1) // n
                qd[:, h0 * g:h1 * g].copy_(qh[:, h0 * g:h1 * g], non_blocking=True)
                kd[:, h0:h1].copy_(kh[:, h0:h1], non_blocking=True)
                vd[:, h0:h1].copy_(vh[:, h0:h1], non_blocking=True)
                e = E(); e.record(s_in); landed.append(e)
        for c in range(n):
            h0, h1 = Hkv * c // n, Hkv * (c + 1) // n
            comp.wait_event(landed[c])
            plans[c].launch(comp)
            e = E(); e.record(comp); kdone.append(e)
            s_out.wait_event(e)
            with torch.cuda.stream(s_out):
                oh[:, h0 * g:h1 * g].copy_(od[:, h0 * g:h1 * g], non_blocking=True)
            e = E(); e.record(s_out); odone.append(e)
        comp.wait_stream(s_out)
        t1 = E(); t1.record(comp); t1.synchronize()
        if rep == 2:
            print(f"chunks {n}: total {t0.elapsed_time(t1):.3f} ms (plans prebuilt)")
            for c in range(n):
                print(f"  chunk {c}: H2D landed {t0.elapsed_time(landed[c]):.3f}  kernel done {t0.elapsed_time(kdone[c]):.3f}"
                      f"  D2H done {t0.elapsed_time(odone[c]):.3f}")
