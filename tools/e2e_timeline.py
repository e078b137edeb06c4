"""Timeline of the streamed execute_ma (query-row chunks): per-chunk H2D / kernel / D2H event times."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200 import _lib
from paper_2604_14825_b200.runtime import AttentionPlan
B, Hq, Hkv, N, D = 1, 32, 8, 8192, 128
g = torch.Generator().manual_seed(0)
qh = torch.randn(B, Hq, N, D, generator=g).to(torch.bfloat16).pin_memory()
kh = torch.randn(B, Hkv, N, D, generator=g).to(torch.bfloat16).pin_memory()
vh = torch.randn(B, Hkv, N, D, generator=g).to(torch.bfloat16).pin_memory()
oh = torch.empty(B, Hq, N, D, dtype=torch.bfloat16).pin_memory()
qd, kd, vd, od = (torch.empty_like(t, device="cuda") for t in (qh, kh, vh, oh))
L = _lib.lib()
comp = torch.cuda.current_stream()
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
def copy2d(dst, src, r0, r1, rows, height, st):
    pitch = rows * D * 2
    L.nt_memcpy2d_async(dst.data_ptr() + r0 * D * 2, pitch, src.data_ptr() + r0 * D * 2, pitch, (r1 - r0) * D * 2, height, st.cuda_stream)
for n in (4, 8):
    for rep in range(3):
        bounds = [N * c // n for c in range(n + 1)]
        E = lambda: torch.cuda.Event(enable_timing=True)
        t0 = E(); t0.record(comp)
        s_in.wait_stream(comp)
        marks = []
        kv = 0
        for r0, r1 in zip(bounds[:-1], bounds[1:]):
            copy2d(qd, qh, r0, r1, N, B * Hq, s_in); copy2d(kd, kh, kv, r1, N, B * Hkv, s_in); copy2d(vd, vh, kv, r1, N, B * Hkv, s_in)
            kv = r1
            e_in = E(); e_in.record(s_in)
            comp.wait_stream(s_in)
            p = AttentionPlan(qd[:, :, r0:r1], kd[:, :, :r1], vd[:, :, :r1], od[:, :, r0:r1], 0.088, "causal", causal_offset=r0)
            p.launch(comp)
            e_k = E(); e_k.record(comp)
            s_out.wait_stream(comp)
            copy2d(oh, od, r0, r1, N, B * Hq, s_out)
            e_out = E(); e_out.record(s_out)
            marks.append((e_in, e_k, e_out, p))
        comp.wait_stream(s_out)
        t1 = E(); t1.record(comp); t1.synchronize()
    print(f"n={n}: total {t0.elapsed_time(t1):.3f} ms")
    for i, (a, b, c, _) in enumerate(marks):
        print(f"  chunk {i}: h2d done {t0.elapsed_time(a):.3f}  kernel done {t0.elapsed_time(b):.3f}  d2h done {t0.elapsed_time(c):.3f}")
