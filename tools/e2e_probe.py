"""Streamed execute_ma timing vs chunk count; host enqueue time (Llama 8K causal, B=1)."""
import json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2604_14825_b200 import execute_ma, ma_ir
mod = ma_ir.from_json(open("tests/golden/causal8k.seed0.ma.json").read())
B, Hq, Hkv, N, D = 1, 32, 8, 8192, 128
g = torch.Generator().manual_seed(0)
host = {"Q": torch.randn(B, Hq, N, D, generator=g).to(torch.bfloat16).pin_memory(),
        "K": torch.randn(B, Hkv, N, D, generator=g).to(torch.bfloat16).pin_memory(),
        "V": torch.randn(B, Hkv, N, D, generator=g).to(torch.bfloat16).pin_memory()}
out = torch.empty(B, Hq, N, D, dtype=torch.bfloat16).pin_memory()
kw = dict(outer=(B, Hq, Hkv), mask_kind="causal", out_dtype="bf16", return_torch=True, out=out)
for chunks in (1, 2, 3, 4, 6, 8, 16):
    for _ in range(3):
        execute_ma(mod, host, chunks=chunks, **kw)
    ts, hs = [], []
    for _ in range(10):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        _, rep = execute_ma(mod, host, chunks=chunks, **kw)
        e1.record(); e1.synchronize()
        hs.append(time.perf_counter() - t0)
        ts.append(e0.elapsed_time(e1))
    print(f"chunks {chunks:3d}: e2e {min(ts):.3f} ms (median {sorted(ts)[5]:.3f}), wall {min(hs)*1e3:.3f} ms, "
          f"device_ms {rep.device_ms:.3f}")
