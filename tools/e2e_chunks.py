import sys, time, json
sys.path.insert(0, '.')
import torch
from bench import CONFIGS, load_ma
from paper_2604_14825_b200 import execute_ma
from paper_2604_14825_b200.recognize import recognize
for cfgname in ("llama8k_causal", "bert512"):
    cfg = CONFIGS[cfgname]
    mod, _ = load_ma(cfg)
    spec = recognize(mod)[0]
    B, Hq, Hkv, N, D = cfg["B"], cfg["Hq"], cfg["Hkv"], cfg["N"], cfg["D"]
    q = torch.randn(B, Hq, N, D).bfloat16().pin_memory()
    k = torch.randn(B, Hkv, N, D).bfloat16().pin_memory()
    v = torch.randn(B, Hkv, N, D).bfloat16().pin_memory()
    out = torch.empty(B, Hq, N, D, dtype=torch.bfloat16).pin_memory()
    for ch in (2, 4, 8, 16):
        kw = dict(outer=(B, Hq, Hkv), mask_kind="causal" if cfg["causal"] else "none", out_dtype="bf16", return_torch=True, out=out, chunks=ch)
        for _ in range(3): execute_ma(mod, {spec.q: q, spec.k: k, spec.v: v}, **kw)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); execute_ma(mod, {spec.q: q, spec.k: k, spec.v: v}, **kw); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(cfgname, "chunks", ch, "e2e ms", round(min(ts), 3), round(sorted(ts)[2], 3))
