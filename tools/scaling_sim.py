"""Per-rank compute of the (batch, kv-head) sharding at 1/2/4/8 GPUs, measured on one B200.

For world size N every rank holds Hkv/N kv-groups of Llama-3-8B 8K causal (B=1) --
identical shards -- so the box's compute-only time is one rank's kernel time and the
compute-only box throughput is total FLOPs / that time.  The NCCL all-gather of O
(67 MB at N=8) is not included (this run has one GPU; bench.py reports it as
ms_per_step_with_gather when it runs under torchrun).
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_14825_b200.runtime import AttentionPlan  # noqa: E402
from paper_2604_14825_b200.shard import plan_shard  # noqa: E402

B, HQ, HKV, N, D = 1, 32, 8, 8192, 128
total = 2.0 * B * HQ * D * N * (N + 1)
flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
rows = []
for world in (1, 2, 4, 8):
    sh = plan_shard(B, HKV, world, 0)
    hkv = sh.h1 - sh.h0
    hq = hkv * (HQ // HKV)
    q = torch.randn(B, hq, N, D, device="cuda").bfloat16()
    k = torch.randn(B, hkv, N, D, device="cuda").bfloat16()
    v = torch.randn(B, hkv, N, D, device="cuda").bfloat16()
    o = torch.empty(B, hq, N, D, device="cuda").bfloat16()
    plan = AttentionPlan(q, k, v, o, D ** -0.5, "causal")
    for _ in range(3):
        plan.launch()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.launch()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    rows.append({"gpus": world, "rank_q_heads": hq, "rank_kernel_us": ms * 1e3, "split_kv": plan.ws is not None,
                 "box_tflops_compute_only": total / (ms * 1e-3) / 1e12})
base = rows[0]["box_tflops_compute_only"]
for r in rows:
    r["compute_only_scaling_efficiency"] = r["box_tflops_compute_only"] / (base * r["gpus"])
print(json.dumps(rows, indent=1))
