"""Regenerate DESIGN.md §7's measured table from profiles/<dir>/ (bench lines, ncu summaries,
latency / smoke / tuner files): python tools/design_table.py r02_final"""
import json
import os
import re
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(REPO, "profiles", sys.argv[1] if len(sys.argv) > 1 else "r02_final") + "/"


def b(n):
    return json.load(open(P + f"bench_{n}.json"))


def v(n):
    return b(n)["value"]


def f(n):
    return b(n)["roofline"]["frac"]


def ms(n):
    return b(n)["ms_per_step"]


def rc(n):
    return b(n)["roofline"].get("frac_of_read_ceiling")


def e2e(n):
    return (b(n).get("e2e") or {}).get("value")


ncu = json.load(open(P + "attn_llama8k_ncu.json"))
dn = json.load(open(P + "decode32k_ncu.json"))
gr = re.search(r"graph replay: ([0-9.]+) us", open(P + "latency_attn256.txt").read()).group(1)
sd = re.search(r"device ([0-9.]+) us", open(P + "smoke.log").read()).group(1)
tb = json.load(open(P + "tune_bert512.json"))
ref, ref8 = b("reference"), b("llama8k_causal")["cpu_baseline"]
npass = re.search(r"(\d+) passed", open(P + "pytest_gpu_tail.txt").read()).group(1)
rows = f"""| workload | value | roofline frac (of MEASURED_PEAKS) |
|---|---|---|
| Llama-3-8B causal prefill, 8K, B=1 (config 4, default bench) | {v('llama8k_causal'):.0f} TFLOP/s (e2e {e2e('llama8k_causal'):.0f}) | {f('llama8k_causal'):.3f} of 1643.8 (≥60 % target met); ncu tensor pipe {ncu['tensor_pipe_active_pct']:.1f} % |
| Llama 16K / 4K / 2K causal | {v('llama16k_causal'):.0f} / {v('llama4k_causal'):.0f} / {v('llama2k_causal'):.0f} TFLOP/s | {f('llama16k_causal'):.2f} / {f('llama4k_causal'):.2f} / {f('llama2k_causal'):.2f} |
| Llama 8K causal, one kv-group (the 8-GPU per-rank load, split-KV) | {v('llama8k_causal_1group'):.0f} TFLOP/s | {f('llama8k_causal_1group'):.2f} (r01: 0.39) |
| Llama 8K causal, FP8-E4M3 inputs | {v('llama8k_causal_e4m3'):.0f} TFLOP/s (e2e {e2e('llama8k_causal_e4m3'):.0f}) | {f('llama8k_causal_e4m3'):.2f} of 2 × 1643.8 |
| Llama 4K, random 0 / −inf mask as bits (the same mask as fp32) | {v('llama4k_mask_bits'):.0f} ({v('llama4k_mask_f32'):.0f}) TFLOP/s, dense-equivalent | {f('llama4k_mask_bits'):.2f} ({f('llama4k_mask_f32'):.2f}) |
| BERT-base MHA 512, B=32 (config 3) | {v('bert512'):.0f} TFLOP/s (e2e {e2e('bert512'):.1f}) | {f('bert512'):.2f} (r01: 0.26) |
| GEMM chain 4096³×4096 (config 2, two K3 GEMMs on CTA pairs) | {v('gemm_chain_e4096'):.0f} TFLOP/s | {f('gemm_chain_e4096'):.2f} |
| GEMM chain 4096³×128 (config 2 parity shape; T·W2 split-K) | {v('gemm_chain_e128'):.0f} TFLOP/s | {f('gemm_chain_e128'):.2f} |
| decode B=64, 32K (config 5), K2b tensor-core decode | {ms('decode32k'):.3f} ms | {rc('decode32k'):.2f} of the 7.4 TB/s read ceiling ({f('decode32k'):.2f} of the 6450 GB/s copy peak); ncu DRAM {dn['dram_throughput_pct']:.1f} % |
| decode B=64, 64K / 128K (config 5 sweep; 17.2 / 34.4 GB of K/V) | {ms('decode64k'):.3f} / {ms('decode128k'):.3f} ms | {rc('decode64k'):.2f} / {rc('decode128k'):.2f} of the read ceiling |
| decode 32K, paged KV, 64- / 16-token pages (K2b) | {ms('decode32k_paged64'):.3f} / {ms('decode32k_paged16'):.3f} ms | {rc('decode32k_paged64'):.2f} / {rc('decode32k_paged16'):.2f} of the read ceiling |
| decode B=64, 32K, FP8 (e4m3) KV cache (K2b `kind::f8f6f4`) | {ms('decode32k_e4m3'):.3f} ms (half the bytes) | {rc('decode32k_e4m3'):.2f} of the read ceiling |
| decode 32K, FP8 paged KV, 64- / 16-token pages | {ms('decode32k_e4m3_paged64'):.3f} / {ms('decode32k_e4m3_paged16'):.3f} ms | {rc('decode32k_e4m3_paged64'):.2f} / {rc('decode32k_e4m3_paged16'):.2f} of the read ceiling |
| config 1 (attn256) | {ms('attn256')*1e3:.1f} µs per bench step (a CUDA-graph replay after a 256 MiB L2 flush; 13-17 µs across boxes); {gr} µs per back-to-back graph replay (paper, GH200: 7.43 µs); `smoke()` device time {sd} µs | latency-bound |
| reference CPU executor (Llama 8K), 1 core / {ref['cpu_baseline']['cores']} processes | {ref8['value']:.5f} / {ref['value']:.4f} TFLOP/s | — |

GPU tests {npass} passed; compute-sanitizer memcheck / synccheck / initcheck / racecheck over
every kernel family 0 errors, 0 hazards (`sanitize_summary.txt`).
Tuner: BERT device pick {tb['device_pick']['device_us']:.1f} µs vs analytic pick {tb['analytic_pick']['device_us']:.1f} µs ({tb['device_pick_speedup']:.2f}x).
"""
path = os.path.join(REPO, "DESIGN.md")
s = open(path).read()
a = s.index("| workload | value | roofline frac (of MEASURED_PEAKS) |")
z = s.index("GPU tests ", a)
z = s.index("\n", s.index("Tuner: BERT device pick", z)) + 1
s = s[:a] + rows + s[z:]
open(path, "w").write(s)
print(rows)
