"""Copy one tools/gpu_round.sh + tools/gpu_sanitize.sh run (gpurun_out/round, gpurun_out/sanitize)
into profiles/<dest>/ and refresh profiles/latest_<config>_ncu.json (bench.py's `traffic` source).

    python tools/collect_round.py r02_final
"""
import glob
import json
import os
import shutil
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(REPO, "gpurun_out", "round")
san = os.path.join(REPO, "gpurun_out", "sanitize")
dst = os.path.join(REPO, "profiles", sys.argv[1] if len(sys.argv) > 1 else "latest_round")
os.makedirs(dst, exist_ok=True)
for f in glob.glob(os.path.join(src, "bench_*.json.log")):
    lines = [ln for ln in open(f).read().splitlines() if ln.startswith("{")]
    if lines:
        with open(os.path.join(dst, os.path.basename(f)[:-4]), "w") as o:
            o.write(lines[-1] + "\n")
for pat in ("*_ncu.json", "*_stalls.txt", "launches_llama8k.csv", "latency_attn256.txt", "tune_*.json",
            "nvidia_smi.txt", "smoke.log"):
    for f in glob.glob(os.path.join(src, pat)):
        shutil.copy(f, dst)
with open(os.path.join(src, "pytest_gpu.log")) as f:
    tail = f.read().splitlines()[-3:]
with open(os.path.join(dst, "pytest_gpu_tail.txt"), "w") as o:
    o.write("\n".join(tail) + "\n")
with open(os.path.join(dst, "sanitize_summary.txt"), "w") as o:
    for f in sorted(glob.glob(os.path.join(san, "*.log"))):
        last = [ln for ln in open(f).read().splitlines() if "ERROR SUMMARY" in ln or "RACECHECK SUMMARY" in ln]
        o.write(f"== {os.path.basename(f)[:-4]}: {last[-1] if last else ''}\n")
    p = os.path.join(san, "plain.log")
    if os.path.exists(p):
        o.write("\nplain:\n" + "\n".join(open(p).read().splitlines()[-30:]) + "\n")
# bench.py reads profiles/latest_<config>_ncu.json for the roofline's `traffic`
latest = {"llama8k_causal": "attn_llama8k", "bert512": "attn_bert512", "decode32k": "decode32k",
          "decode32k_paged16": "decode32k_paged16", "decode32k_e4m3": "decode32k_e4m3",
          "gemm_chain_e4096": "gemm4k", "gemm_chain_e128": "gemm_e128",
          "llama8k_causal_1group": "attn_1group", "llama8k_causal_e4m3": "attn_llama8k_e4m3"}
for cfg, cap in latest.items():
    f = os.path.join(dst, f"{cap}_ncu.json")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(REPO, "profiles", f"latest_{cfg}_ncu.json"))
for f in sorted(glob.glob(os.path.join(dst, "bench_*.json"))):
    d = json.load(open(f))
    r = d.get("roofline", {})
    print(f"{os.path.basename(f)[6:-5]:28s} {d.get('value', 0):10.2f} {d.get('unit', ''):8s} "
          f"ms {d.get('ms_per_step', 0):8.4f} frac {r.get('frac', 0):.3f} read-ceiling {r.get('frac_of_read_ceiling', '-')}")
