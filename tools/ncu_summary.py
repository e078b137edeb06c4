"""Summarise an `ncu --set full` report (read here, no GPU needed) into profiles/*.json.

    python tools/ncu_summary.py gpurun_out/attn8k.ncu-rep profiles/attn_fwd_ncu_summary.json \
        --workload llama8k_causal --algorithmic-bytes 167772160 --algorithmic-flops 5.4976e11
"""

import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1.0),
    "sm_clock_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "dram_read_MB": ("dram__bytes_read.sum", 1.0),
    "dram_write_MB": ("dram__bytes_write.sum", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tcgen05_bf16_ops_pct": ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 1.0),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    "fma_pipe_pct": ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pipe_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    "registers_per_thread": ("launch__registers_per_thread", 1.0),
    "smem_tc_wavefronts_pct": ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1.0),
}
STALLS = ["long_scoreboard", "wait", "barrier", "selected", "not_selected", "short_scoreboard",
          "branch_resolving", "no_instructions", "math_pipe_throttle", "mio_throttle", "dispatch_stall"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        launches.append({h: (u, v) for h, u, v in zip(hdr, units, vals)})
    return launches


def to_float(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return None


def summarise(rep, workload, alg_bytes=None, alg_flops=None):
    ls = raw(rep)
    d = ls[0]
    out = {"report": rep, "workload": workload, "kernel": d.get("Kernel Name", ("", ""))[1]}
    for k, (m, _) in KEYS.items():
        if m in d:
            out[k] = to_float(d[m][1])
            out[k + "_unit"] = d[m][0]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = (out.get("dram_read_MB") or 0.0) * scale.get(out.get("dram_read_MB_unit", "Mbyte"), 1.0)
    wr = (out.get("dram_write_MB") or 0.0) * scale.get(out.get("dram_write_MB_unit", "Mbyte"), 1.0)
    out["dram_read_MB"], out["dram_write_MB"] = rd / 1e6, wr / 1e6
    out["dram_read_MB_unit"] = out["dram_write_MB_unit"] = "Mbyte"
    out["dram_bytes_per_launch"] = rd + wr
    tscale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    if "duration_us" in out:
        out["duration_us"] = out["duration_us"] * tscale.get(out.get("duration_us_unit", "us"), 1.0)
        out["duration_us_unit"] = "us"
    tot = to_float(d.get("smsp__pcsamp_sample_count", ("", "0"))[1]) or 1.0
    out["stall_samples_pct"] = {s: round(100.0 * (to_float(d.get(f"smsp__pcsamp_warps_issue_stalled_{s}", ("", "0"))[1]) or 0.0) / tot, 1)
                                for s in STALLS}
    if alg_bytes:
        out["algorithmic_bytes"] = alg_bytes
    if alg_flops and out.get("duration_us"):
        out["algorithmic_flops"] = alg_flops
        out["tflops_under_ncu_clock"] = alg_flops / (out["duration_us"] * 1e-6) / 1e12
    if alg_bytes and out.get("duration_us"):
        out["gbs_under_ncu_clock"] = alg_bytes / (out["duration_us"] * 1e-6) / 1e9
        out["traffic_over_algorithmic"] = out["dram_bytes_per_launch"] / alg_bytes
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--workload", default="")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--algorithmic-flops", type=float, default=None)
    a = ap.parse_args()
    s = summarise(a.report, a.workload, a.algorithmic_bytes, a.algorithmic_flops)
    with open(a.out, "w") as f:
        json.dump(s, f, indent=1, sort_keys=True)
    print(json.dumps(s, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
