#!/usr/bin/env python
"""Benchmark: Nautilus-discovered fused attention on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Default workload (the one BASELINE.json's metric/target is quoted on):
Llama-3-8B GQA causal prefill, bf16, B=1, Hq=32, Hkv=8, D=128, seq 8192, the
MA kernel the reference auto-scheduler discovers for SURVEY.md Appendix A.3
(seed 0, default tiles), executed by the sm_100a K1 kernel over the runtime's
batch x head outer grid.  A "step" is one pass of the hot path over that batch.

Timing: W untimed warm-up steps, then K steps each bracketed by CUDA events on
the launching stream, with a >L2 (256 MiB) write between steps to flush L2;
barrier + synchronize on both sides; max over ranks.  Multi-GPU: (batch,
kv-head) groups are sharded across ranks (no data-path collective) and O is
all-gathered with NCCL inside the step.

Extra keys: e2e (same metric through the public API execute_ma with pinned
host inputs, H2D + kernel + D2H in the timed region), roofline (dominant
kernel vs MEASURED_PEAKS.json), cpu_baseline (the reference CPU executor on a
bounded sample), clocks (nvidia-smi during the timed region), gpu_launches.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)
REF_PATH = os.path.join(REPO, "baseline", "_ref")

LLAMA_SCALE = 0.08838834764831845

CONFIGS = {
    # name: workload (MA program + runtime outer grid)
    "llama8k_causal": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=8192, D=128, causal=True,
                           golden="causal8k", scale=LLAMA_SCALE),
    "llama2k_causal": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=2048, D=128, causal=True,
                           golden="causal2k", scale=LLAMA_SCALE),
    "llama4k_causal": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=4096, D=128, causal=True,
                           golden="causal4k", scale=LLAMA_SCALE),
    "llama16k_causal": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=16384, D=128, causal=True,
                            golden="causal16k", scale=LLAMA_SCALE),
    # one GPU's share at 8 GPUs (batch x head sharding: one kv-group, 4 q-heads): few,
    # long causal items -> K1 split-KV work units
    "llama8k_causal_1group": dict(prog="llama_causal", B=1, Hq=4, Hkv=1, N=8192, D=128, causal=True,
                                  golden="causal8k", scale=LLAMA_SCALE),
    # the paper's FP8 regime: e4m3 Q/K/V with per-tensor descales, kind::f8f6f4
    "llama8k_causal_e4m3": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=8192, D=128, causal=True,
                                golden="causal8k", scale=LLAMA_SCALE, in_dtype="e4m3"),
    # a general (non-causal) 0 / -inf Mask input to the masked MA program: random 50 %
    # key visibility per row, realised as visibility bits (NT_MASK_BITS) or, for
    # comparison, as the fp32 tensor the MA reads (NT_MASK_TENSOR)
    "llama4k_mask_bits": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=4096, D=128, causal=False,
                              golden="causal4k", scale=LLAMA_SCALE, mask="bits"),
    "llama4k_mask_f32": dict(prog="llama_causal", B=1, Hq=32, Hkv=8, N=4096, D=128, causal=False,
                             golden="causal4k", scale=LLAMA_SCALE, mask="tensor"),
    "bert512": dict(prog="scaled_0p125", B=32, Hq=12, Hkv=12, N=512, D=64, causal=False,
                    golden="bert512", scale=0.125),
    # latency-bound (two CTAs): each step replays a CUDA graph of the launch, the way a
    # serving loop issues it (the paper's GH200 ablation: 7.43 us)
    "attn256": dict(prog="attention", B=1, Hq=1, Hkv=1, N=256, D=64, causal=False,
                    golden="attn256", scale=None, graph=True),
    # config 5: decode, the 4 q-heads of a GQA group packed as the MA's 4 rows
    "decode32k": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128, causal=False,
                      golden="decode4_32k", scale=LLAMA_SCALE),
    # the long end of config 5 (KV 128K: 34.4 GB of K/V; e2e skipped -- the pinned host
    # copy alone would be 34 GB per step)
    # the same decode over an FP8 (e4m3) KV cache: half the bytes per key (kind::f8f6f4 dots)
    "decode32k_e4m3": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128, causal=False,
                           golden="decode4_32k", scale=LLAMA_SCALE, in_dtype="e4m3"),
    "decode32k_e4m3_paged16": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128,
                                   causal=False, golden="decode4_32k", scale=LLAMA_SCALE, in_dtype="e4m3",
                                   page_size=16),
    "decode32k_e4m3_paged16_hnd": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128,
                                       causal=False, golden="decode4_32k", scale=LLAMA_SCALE, in_dtype="e4m3",
                                       page_size=16, page_layout="HND"),
    "decode32k_e4m3_paged64": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128,
                                   causal=False, golden="decode4_32k", scale=LLAMA_SCALE, in_dtype="e4m3",
                                   page_size=64),
    "decode64k": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=65536, D=128, causal=False,
                      golden="decode4_64k", scale=LLAMA_SCALE),
    "decode128k": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=131072, D=128, causal=False,
                       golden="decode4_128k", scale=LLAMA_SCALE, no_e2e=True),
    # the same decode over a paged KV cache (16-token pages, shuffled block table)
    "decode32k_paged16": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128, causal=False,
                              golden="decode4_32k", scale=LLAMA_SCALE, page_size=16),
    "decode32k_paged16_hnd": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128,
                                  causal=False, golden="decode4_32k", scale=LLAMA_SCALE, page_size=16,
                                  page_layout="HND"),
    "decode32k_paged64": dict(kind="decode", prog="llama", B=64, Hq=32, Hkv=8, N=1, M=32768, D=128, causal=False,
                              golden="decode4_32k", scale=LLAMA_SCALE, page_size=64),
    # config 2: (X.W1).W2 at 4096^3 x E=4096 (schedulable with max_tile_elems >= 262144)
    "gemm_chain_e4096": dict(kind="gemm_chain", prog="gemm2", N=4096, K=4096, F=4096, E=4096,
                             golden="gemm4k_e4096", causal=False, B=1, Hq=1, Hkv=1, D=0),
    "gemm_chain_e128": dict(kind="gemm_chain", prog="gemm2", N=4096, K=4096, F=4096, E=128,
                            golden="gemm4k_e128", causal=False, B=1, Hq=1, Hkv=1, D=0),
}
DEFAULT_CONFIG = "llama8k_causal"
METRIC = "fused-attention bf16 TFLOP/s & % tensor peak; box throughput at 1/2/4/8 GPUs"
READ_CEILING_GBS = 7398.7  # tools/ubench/bulk_read.cu, B200, r02 (HBM read-only stream through TMA)


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, "fallback"


def load_ma(cfg):
    """The MA module: the committed reference export, else the reference pipeline live."""
    from paper_2604_14825_b200 import ma_ir

    p = os.path.join(REPO, "tests", "golden", f"{cfg['golden']}.seed0.ma.json")
    if os.path.exists(p):
        with open(p) as f:
            return ma_ir.from_json(f.read()), "tests/golden/" + os.path.basename(p)
    sys.path.insert(0, REF_PATH)
    from paper_2604_14825_b200.frontdoor import compile_program
    return compile_program(cfg["prog"], dict(N=cfg["N"], M=cfg["N"], D=cfg["D"]))[0], "tilecc (live)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = f"/tmp/nt_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    rows.append((float(parts[1]), float(parts[2]), parts[4:9]))
                except ValueError:
                    continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, r in rows:
            for n, v in zip(names, r[1:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm = [r[0] for r in rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU baseline
def _sliced_module(ma, nblocks):
    import dataclasses
    k = ma.kernels[0]
    v, ax, _ = k.blocks[0]
    return dataclasses.replace(ma, kernels=(dataclasses.replace(k, blocks=((v, ax, nblocks),)),))


def _cpu_inputs(module):
    """Seeded inputs for every input buffer of the MA module (causal pattern for Mask)."""
    import numpy as np
    rng = np.random.default_rng(0)
    inp = {}
    for b in module.buffers:
        if not b.is_input:
            continue
        shape = tuple(b.shape)
        if b.name == "Mask":
            n, m = shape
            inp[b.name] = np.where(np.arange(m)[None, :] <= np.arange(n)[:, None], np.float32(0),
                                   np.float32(-np.inf)).astype(np.float32)
        else:
            inp[b.name] = (rng.standard_normal(shape) / (np.sqrt(shape[0]) if b.name.startswith("W") else 1.0)
                           ).astype(np.float32)
    return inp


_POOL_STATE = {}


def _port_worker(nblocks):
    from oracle import ma_interp
    t = time.perf_counter()
    ma_interp.interpret_ma(_sliced_module(_POOL_STATE["ma"], nblocks), _POOL_STATE["inp"], account=True)
    return time.perf_counter() - t


def _ref_worker(nblocks):
    from tilecc.ma.device import DEFAULT_DEVICE
    from tilecc.ma.interp import interpret_ma
    ma, inp = _POOL_STATE["ma"], _POOL_STATE["inp"]
    t = time.perf_counter()
    interpret_ma(_sliced_module(ma, nblocks), inp, DEFAULT_DEVICE, "fp32")
    return time.perf_counter() - t


def reference_module(cfg):
    """Reference MA via the reference's own pipeline (baseline/_ref), or None."""
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        import dataclasses
        from tilecc.autosched.scheduler import SchedulerOptions, run_autoscheduler
        from tilecc.ma.device import DEFAULT_DEVICE
        from tilecc.pipeline import frontend, lower_seed
        from paper_2604_14825_b200.programs import PROGRAMS
    except Exception:
        return None
    binding, devo, _ = cpu_binding(cfg)
    device = dataclasses.replace(DEFAULT_DEVICE, **devo) if devo else DEFAULT_DEVICE
    bound, base = frontend(PROGRAMS[cfg["prog"]], binding)
    seeds = run_autoscheduler(base, device, SchedulerOptions())
    return lower_seed(base, seeds[0].schedule, device).ma


def cpu_baseline_sample(cfg, full_flops, target_s=10.0):
    """Time the reference CPU executor (or the oracle port) on a bounded sample, 1 core."""
    ma = reference_module(cfg)
    total_blocks_per_slice = None
    if ma is not None:
        inp = _cpu_inputs(ma)
        from tilecc.ma.device import DEFAULT_DEVICE
        from tilecc.ma.interp import interpret_ma
        kind = "reference"
        total_blocks_per_slice = ma.kernels[0].blocks[0][2]
        run = lambda nb: interpret_ma(_sliced_module(ma, nb), inp, DEFAULT_DEVICE, "fp32")
    else:
        from oracle import ma_interp
        from paper_2604_14825_b200 import ma_ir
        mod, _ = load_ma(cfg)
        inp = _cpu_inputs(mod)
        kind = "port"
        total_blocks_per_slice = mod.kernels[0].blocks[0][2]
        run = lambda nb: ma_interp.interpret_ma(_sliced_module(mod, nb), inp)
    t = time.perf_counter()
    run(1)
    per_block = time.perf_counter() - t
    nb = max(1, min(total_blocks_per_slice, int(target_s / max(per_block, 1e-3))))
    t = time.perf_counter()
    run(nb)
    dt = time.perf_counter() - t
    per_block = dt / nb
    slices = cpu_binding(cfg)[2]
    total_s = per_block * total_blocks_per_slice * slices
    return {"value": full_flops / total_s / 1e12, "unit": "TFLOP/s", "cores": 1, "kind": kind,
            "sample": f"{nb} of {total_blocks_per_slice} MA blocks of one (b,h) slice "
                      f"({dt:.1f} s), extrapolated x{total_blocks_per_slice * slices / nb:.0f} "
                      f"to {slices} slices = {total_s:.0f} s on 1 core",
            "seconds_full_workload": total_s}


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's CPU tile executor on all host cores."""
    import multiprocessing as mp
    if rank != 0:
        return
    ma = reference_module(cfg)
    flops = attention_flops(cfg)
    if ma is None:
        kind = "port"
        mod, _ = load_ma(cfg)
    else:
        kind = "reference"
    inp = _cpu_inputs(ma if ma is not None else mod)
    cores = os.cpu_count() or 1
    total_blocks = (ma.kernels[0].blocks[0][2] if ma is not None else mod.kernels[0].blocks[0][2])
    _POOL_STATE["ma"] = ma if ma is not None else mod
    _POOL_STATE["inp"] = inp
    worker = _port_worker if kind == "port" else _ref_worker
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores) as pool:
        for step in range(args.warmup + args.steps):
            t = time.perf_counter()
            pool.map(worker, [1] * cores)
            dt = time.perf_counter() - t
            if step >= args.warmup:
                times.append(dt)
    step_s = statistics.mean(times)
    blocks_total = total_blocks * cpu_binding(cfg)[2]
    full_s = step_s * blocks_total / cores
    value = flops / full_s / 1e12
    out = {"metric": METRIC, "value": value,
           "unit": "TFLOP/s", "impl": "reference", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
           "config": config_block(cfg, args, world),
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                            "sample": f"each step: {cores} processes x 1 MA block of the "
                                      f"{args.config} slice program; extrapolated to {blocks_total} blocks "
                                      f"({full_s:.0f} s for the full workload)"},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def attention_flops(cfg):
    B, Hq, N, D = cfg["B"], cfg["Hq"], cfg["N"], cfg["D"]
    M = cfg.get("M", N)
    if cfg.get("kind") == "gemm_chain":
        return 2.0 * cfg["N"] * cfg["F"] * (cfg["K"] + cfg["E"])
    if cfg["causal"]:
        return 2.0 * B * Hq * D * N * (N + 1)
    return 4.0 * B * Hq * N * M * D  # (masked configs: dense-equivalent, every pair is computed)


def config_block(cfg, args, world):
    """The workload keys only (identical in both arms); ``world`` = ranks that actually ran."""
    blk = {"workload": args.config}
    blk.update({k: v for k, v in cfg.items() if k not in ("golden",)})
    if world == 1:
        blk["parallelism"] = "single GPU"
    else:
        blk["parallelism"] = (f"row-block sharding over {world} GPUs" if cfg.get("kind") == "gemm_chain"
                              else f"(batch, kv-head) group sharding over {world} GPUs")
    blk["l2"] = "flushed between timed steps (256 MiB write)"
    return blk


def cpu_binding(cfg):
    """(binding, device overrides, number of MA slices in the full workload) of the CPU baseline."""
    kind = cfg.get("kind", "prefill")
    if kind == "gemm_chain":
        dev = {"max_tile_elems": 1000000} if cfg["E"] > 128 else {}
        return dict(N=cfg["N"], K=cfg["K"], F=cfg["F"], E=cfg["E"]), dev, 1
    if kind == "decode":
        g = cfg["Hq"] // cfg["Hkv"]
        return dict(N=g * cfg["N"], M=cfg["M"], D=cfg["D"]), {}, cfg["B"] * cfg["Hkv"]
    return dict(N=cfg["N"], M=cfg.get("M", cfg["N"]), D=cfg["D"]), {}, cfg["B"] * cfg["Hq"]


def shard(cfg, rank, world):
    """(b0, b1, h0, h1) kv-group range of this rank (paper_2604_14825_b200.shard.plan_shard)."""
    from paper_2604_14825_b200.shard import plan_shard
    sh = plan_shard(cfg["B"], cfg["Hkv"], world, rank)
    return sh.b0, sh.b1, sh.h0, sh.h1


def build_workload(cfg, spec, rank, world, dev):
    """Device tensors + launch plan for this rank's shard of the configured workload."""
    import torch
    from paper_2604_14825_b200.gemm import ChainPlan
    from paper_2604_14825_b200.runtime import AttentionPlan, DecodePlan

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    kind = cfg.get("kind", "prefill")
    w = {"kind": kind}
    if kind == "gemm_chain":
        from paper_2604_14825_b200.shard import plan_row_shard
        N, K, F, E = cfg["N"], cfg["K"], cfg["F"], cfg["E"]
        rs = plan_row_shard(N, world, rank)
        rows = rs.r1 - rs.r0
        x = torch.randn((rows, K), generator=gen, device=dev).to(torch.bfloat16)
        w1 = (torch.randn((K, F), generator=gen, device=dev) / K ** 0.5).to(torch.bfloat16)
        w2 = (torch.randn((F, E), generator=gen, device=dev) / F ** 0.5).to(torch.bfloat16)
        y = torch.empty((rows, E), dtype=torch.bfloat16, device=dev)
        w.update(plan=ChainPlan(x, w1, w2, y), out=y, local_flops=2.0 * rows * F * (K + E),
                 total_flops=2.0 * N * F * (K + E), bound="tensor",
                 host_inputs={spec.x: x, spec.w1: w1, spec.w2: w2}, outer=None, mask_kind=None,
                 in_bytes=(x.numel() + w1.numel() + w2.numel()) * 2, rows=N)
        return w
    b0, b1, h0, h1 = shard(cfg, rank, world)
    g = cfg["Hq"] // cfg["Hkv"]
    Bl, Hkvl = b1 - b0, h1 - h0
    N, D = cfg["N"], cfg["D"]
    M = cfg.get("M", N)
    if kind == "decode":
        # the MA's rows are the g q-heads of one kv group: Q [B, Hkv, g, D]
        q = torch.randn((Bl, Hkvl, g * N, D), generator=gen, device=dev).to(torch.bfloat16)
        k = torch.randn((Bl, Hkvl, M, D), generator=gen, device=dev).to(torch.bfloat16)
        v = torch.randn((Bl, Hkvl, M, D), generator=gen, device=dev).to(torch.bfloat16)
        o = torch.empty((Bl, Hkvl, g * N, D), dtype=torch.bfloat16, device=dev)
        esz, kw = 2, {}
        host_inputs = {spec.q: q, spec.k: k, spec.v: v}
        if cfg.get("in_dtype") == "e4m3":
            # per-tensor e4m3 quantisation (descale = amax / 448) of the same q/k/v: an FP8 KV cache
            ts, ds = [], []
            for t in (q, k, v):
                d = float(t.abs().max().float()) / 448.0
                ts.append((t.float() / d).to(torch.float8_e4m3fn))
                ds.append(d)
            q, k, v = ts
            del ts
            kw = dict(q_descale=ds[0], k_descale=ds[1], v_descale=ds[2])
            host_inputs = {"q": q, "k": k, "v": v}
            esz = 1
            w["e4m3"] = True
        plan = DecodePlan(q, k, v, o, spec.scale, **kw)
        if cfg.get("page_size"):
            # NHD page pools [pages, page_size, Hkv, D] in a shuffled physical order
            from paper_2604_14825_b200.runtime import PagedDecodePlan
            ps = cfg["page_size"]
            npp = M // ps
            perm = torch.randperm(Bl * npp, generator=gen, device=dev).to(torch.int32)
            layout = cfg.get("page_layout", "NHD")
            pools = []
            for t in (k, v):
                # scatter as raw bytes / bf16 (index_put has no float8 kernel)
                tb = t.view(torch.uint8) if esz == 1 else t
                if layout == "NHD":
                    pool = torch.empty((Bl * npp, ps, Hkvl, D), dtype=tb.dtype, device=dev)
                    pool[perm.long()] = tb.permute(0, 2, 1, 3).reshape(Bl * npp, ps, Hkvl, D)
                else:
                    pool = torch.empty((Bl * npp, Hkvl, ps, D), dtype=tb.dtype, device=dev)
                    pool[perm.long()] = tb.reshape(Bl, Hkvl, npp, ps, D).permute(0, 2, 1, 3, 4).reshape(
                        Bl * npp, Hkvl, ps, D)
                pools.append(pool.view(t.dtype))
            block_table = perm.reshape(Bl, npp).contiguous()
            seq_lens = torch.full((Bl,), M, dtype=torch.int32, device=dev)
            plan = PagedDecodePlan(q, pools[0], pools[1], block_table, seq_lens, o, spec.scale, layout=layout,
                                   max_seq_kv=M, **kw)
            w["pools"] = pools
            if esz == 1:  # e2e: the e4m3 page pools are what a serving runtime ships
                host_inputs = {"q": q, "k": pools[0], "v": pools[1]}
        kv_bytes = 2 * Bl * Hkvl * M * D * esz
        # O is written in bf16 (2 bytes) whatever the input type
        w.update(plan=plan, out=o, local_flops=4.0 * Bl * Hkvl * g * N * M * D,
                 total_flops=4.0 * cfg["B"] * cfg["Hq"] * N * M * D, bound="hbm",
                 local_bytes=kv_bytes + q.numel() * esz + o.numel() * 2, host_inputs=host_inputs,
                 outer=(Bl, Hkvl, Hkvl), mask_kind="none",
                 in_bytes=(q.numel() + k.numel() + v.numel()) * esz)
        return w
    Hql = Hkvl * g
    q = torch.randn((Bl, Hql, N, D), generator=gen, device=dev).to(torch.bfloat16)
    k = torch.randn((Bl, Hkvl, M, D), generator=gen, device=dev).to(torch.bfloat16)
    v = torch.randn((Bl, Hkvl, M, D), generator=gen, device=dev).to(torch.bfloat16)
    o = torch.empty((Bl, Hql, N, D), dtype=torch.bfloat16, device=dev)
    mask_kind = "causal" if cfg["causal"] else "none"
    if cfg.get("in_dtype") == "e4m3":
        # per-tensor e4m3 quantisation (descale = amax / 448); e2e goes through the
        # AttentionPlan / nt_attn_fwd call with host e4m3 buffers (the MA has no fp8)
        q8, k8, v8, ds = [], [], [], []
        for t, lst in ((q, q8), (k, k8), (v, v8)):
            d = float(t.float().abs().max()) / 448.0
            lst.append((t.float() / d).to(torch.float8_e4m3fn))
            ds.append(d)
        q, k, v = q8[0], k8[0], v8[0]
        plan = AttentionPlan(q, k, v, o, spec.scale, mask_kind, q_descale=ds[0], k_descale=ds[1], v_descale=ds[2])
        w.update(plan=plan, out=o, local_flops=plan.flops(), total_flops=attention_flops(cfg), bound="tensor",
                 host_inputs={"q": q, "k": k, "v": v}, outer=None, mask_kind=mask_kind, e4m3=True,
                 in_bytes=q.numel() + k.numel() + v.numel())
        return w
    mask_t = None
    if cfg.get("mask"):
        # dense-equivalent FLOPs (every (query, key) pair is computed; masked ones exp to 0)
        from paper_2604_14825_b200.runtime import pack_mask_bits
        gm = torch.Generator(device=dev)
        gm.manual_seed(99)
        mf = torch.where(torch.rand((N, M), generator=gm, device=dev) < 0.5, float("-inf"), 0.0)
        mf[:, 0] = 0.0
        mask_kind = cfg["mask"]
        mask_t = pack_mask_bits(mf)[0] if mask_kind == "bits" else mf
        w["mask_f32"] = mf
    plan = AttentionPlan(q, k, v, o, spec.scale, mask_kind, mask_t, item_rows=cfg.get("item_rows", 0))
    host_inputs = {spec.q: q, spec.k: k, spec.v: v}
    in_bytes = (q.numel() + k.numel() + v.numel()) * 2
    if cfg.get("mask"):
        host_inputs[spec.mask] = w["mask_f32"]  # the MA's fp32 Mask input, packed on the device per call
        in_bytes += w["mask_f32"].numel() * 4
    w.update(plan=plan, out=o, local_flops=plan.flops(), total_flops=attention_flops(cfg), bound="tensor",
             host_inputs=host_inputs, outer=(Bl, Hql, Hkvl), mask_kind=mask_kind, in_bytes=in_bytes)
    return w


def run_ours(args, cfg, rank, world, dist):
    import torch
    from paper_2604_14825_b200 import _lib, execute_ma
    from paper_2604_14825_b200.recognize import recognize

    dev = torch.device("cuda", torch.cuda.current_device())
    mod, ma_src = load_ma(cfg)
    spec = recognize(mod)[0]
    w = build_workload(cfg, spec, rank, world, dev)
    plan, o = w["plan"], w["out"]
    full = torch.empty((world,) + tuple(o.shape), dtype=o.dtype, device=dev) if world > 1 else None
    if world > 1 and w["kind"] == "gemm_chain":
        from paper_2604_14825_b200.shard import gather_rows

        def gather():
            gather_rows(o, w["rows"], world, dist)
    elif world > 1:
        def gather():
            dist.all_gather_into_tensor(full, o)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        flush.zero_()
        plan.launch(stream)
        if world > 1:
            gather()
    torch.cuda.synchronize()
    if hasattr(plan, "check_errors") and not os.environ.get("NT_BENCH_NOCHECK"):
        plan.check_errors()
    launch = plan.launch
    if cfg.get("graph") and world == 1:
        # one CUDA graph of the plan's launch (the persistent kernel's work counter resets
        # itself, so replays are independent); each timed step is one replay
        graph = torch.cuda.CUDAGraph()
        c0 = _lib.launch_count()
        with torch.cuda.graph(graph):
            plan.launch(torch.cuda.current_stream())
        graph_kernels = _lib.launch_count() - c0  # our kernels per replay
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()

        def launch(_stream):
            graph.replay()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            launch(stream)
            ev[i][1].record(stream)
            if world > 1:
                # the step adds the all-gather; one process has nothing to add (a third
                # back-to-back event record alone measured ~2.5 us on the device timeline)
                gather()
                ev[i][2].record(stream)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - l0
    if cfg.get("graph") and world == 1:
        launches = graph_kernels * args.steps  # replays do not pass through the library's counter
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kern_ms = [a.elapsed_time(b) for a, b, _ in ev]
    step_ms = [a.elapsed_time(c) for a, _, c in ev] if world > 1 else kern_ms
    ms_kernel_local = statistics.mean(kern_ms)
    ms_kernel, ms_step = ms_kernel_local, statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms_step, ms_kernel], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, ms_kernel = float(t[0]), float(t[1])
    ms_compute = ms_kernel  # max over ranks of the kernel-only time (no gather)
    total_flops = w["total_flops"]
    value = total_flops / (ms_step * 1e-3) / 1e12
    peaks, peak_src = load_peaks()
    clocks = clk.summary()

    # ---------------- e2e through the public API (pinned host in, host out)
    e2e = None if (cfg.get("no_e2e") or args.no_e2e) else measure_e2e(args, cfg, w, plan, o, mod, stream, flush, world, dist,
                                                     total_flops)
    if rank != 0:
        return
    emit(args, cfg, w, plan, world, ma_src, ms_step, ms_kernel, ms_kernel_local, ms_compute, total_flops, value,
         peaks, peak_src, clocks, launches, e2e)


def measure_e2e(args, cfg, w, plan, o, mod, stream, flush, world, dist, total_flops):
    """The same metric through the public API with pinned host buffers (H2D + kernel + D2H timed)."""
    import torch
    from paper_2604_14825_b200 import execute_ma

    host_in = {n: t.cpu().pin_memory() for n, t in w["host_inputs"].items()}
    host_out = torch.empty(tuple(o.shape), dtype=o.dtype).pin_memory()

    dev_in = w["host_inputs"]

    def e2e_step():
        if w.get("e4m3"):
            # host e4m3 q/k/v -> device, one nt_attn_fwd, O -> host (no fp8 MA precision)
            for n, t in host_in.items():
                dev_in[n].copy_(t, non_blocking=True)
            plan.launch(stream)
            host_out.copy_(o, non_blocking=True)
            return
        # host q/k/v in, host O out: execute_ma streams the (batch, kv-head) groups
        # (H2D, kernel and D2H of consecutive chunks overlap on three streams)
        execute_ma(mod, host_in, outer=w["outer"], mask_kind=w["mask_kind"], out_dtype="bf16",
                   return_torch=True, out=host_out)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        e1.synchronize()
        e_ms.append(e0.elapsed_time(e1))
    em = statistics.mean(e_ms)
    if world > 1:
        t = torch.tensor([em], device=o.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        em = float(t[0])
    e2e = {"value": total_flops / (em * 1e-3) / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": int(w["in_bytes"] * world), "d2h_bytes_per_step": int(o.numel() * 2 * world),
           "ms_per_step": em, "api": ("PagedDecodePlan / nt_attn_decode_paged (pinned host e4m3 q + page pools -> "
                                      "device, O -> pinned host)"
                                      if w.get("e4m3") and cfg.get("page_size") else
                                      "DecodePlan / nt_attn_decode (pinned host e4m3 q/k/v -> device, O -> pinned host)"
                                     if w.get("e4m3") and w["kind"] == "decode" else
                                     "AttentionPlan / nt_attn_fwd (pinned host e4m3 q/k/v -> device, O -> pinned host)"
                                     if w.get("e4m3") else
                                     "paper_2604_14825_b200.execute_ma(pinned host q/k/v, out=pinned host O): chunked H2D/kernel/D2H streams")}

    return e2e


def emit(args, cfg, w, plan, world, ma_src, ms_step, ms_kernel, ms_kernel_local, ms_compute, total_flops, value,
         peaks, peak_src, clocks, launches, e2e):
    """Rank 0's JSON line."""
    traffic = None
    prof = os.path.join(REPO, "profiles", f"latest_{args.config}_ncu.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    if w["bound"] == "hbm":
        achieved = w["local_bytes"] / (ms_kernel_local * 1e-3) / 1e9
        peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src}; a copy: read + write)",
                # the decode stream only reads: its ceiling is the TMA read rate, measured with
                # tools/ubench/bulk_read.cu on this pool's B200 (r02: 7398 GB/s, 192 KB in flight per SM)
                "read_ceiling_gbs": READ_CEILING_GBS, "frac_of_read_ceiling": achieved / READ_CEILING_GBS,
                "algorithmic_bytes_per_launch": w["local_bytes"],
                "kernel": ("decode_tc_kernel" + ("<paged" if cfg.get("page_size") else "<dense")
                           + (", e4m3> (tcgen05 kind::f8f6f4 dots" if w.get("e4m3") else "> (tcgen05 kind::f16 dots")
                           + (", page-slice TMA gathers) + combine" if cfg.get("page_size") else ") + combine"))}
    else:
        achieved = w["local_flops"] / (ms_kernel_local * 1e-3) / 1e12
        peak = peaks["bf16_tflops"] * (2.0 if w.get("e4m3") else 1.0)
        psrc = (f"2 x MEASURED_PEAKS.json bf16_tflops (fp8 dense = 2x bf16; no measured fp8 peak; {peak_src})"
                if w.get("e4m3") else f"MEASURED_PEAKS.json bf16_tflops (burst; {peak_src})")
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": psrc,
                "algorithmic_flops_per_launch": w["local_flops"],
                "kernel": {"prefill": "attn_fwd_kernel", "gemm_chain": getattr(plan, "realisation", "gemm")}[w["kind"]]}
    peak_t = peaks["bf16_tflops"]
    out = {
        "metric": METRIC,
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "e4m3" if w.get("e4m3") else "bf16", "data": "synthetic (torch.randn, seeded)",
        "config": config_block(cfg, args, world),
        "ma_source": ma_src, "kernel_ms": ms_kernel,
        "k1_item_rows": getattr(plan, "item_rows", None), "k1_ctas_per_sm": getattr(plan, "ctas_per_sm", None),
        "ms_per_step_compute_only": ms_compute, "ms_per_step_with_gather": ms_step,
        "pct_of_peak": {"measured_burst": value / peak_t,
                        "measured_sustained": value / peaks.get("bf16_tflops_sustained", peak_t),
                        "nominal_2250": value / 2250.0, "peak_source": peak_src},
        "roofline": roof,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": launches,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(cfg, total_flops, args.cpu_seconds)
        except Exception as ex:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "error": repr(ex)}
    print(json.dumps(out), flush=True)


def spawn_ranks(n):
    """``bench.py --gpus N`` outside torchrun: launch N ranks (one per GPU, NCCL) the way
    the driver does and return rank 0's exit status; rank 0 prints the JSON line.
    NCCL's init log (transport, NVLS/NVLink choice) goes to stderr."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (A/B runs)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--item-rows", type=int, default=0, choices=[0, 128, 256],
                    help="K1 query rows per work item (0 = library choice)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.item_rows:
        cfg = dict(cfg, item_rows=args.item_rows)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    args.gpus = world if world > 1 else args.gpus
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    run_ours(args, cfg, rank, world, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
