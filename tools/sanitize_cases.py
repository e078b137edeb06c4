"""Small launches of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck|synccheck|racecheck|initcheck \
        python tools/sanitize_cases.py [family ...]

Families: k1 (attn_fwd: masks none/causal/tensor, bf16/fp32 out, D=64/128,
split-KV units + combine, e4m3), k2 (decode split-KV dense + paged NHD/HND,
pages 16/64), k3 (gemm2 CTA pair, split-K gemm + reduce), chain (fused K3b),
simt (one SIMT-lowered corpus program).  Each case is checked against a
float64 reference of the same op so a sanitizer run is also a numerics run.
"""

import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import reference_math  # noqa: E402  (checker only)
from oracle.ma_interp import round_bf16  # noqa: E402

DEV = torch.device("cuda")


def nan_filled(shape, dtype, device):
    """Outputs start as NaN (written by a plain fill kernel): initcheck then sees
    initialised memory -- it does not track TMA (cp.async.bulk.tensor) stores, so a
    torch.empty output written only by TMA stores reads as uninitialised -- and the
    NaN-free check in close() proves every element was overwritten by the kernel."""
    return torch.full(shape, float("nan"), dtype=dtype, device=device)


def rnd(shape, seed, scale=1.0):
    return round_bf16(np.random.default_rng(seed).standard_normal(shape) * scale)


def close(got, ref, tol=2e-2, what=""):
    got = np.asarray(got, np.float64)
    err = float(np.max(np.abs(got - ref)))
    assert np.all(np.isfinite(got)) and err <= tol, (what, err)
    print(f"  {what}: max-abs {err:.2e}", flush=True)


def k1():
    from paper_2604_14825_b200.runtime import AttentionPlan

    cases = [  # B, Hq, Hkv, N, M, D, kind, out_f32
        (1, 2, 1, 300, 300, 128, "causal", True),
        (1, 2, 2, 256, 384, 64, "none", False),
        (1, 1, 1, 200, 256, 64, "tensor", True),
        (1, 1, 1, 129, 129, 128, "none", True),
        (1, 4, 1, 2048, 2048, 128, "causal", True),   # split-KV units + combine
        (1, 2, 2, 2048, 2048, 64, "none", False),       # split-KV D=64
        (1, 2, 1, 640, 700, 128, "bits", True),         # 0 / -inf mask as bits (128-row items)
        (4, 8, 8, 512, 512, 64, "bits", False),
    ]
    for B, Hq, Hkv, N, M, D, kind, f32 in cases:
        q, k, v = rnd((B, Hq, N, D), 1), rnd((B, Hkv, M, D), 2), rnd((B, Hkv, M, D), 3)
        mask = None
        if kind in ("tensor", "bits"):
            g = np.random.default_rng(4)
            mask = np.where(g.random((N, M)) < 0.3, -np.inf, 0.0).astype(np.float32)
            mask[:, 0] = 0.0
        tq, tk, tv = (torch.from_numpy(x).to(DEV).bfloat16() for x in (q, k, v))
        o = nan_filled((B, Hq, N, D), dtype=torch.float32 if f32 else torch.bfloat16, device=DEV)
        mt = torch.from_numpy(mask).to(DEV) if mask is not None else None
        if kind == "bits":
            from paper_2604_14825_b200.runtime import pack_mask_bits
            mt = pack_mask_bits(mt)[0]
        plan = AttentionPlan(tq, tk, tv, o, 1 / np.sqrt(D), kind, mt)
        plan.launch()
        torch.cuda.synchronize()
        plan.check_errors()
        if mask is not None:
            ref = np.stack([np.stack([reference_math.attention_fp64(q[b, h], k[b, h * Hkv // Hq], v[b, h * Hkv // Hq],
                                                                    1 / np.sqrt(D), mask=mask)
                                      for h in range(Hq)]) for b in range(B)])
        else:
            ref = reference_math.attention_batched_fp64(q, k, v, 1 / np.sqrt(D), kind == "causal")
        close(o.float().cpu().numpy(), ref,
              what=f"k1 {kind} D={D} N={N} rows={plan.item_rows} split={plan.ws is not None}")
    # e4m3
    B, Hq, Hkv, N, D = 1, 2, 1, 384, 128
    q, k, v = rnd((B, Hq, N, D), 5), rnd((B, Hkv, N, D), 6), rnd((B, Hkv, N, D), 7)
    tq, tk, tv = (torch.from_numpy(x).to(DEV).to(torch.float8_e4m3fn) for x in (q, k, v))
    deq = [t.float().cpu().numpy() for t in (tq, tk, tv)]
    o = nan_filled((B, Hq, N, D), dtype=torch.float32, device=DEV)
    plan = AttentionPlan(tq, tk, tv, o, 1 / np.sqrt(D), "causal")
    plan.launch()
    torch.cuda.synchronize()
    ref = reference_math.attention_batched_fp64(*deq, 1 / np.sqrt(D), True)
    close(o.cpu().numpy(), ref, tol=1e-1, what="k1 e4m3 causal")


def k2():
    from paper_2604_14825_b200.runtime import DecodePlan, PagedDecodePlan

    B, Hq, Hkv, D, M = 2, 8, 2, 128, 1500
    q, k, v = rnd((B, Hq, 1, D), 8), rnd((B, Hkv, M, D), 9), rnd((B, Hkv, M, D), 10)
    tq, tk, tv = (torch.from_numpy(x).to(DEV).bfloat16() for x in (q, k, v))
    o = nan_filled((B, Hq, 1, D), dtype=torch.float32, device=DEV)
    plan = DecodePlan(tq, tk, tv, o, 1 / np.sqrt(D), num_splits=3)
    plan.launch()
    torch.cuda.synchronize()
    ref = reference_math.attention_batched_fp64(q, k, v, 1 / np.sqrt(D), False)
    close(o.cpu().numpy(), ref, what="k2 dense")
    for ps, layout in ((16, "NHD"), (64, "HND")):
        npp = -(-M // ps)
        P = B * npp + 2
        perm = np.random.default_rng(ps).permutation(P)[: B * npp].reshape(B, npp)
        shape = (P, ps, Hkv, D) if layout == "NHD" else (P, Hkv, ps, D)
        kp = torch.zeros(shape, dtype=torch.bfloat16, device=DEV)
        vp = torch.zeros(shape, dtype=torch.bfloat16, device=DEV)
        for b in range(B):
            for j in range(npp):
                lo, hi = j * ps, min(M, (j + 1) * ps)
                kk = torch.from_numpy(k[b, :, lo:hi]).to(DEV).bfloat16()
                vv = torch.from_numpy(v[b, :, lo:hi]).to(DEV).bfloat16()
                if layout == "NHD":
                    kp[perm[b, j], : hi - lo] = kk.transpose(0, 1)
                    vp[perm[b, j], : hi - lo] = vv.transpose(0, 1)
                else:
                    kp[perm[b, j], :, : hi - lo] = kk
                    vp[perm[b, j], :, : hi - lo] = vv
        bt = torch.from_numpy(perm.astype(np.int32)).to(DEV)
        sl = torch.full((B,), M, dtype=torch.int32, device=DEV)
        o.zero_()
        plan = PagedDecodePlan(tq, kp, vp, bt, sl, o, 1 / np.sqrt(D), layout=layout, max_seq_kv=M)
        plan.launch()
        torch.cuda.synchronize()
        close(o.cpu().numpy(), ref, what=f"k2 paged {ps} {layout}")
    # FP8 (e4m3) cache, dense and 32-token pages, checked against fp64 of the dequantised inputs
    def q8(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        d = float(t.abs().max()) / 448.0
        t8 = (t / d).to(torch.float8_e4m3fn)
        return t8, d, (t8.float() * d).double().numpy()
    (q8_, qd, qf), (k8_, kd, kf), (v8_, vd, vf) = q8(q), q8(k), q8(v)
    ref8 = reference_math.attention_batched_fp64(qf, kf, vf, 1 / np.sqrt(D), False)
    o8 = nan_filled((B, Hq, 1, D), dtype=torch.float32, device=DEV)
    kw = dict(q_descale=qd, k_descale=kd, v_descale=vd)
    DecodePlan(q8_.to(DEV), k8_.to(DEV), v8_.to(DEV), o8, 1 / np.sqrt(D), num_splits=3, **kw).launch()
    torch.cuda.synchronize()
    close(o8.cpu().numpy(), ref8, tol=8e-2, what="k2 e4m3 dense")
    ps = 32
    npp = -(-M // ps)
    kp8 = torch.zeros((B * npp, ps, Hkv, D), dtype=torch.uint8, device=DEV)
    vp8 = torch.zeros_like(kp8)
    for b in range(B):
        for j in range(npp):
            lo, hi = j * ps, min(M, (j + 1) * ps)
            kp8[b * npp + j, : hi - lo] = k8_[b, :, lo:hi].view(torch.uint8).to(DEV).transpose(0, 1)
            vp8[b * npp + j, : hi - lo] = v8_[b, :, lo:hi].view(torch.uint8).to(DEV).transpose(0, 1)
    bt = torch.arange(B * npp, dtype=torch.int32, device=DEV).reshape(B, npp)
    o8.fill_(float("nan"))
    PagedDecodePlan(q8_.to(DEV), kp8.view(torch.float8_e4m3fn), vp8.view(torch.float8_e4m3fn), bt,
                    torch.full((B,), M, dtype=torch.int32, device=DEV), o8, 1 / np.sqrt(D), max_seq_kv=M,
                    **kw).launch()
    torch.cuda.synchronize()
    close(o8.cpu().numpy(), ref8, tol=8e-2, what="k2 e4m3 paged 32")


def k3():
    from paper_2604_14825_b200.gemm import GemmPlan

    for M, N, K, f32 in ((2048, 2048, 512, False), (256, 128, 2048, True)):
        a, b = rnd((M, K), 11), rnd((K, N), 12, 1 / np.sqrt(K))
        c = nan_filled((M, N), dtype=torch.float32 if f32 else torch.bfloat16, device=DEV)
        plan = GemmPlan(torch.from_numpy(a).to(DEV).bfloat16(), torch.from_numpy(b).to(DEV).bfloat16(), c)
        plan.launch()
        torch.cuda.synchronize()
        close(c.float().cpu().numpy(), a.astype(np.float64) @ b, what=f"k3 {M}x{N}x{K} splits={plan.args.k_splits}")


def chain():
    from paper_2604_14825_b200.gemm import ChainPlan

    N, K, F, E = 256, 256, 512, 128
    x, w1, w2 = rnd((N, K), 13), rnd((K, F), 14, 1 / 16), rnd((F, E), 15, 1 / np.sqrt(F))
    y = nan_filled((N, E), dtype=torch.float32, device=DEV)
    plan = ChainPlan(*(torch.from_numpy(t).to(DEV).bfloat16() for t in (x, w1, w2)), y)
    assert plan.fused
    plan.launch()
    torch.cuda.synchronize()
    close(y.cpu().numpy(), reference_math.gemm_chain_fp64(x, w1, w2), tol=5e-2, what="chain fused")


def simt():
    from paper_2604_14825_b200 import execute_ma
    from conftest_path import load_golden  # noqa: F401  (set up below)

    mod, inputs, interp32, _ = load_golden("attn256")
    bufs, _ = execute_ma(mod, inputs, backend="simt")
    close(bufs[mod.output], interp32, tol=1e-5, what="simt attn256 (fp32 lowering)")


FAMILIES = {"k1": k1, "k2": k2, "k3": k3, "chain": chain, "simt": simt}

if __name__ == "__main__":
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import conftest as conftest_path  # noqa: E402

    sys.modules["conftest_path"] = conftest_path
    for name in sys.argv[1:] or list(FAMILIES):
        print(name, flush=True)
        FAMILIES[name]()
    print("sanitize cases ok", flush=True)
