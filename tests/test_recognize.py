"""MA -> KernelSpec recognition, index-math parity and static-cost parity (CPU)."""

import json
import os

import pytest

from conftest import GOLDEN, all_ma_files
from paper_2604_14825_b200 import cost, ma_ir
from paper_2604_14825_b200.errors import UnsupportedMA
from paper_2604_14825_b200.recognize import AttentionSpec, GemmChainSpec, recognize


def _load(fname):
    with open(os.path.join(GOLDEN, fname)) as f:
        return ma_ir.from_json(f.read())


@pytest.mark.parametrize("fname", all_ma_files())
def test_every_golden_kernel_is_recognised(fname):
    mod = _load(fname)
    specs = recognize(mod)
    assert len(specs) == 1
    spec = specs[0]
    if fname.startswith(("gemm", "b200_gemm")):
        assert isinstance(spec, GemmChainSpec)
        assert spec.n_blocks * spec.block_m == spec.n
        assert spec.n_iters * spec.block_f == spec.f
    else:
        assert isinstance(spec, AttentionSpec)
        assert spec.n_blocks * spec.block_m == spec.n
        assert spec.n_iters * spec.block_n == spec.m
        txt = open(os.path.join(GOLDEN, fname.replace(".ma.json", ".ma.txt"))).read()
        if "0.125" in txt:
            assert spec.scale == 0.125
        elif "0.0883883" in txt:
            assert spec.scale == 0.08838834764831845
        else:
            assert spec.scale is None
        assert (spec.mask is not None) == ("Mask" in txt)


@pytest.mark.parametrize("fname", all_ma_files())
def test_static_cost_matches_reference_cost_model(fname):
    mod = _load(fname)
    # b200_* goldens were scheduled under paper_2604_14825_b200/b200.device
    mine = cost.cost_model(mod, cost.b200_profile() if fname.startswith("b200_") else cost.DEFAULT)
    with open(os.path.join(GOLDEN, fname.replace(".ma.json", ".cost.json"))) as f:
        ref = json.load(f)
    assert mine.bytes_global == ref["bytes"]["Global"]
    assert mine.bytes_shared == ref["bytes"]["Shared"]
    assert mine.bytes_register == ref["bytes"]["Register"]
    assert mine.flops == ref["flops"]
    assert mine.steps == ref["steps"]
    assert round(mine.modeled_cost, 6) == ref["modeled_cost"]


def _ma_slices(mod):
    """Evaluate every slice offset of the MA kernel at every (block, loop) point."""
    k = mod.kernels[0]
    (bvar, _, nb), = k.blocks
    loop = [s for s in k.body if isinstance(s, ma_ir.Loop)][0]
    out = []
    for i in range(nb):
        for j in range(loop.extent):
            env = {bvar: i, loop.var: j}
            for st in loop.body:
                exprs = [st.expr] if isinstance(st, ma_ir.Compute) else []
                for e in exprs:
                    for n in e.walk():
                        if isinstance(n, ma_ir.Ref) and mod.buffer(n.buffer).is_input:
                            out.append((i, j, n.buffer, tuple((s.off.evaluate(env), s.length) for s in n.slices)))
                if isinstance(st, ma_ir.Copy) and mod.buffer(st.src).is_input:
                    out.append((i, j, st.src, tuple((s.off.evaluate(env), s.length) for s in st.src_slices)))
    return out


@pytest.mark.parametrize("fname", [f for f in all_ma_files() if "gemm" not in f
                                   and ("256" in f or "512" in f or "decode" in f)])
def test_attention_index_math_matches_gpu_tiling(fname):
    """Each GPU (CTA, kv-tile) is exactly the union of the MA (block, j0) tiles
    it covers, visited in the MA's ascending j0 order."""
    mod = _load(fname)
    spec = recognize(mod)[0]
    ma = _ma_slices(mod)
    k_rows = {}
    for i, j, buf, sl in ma:
        if buf == spec.k:
            k_rows.setdefault(j, set()).add(sl[0])
    q_rows = {}
    for st in mod.kernels[0].body:
        if isinstance(st, ma_ir.Copy) and st.src == spec.q:
            for i in range(spec.n_blocks):
                q_rows[i] = (st.src_slices[0].off.evaluate({spec.block_var: i}), st.src_slices[0].length)
    seen_q, seen_k = set(), set()
    for cta, blocks, kv, iters in spec.gpu_tiles():
        rows = sorted(q_rows[b] for b in blocks)
        lo = cta * spec.gpu_bm
        hi = min(spec.n, lo + spec.gpu_bm)
        covered = sorted(r for o, l in rows for r in range(o, o + l))
        assert covered == list(range(lo, hi))
        assert iters == sorted(iters)
        kcov = sorted(r for t in iters for (o, l) in k_rows[t] for r in range(o, o + l))
        assert kcov == list(range(kv * 128, min(spec.m, kv * 128 + 128)))
        seen_q.update(blocks)
        seen_k.update(iters)
    assert seen_q == set(range(spec.n_blocks)) and seen_k == set(range(spec.n_iters))


def test_unrecognised_program_raises():
    mod = _load("attn256.seed0.ma.json")
    d = ma_ir.to_dict(mod)
    # corrupt: make the epilogue multiply instead of divide
    k = d["kernels"][0]
    k["body"][-2]["expr"]["op"] = "mul"
    with pytest.raises(UnsupportedMA):
        recognize(ma_ir.from_dict(d))


def test_precision_without_device_realisation_raises():
    mod = _load("attn256.seed0.ma.json")
    d = ma_ir.to_dict(mod)
    d["precision"] = "fp64"
    with pytest.raises(UnsupportedMA):
        recognize(ma_ir.from_dict(d))


@pytest.mark.parametrize("case", [c for c in __import__("conftest").io_cases()])
def test_access_audit_equals_reference_cost_report(case):
    """unique_global_bytes and read_audit of interpret_ma's CostReport, derived statically."""
    import json

    from conftest import golden_stem, load_golden
    from paper_2604_14825_b200 import cost

    mod, _, _, _ = load_golden(case)
    with open(golden_stem(case) + ".interp_cost.json") as f:
        ref = json.load(f)
    unique, audit = cost.access_audit(mod)
    assert unique == ref["unique_global_bytes"]
    assert audit == ref["read_audit"]


def test_b200_profile_parses_like_the_reference():
    """cost.parse_profile and the reference's parse_device read b200.device identically."""
    import dataclasses

    from paper_2604_14825_b200.frontdoor import B200_PROFILE, b200_device, import_tilecc
    try:
        import_tilecc()
    except ImportError:
        pytest.skip("reference front end not importable")
    ref = b200_device()
    mine = cost.b200_profile()
    for f in dataclasses.fields(mine):
        assert getattr(mine, f.name) == getattr(ref, f.name), f.name
    assert ref.inner_cap == 256 and ref.max_tile_elems >= 262144 and ref.warp_choices == (4, 8)
    assert "sm100a" in ref.backends()


def test_b200_profile_schedules_config2_e4096_without_overrides():
    """the default profile rejects the E=4096 chain; the B200 profile schedules it."""
    import json as _json
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        man = _json.load(f)
    e = man["b200_gemm4k_e4096"]
    assert e["profile"] == "b200" and e["device"] is None and e["n_seeds"] >= 1
    spec = recognize(_load("b200_gemm4k_e4096.seed0.ma.json"))[0]
    assert isinstance(spec, GemmChainSpec) and spec.e == 4096
    assert _load("b200_gemm4k_e4096.seed0.ma.json").kernels[0].backend == "sm100a"


def test_tile_tunables_select_distinct_realisations():
    """The MA's t0_i picks K1's work-item rows and `stages` its K/V ring: the device
    tuner sees distinct kernels for distinct tile choices (tuner.realisation_key)."""
    from dataclasses import replace as dc_replace

    from paper_2604_14825_b200.tuner import realisation_key

    spec = recognize(_load("attn256.seed0.ma.json"))[0]
    keys = set()
    for bm in (16, 32, 64, 128):
        for st in (1, 2, 3):
            keys.add(realisation_key(dc_replace(spec, block_m=bm, stages=st), None, "none"))
    assert len(keys) == 2  # one 256-row item -> always 128 rows here; {shallow, deep} ring at D=64
    # short D=64 KV ranges (<= 1024 keys) always take 128-row items (capi.cu
    # attn_item_rows); at 2048 keys the (4 x 32 x 8) items choose {128, 256} rows
    keys = {realisation_key(dc_replace(spec, block_m=bm, stages=st), (4, 32, 8), "none")
            for bm in (16, 32, 64, 128) for st in (1, 2, 3)}
    assert len(keys) == 2
    keys = {realisation_key(dc_replace(spec, block_m=bm, stages=st, n=2048, m=2048), (4, 32, 8), "none")
            for bm in (16, 32, 64, 128) for st in (1, 2, 3)}
    assert len(keys) == 4  # {128, 256} rows x {shallow, deep} ring
    assert recognize(_load("attn256_t32x64.seed0.ma.json"))[0].gpu_bm == 128
    assert recognize(_load("bert512.seed0.ma.json"))[0].gpu_bm == 128  # 2 items of 256 < 148 / 2


def test_item_rows_rule_matches_the_library():
    """recognize.attn_effective_rows restates csrc/capi.cu attn_item_rows: explicit 128 /
    256 win; head_dim 64 with <= 1024 keys -> 128; else 128 only when 256-row items
    would leave more than half of the SMs idle."""
    from paper_2604_14825_b200.recognize import attn_effective_rows

    assert attn_effective_rows(256, 512, 384, d=64, m=512) == 256
    assert attn_effective_rows(0, 512, 384, d=64, m=512) == 128      # BERT-base
    assert attn_effective_rows(0, 2048, 384, d=64, m=2048) == 256
    assert attn_effective_rows(0, 512, 384, d=128, m=512) == 256
    assert attn_effective_rows(0, 256, 1, d=128, m=256) == 128        # one item
    assert attn_effective_rows(0, 8192, 32, d=128, m=8192) == 256     # Llama 8K
