"""Static counters of the reference cost model and a B200 viability check.

* ``cost_model`` restates tilecc/ma/cost.py:66-104 (closed-form bytes per
  scope, weighted flops via ``expr_flops`` tilecc/ma/cost.py:30-52, steps) and
  ``modeled_cost`` tilecc/ma/interp.py:86-99, so ``ExecReport`` carries the
  same static numbers the reference ``CostReport`` does.
* ``DeviceProfile`` mirrors ``VirtualDevice`` (tilecc/ma/device.py:17-49) with
  the reference's default values; ``B200`` describes the real part.
* ``b200_viable`` replaces ``check_capacity`` (tilecc/ma/cost.py:107-173),
  whose fp32-sized model rejects tiles that fit the bf16/TMEM realisation
  (SURVEY.md B.6, B.11).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import ma_ir as ir

ITEM_BYTES = {"fp32": 4, "fp64": 8, "rational": 8}
FLOP_WEIGHTS = {"add": 1, "sub": 1, "mul": 1, "div": 4, "max": 1, "min": 1,
                "exp": 8, "exp2": 4, "log2": 4, "neg": 1, "scale": 1}


@dataclass(frozen=True)
class DeviceProfile:
    name: str = "virtual-h100"
    shared_bytes: int = 228 * 1024
    register_bytes: int = 256 * 1024
    cost_global: float = 100.0
    cost_shared: float = 10.0
    cost_register: float = 1.0
    cost_flop: float = 0.25
    launch_cost: float = 10000.0
    warp_default: int = 4
    stage_default: int = 2
    stage_discount: float = 0.15
    backend_factors: tuple = (("generic", (1.0, 1.0)), ("triton-like", (1.0, 0.95)),
                              ("tilelang-like", (0.95, 1.0)))

    def factors(self, backend):
        for n, f in self.backend_factors:
            if n == backend:
                return f
        return (1.0, 1.0)


DEFAULT = DeviceProfile()

_INT_KEYS = {"shared_bytes", "register_bytes", "warp_default", "stage_default"}
_IGNORED_INT_KEYS = {"inner_cap", "max_tile_elems", "stage_min", "stage_max"}  # scheduler-only
_FLOAT_KEYS = {"cost_global", "cost_shared", "cost_register", "cost_flop", "launch_cost", "stage_discount"}


def parse_profile(text: str) -> DeviceProfile:
    """``key = value`` device profile -> DeviceProfile (restates parse_device,
    tilecc/ma/device.py:59-95, for the fields the cost model reads; the
    scheduler-only keys are accepted and ignored).  Unknown keys raise."""
    from dataclasses import replace

    dev = DEFAULT
    factors = dict(dev.backend_factors)
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"device profile line {lineno}: expected key = value")
        key, _, val = (x.strip() for x in line.partition("="))
        if key in _INT_KEYS:
            dev = replace(dev, **{key: int(val)})
        elif key in _FLOAT_KEYS:
            dev = replace(dev, **{key: float(val)})
        elif key in _IGNORED_INT_KEYS:
            int(val)
        elif key == "warp_choices":
            tuple(int(x) for x in val.split(","))
        elif key == "name":
            dev = replace(dev, name=val)
        elif key.startswith("backend.") and key.endswith((".byte_factor", ".flop_factor")):
            b = key.split(".")[1]
            bf, ff = factors.get(b, (1.0, 1.0))
            factors[b] = (float(val), ff) if key.endswith(".byte_factor") else (bf, float(val))
        else:
            raise ValueError(f"device profile line {lineno}: unknown key {key!r}")
    return replace(dev, backend_factors=tuple(sorted(factors.items())))


def b200_profile() -> DeviceProfile:
    """The B200 profile (``b200.device``, also what ``frontdoor.b200_device`` feeds the scheduler)."""
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "b200.device")) as f:
        return parse_profile(f.read())


@dataclass(frozen=True)
class B200:
    sms: int = 148
    smem_per_cta: int = 227 * 1024
    tmem_cols: int = 512
    tmem_lanes: int = 128


@dataclass
class StaticCost:
    bytes_global: int = 0
    bytes_shared: int = 0
    bytes_register: int = 0
    flops: int = 0
    kernels: int = 0
    steps: int = 0
    modeled_cost: float = 0.0

    def add(self, scope, n):
        if scope == "Global":
            self.bytes_global += n
        elif scope == "Shared":
            self.bytes_shared += n
        else:
            self.bytes_register += n


def expr_flops(e: ir.Expr) -> int:
    total = 0
    for n in e.walk():
        size = 1
        for d in n.shape:
            size *= d
        if isinstance(n, (ir.Bin, ir.Un)):
            total += size * FLOP_WEIGHTS[n.op]
        elif isinstance(n, ir.Scale):
            total += size * FLOP_WEIGHTS["scale"]
        elif isinstance(n, ir.Dot):
            m, k = n.a.shape
            total += 2 * m * k * n.b.shape[1]
        elif isinstance(n, ir.Reduce):
            sz = 1
            for d in n.x.shape:
                sz *= d
            total += sz
    return total


def modeled_cost(rep: StaticCost, dev: DeviceProfile, backend: str, warps: int, stages: int) -> float:
    byte_f, flop_f = dev.factors(backend)
    wg = dev.cost_global / (1.0 + dev.stage_discount * (stages - 1))
    c = (rep.bytes_global * wg + rep.bytes_shared * dev.cost_shared +
         rep.bytes_register * dev.cost_register) * byte_f
    c += rep.flops * dev.cost_flop * (4.0 / warps) ** 0.5 * flop_f
    c += rep.kernels * dev.launch_cost
    return c


def cost_model(module, dev: DeviceProfile = DEFAULT) -> StaticCost:
    module = ir.as_module(module)
    item = ITEM_BYTES[module.precision]
    scope_of = {b.name: b.scope for b in module.buffers}
    rep = StaticCost(kernels=len(module.kernels))

    def walk(body, mult):
        for st in body:
            if isinstance(st, ir.Loop):
                rep.steps += mult * st.extent
                walk(st.body, mult * st.extent)
                continue
            rep.steps += mult
            if isinstance(st, ir.Copy):
                size = 1
                for s in st.src_slices:
                    size *= s.length
                rep.add(scope_of[st.src], mult * size * item)
                rep.add(scope_of[st.dst], mult * size * item)
                continue
            dsize = 1
            for s in st.dst_slices:
                dsize *= s.length
            rep.add(scope_of[st.dst], mult * dsize * item)
            for n in st.expr.walk():
                if isinstance(n, ir.Ref):
                    size = 1
                    for s in n.slices:
                        size *= s.length
                    rep.add(scope_of[n.buffer], mult * size * item)
            rep.flops += mult * expr_flops(st.expr)

    for k in module.kernels:
        mult = 1
        for _, _, e in k.blocks:
            mult *= e
        walk(k.body, mult)
    k0 = module.kernels[0] if module.kernels else None
    warps = k0.param("warps", dev.warp_default) if k0 else dev.warp_default
    stages = k0.param("stages", dev.stage_default) if k0 else dev.stage_default
    backend = k0.backend if k0 else "generic"
    rep.modeled_cost = modeled_cost(rep, dev, backend, warps, stages)
    return rep


def b200_viable(spec) -> list[str]:
    """Problems preventing the sm_100a realisation of a recognised spec (empty = viable)."""
    from .recognize import AttentionSpec, GemmChainSpec

    out = []
    if isinstance(spec, AttentionSpec):
        if spec.d not in (64, 128):
            out.append(f"head dim {spec.d} not in (64, 128)")
        if spec.scale is not None and not spec.scale > 0:
            out.append("scale must be positive")
    elif isinstance(spec, GemmChainSpec):
        for nm, v in (("K", spec.k), ("F", spec.f), ("E", spec.e)):
            if v % 8:
                out.append(f"{nm}={v} must be a multiple of 8 (16-byte TMA rows)")
    return out


def access_audit(module) -> tuple[int, dict]:
    """``unique_global_bytes`` and ``read_audit`` of interpret_ma's CostReport, without executing.

    Restates the access accounting of tilecc/ma/interp.py:128-141 and 160-171:
    every Global slice a kernel reads or writes is stamped into a per-kernel
    counter of the buffer's shape (unique bytes = touched elements x item
    size, summed over kernels), and the Global slices each block point reads
    are counted per block (``reads``, ``unique``, ``blocks``, ``single_pass``).
    Like the reference it allocates full-buffer counters, so it is computed
    only when asked for (``ExecReport.read_audit``).
    """
    import itertools

    import numpy as np

    module = ir.as_module(module)
    item = ITEM_BYTES[module.precision]
    shape = {b.name: tuple(b.shape) for b in module.buffers if b.scope == "Global"}
    unique = 0
    audit: dict = {}

    def accesses(body, loops=()):
        for st in body:
            if isinstance(st, ir.Loop):
                yield from accesses(st.body, loops + ((st.var, st.extent),))
            elif isinstance(st, ir.Copy):
                yield st.src, st.src_slices, loops, True
                yield st.dst, st.dst_slices, loops, False
            else:
                for n in st.expr.walk():
                    if isinstance(n, ir.Ref):
                        yield n.buffer, n.slices, loops, True
                yield st.dst, st.dst_slices, loops, False

    for k in module.kernels:
        acc = [a for a in accesses(k.body) if a[0] in shape]
        touched: dict = {}
        names = [v for v, _, _ in k.blocks]
        for point in itertools.product(*[range(e) for _, _, e in k.blocks]):
            benv = dict(zip(names, point))
            reads: dict = {}
            for buf, slices, loops, is_read in acc:
                lnames = [v for v, _ in loops]
                for lp in itertools.product(*[range(e) for _, e in loops]):
                    env = dict(benv, **dict(zip(lnames, lp)))
                    idx = tuple(slice(s.off.evaluate(env), s.off.evaluate(env) + s.length) for s in slices)
                    if buf not in touched:
                        touched[buf] = np.zeros(shape[buf], dtype=np.int32)
                    touched[buf][idx] += 1
                    if is_read:
                        if buf not in reads:
                            reads[buf] = np.zeros(shape[buf], dtype=np.int32)
                        reads[buf][idx] += 1
            for buf, counts in reads.items():
                a = audit.setdefault(buf, {"reads": 0, "unique": 0, "blocks": 0, "single_pass": True})
                total, uniq = int(counts.sum()), int((counts > 0).sum())
                a["reads"] += total
                a["unique"] += uniq
                a["blocks"] += 1
                if total != uniq:
                    a["single_pass"] = False
        for mask in touched.values():
            unique += int((mask > 0).sum()) * item
    return unique, {b: audit[b] for b in sorted(audit)}
