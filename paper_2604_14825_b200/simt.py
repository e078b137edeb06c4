"""Generic MA -> CUDA SIMT lowering.

The tcgen05 kernels (K1 attention, K2 decode, K3 GEMM / chain) realise the MA
families the auto-scheduler produces for the BASELINE workloads.  Every other
MA program -- the reference's element-wise chains, reductions, small matmuls,
softmax / broadcast / multi-use corpus families (tests/conftest.py:109-181 of
the reference), the ``selftest`` programs (tilecc/cli.py:247-298), fp64
programs -- is lowered here to CUDA C that follows ``interpret_ma``
(tilecc/ma/interp.py:102-280) statement by statement, compiled by nvcc for
sm_100a, cached by content hash and launched through the C ABI
(``nt_module_load`` / ``nt_launch``, include/nautilus_b200.h).

Semantics kept from the reference executor:

* one CUDA block per MA block point; block variables are decoded from the
  linear block index in ``itertools.product`` order (interp.py:121-127);
* every ``MACopy`` / ``MACompute`` (interp.py:187-211) is a CTA-wide pass over
  the destination tile followed by ``__syncthreads()``; the value of
  destination element ``f`` is expression element ``f`` in C order (the
  ``reshape`` at interp.py:198, 211); a statement that reads its own
  destination at other positions evaluates into a staging tile first (the
  reference evaluates the whole right-hand side before storing);
* ``MALoop`` is a sequential C loop (interp.py:178-186);
* ``VDot`` is the sequential rank-1 k loop ``acc = acc + a[:, k] * b[k, :]``
  (interp.py:241-251) and ``VReduce`` the seeded sequential fold over the
  reduced axes in their listed order (interp.py:252-271).  The code is
  compiled with ``--fmad=false``, so each product and sum is rounded exactly
  like numpy's: for programs without exp / exp2 / log2 the fp32 and fp64
  results are bit-identical to the reference; the transcendental functions
  are CUDA's (<= 2 ulp), not numpy's;
* ``VScale log2e`` multiplies by the module-precision value of LOG2E_F64
  (tilecc/numerics.py:66); ``max`` / ``min`` propagate NaN like
  ``np.maximum`` / ``np.minimum``; a zero denominator in a tile divide sets a
  device flag and raises ``DivisionByZero`` (tilecc/numerics.py:123-126).

Buffers: Global buffers are device arrays in the module precision
(non-input ones zero-initialised, interp.py:114-115).  Shared / Register
buffers are private per CUDA block (shared memory when they fit, else a
per-block slice of a global scratch arena).  The reference allocates them once
per module and runs blocks one after another, so a block could observe values
a previous block left behind; the lowering proves that every such buffer is
written before it is read in each block, and otherwise runs the module's
blocks sequentially in one CUDA block over one persistent scratch arena --
the reference's own order.  Likewise a kernel whose block points write
overlapping Global regions, or read Global elements another block point
writes, runs its block points sequentially.
"""

from __future__ import annotations

import hashlib
import itertools
import math
import os
import shutil
import subprocess
import tempfile
import threading
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from . import ma_ir as ir
from .errors import DivisionByZero, OutOfBounds, UnsupportedMA

THREADS = 256
SMEM_LIMIT = 200 * 1024          # dynamic shared memory used for private buffers
MAX_GRID = 148 * 8               # CUDA blocks of a parallel kernel (grid-stride over block points)
SCRATCH_CAP = 1 << 30            # bytes of global scratch for private buffers
LOG2E_F64 = 1.4426950408889634   # tilecc/numerics.py:66: log2(e) in fp64
NVCC_FLAGS = ["-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
              "--fmad=false", "-lineinfo"]

_PKG = os.path.dirname(os.path.abspath(__file__))
CACHE_DIR = os.environ.get("NT_JIT_CACHE") or os.path.join(_PKG, "_native", "jit")


# ---------------------------------------------------------------------------
# Small helpers


def _prod(xs) -> int:
    return int(math.prod(int(x) for x in xs))


def _ctype(precision: str) -> str:
    if precision == "fp32":
        return "float"
    if precision == "fp64":
        return "double"
    raise UnsupportedMA(f"precision {precision!r} has no device realisation (exact rationals are CPU-only)")


def _lit(value: float, T: str) -> str:
    v = float(value)
    if math.isnan(v):
        return f"(({T})NAN)"
    if math.isinf(v):
        return f"(({T})INFINITY)" if v > 0 else f"(-({T})INFINITY)"
    return f"(({T}){v.hex()})"


def _affine_c(a: ir.Affine) -> str:
    parts = [f"{c}*{v}" if c != 1 else v for v, c in a.coefs]
    if a.const or not parts:
        parts.append(str(a.const))
    return "(" + " + ".join(parts) + ")"


def _strides(shape) -> list[int]:
    st, acc = [], 1
    for d in reversed(shape):
        st.append(acc)
        acc *= int(d)
    return list(reversed(st))


def _unravel(flat: str, shape) -> list[str]:
    """C expressions for the C-order multi-index of `flat` over `shape`."""
    shape = [int(d) for d in shape]
    st = _strides(shape)
    out = []
    for d, s in zip(shape, st):
        if d == 1:
            out.append("0")
        elif s == 1:
            out.append(f"(({flat}) % {d})")
        else:
            out.append(f"((({flat}) / {s}) % {d})" if s * d != _prod(shape) else f"(({flat}) / {s})")
    return out


def _ravel(idx, shape) -> str:
    st = _strides(shape)
    terms = [f"({i})*{s}" if s != 1 else f"({i})" for i, s, d in zip(idx, st, shape) if int(d) != 1]
    return "(" + " + ".join(terms) + ")" if terms else "0"


def _bcast(idx, out_shape, in_shape) -> list[str]:
    """numpy broadcasting: the index into an operand of `in_shape` (right-aligned)."""
    lead = len(out_shape) - len(in_shape)
    if lead < 0:
        raise UnsupportedMA(f"operand rank {len(in_shape)} exceeds result rank {len(out_shape)}")
    res = []
    for d, n in enumerate(in_shape):
        o = out_shape[lead + d]
        if int(n) == 1 and int(o) != 1:
            res.append("0")
        elif int(n) == int(o):
            res.append(idx[lead + d])
        else:
            raise UnsupportedMA(f"shapes {tuple(in_shape)} and {tuple(out_shape)} do not broadcast")
    return res


def _contains(e: ir.Expr, kinds) -> bool:
    return any(isinstance(n, kinds) for n in e.walk())


def _is_view(e: ir.Expr) -> bool:
    """Ref / Lit reached through index-only adapters: cheap to re-read per use."""
    while isinstance(e, (ir.Transpose, ir.Reshape, ir.Broadcast)):
        e = e.x
    return isinstance(e, (ir.Ref, ir.Lit))


def _refs(e: ir.Expr):
    return [n for n in e.walk() if isinstance(n, ir.Ref)]


def _full_slices(shape) -> tuple:
    return tuple(ir.Slice(ir.Affine.make({}, 0), int(d)) for d in shape)


# ---------------------------------------------------------------------------
# Program preparation: hoisting and analyses


@dataclass
class _Prepared:
    module: ir.Module
    kernels: list                  # list[ir.Kernel] with hoisted temporaries
    private: dict                  # name -> shape of block-private buffers (non-Global + temps)
    stage_elems: int               # staging tile for self-referencing statements
    carried: bool                  # a private buffer is read before written in some block
    sequential: list               # per kernel: run block points sequentially


class _Hoister:
    """Moves expensive Dot / Reduce operands into private temporaries.

    A Dot operand is evaluated K times per output element and a nested Dot or
    Reduce inside a Reduce operand is evaluated per reduced element; hoisting
    them into their own statement (evaluated once per element, like the
    reference's whole-tile numpy evaluation) keeps the work linear.  Values
    are unchanged: the temporary holds exactly the operand tile.
    """

    def __init__(self):
        self.n = 0
        self.temps: dict = {}

    def fresh(self, shape) -> str:
        self.n += 1
        name = f"__h{self.n}"
        self.temps[name] = tuple(int(d) for d in shape)
        return name

    def expr(self, e: ir.Expr, pre: list) -> ir.Expr:
        if isinstance(e, ir.Dot):
            a = self.expr(e.a, pre)
            b = self.expr(e.b, pre)
            seed = self.expr(e.seed, pre) if e.seed is not None else None
            a = a if _is_view(a) else self.spill(a, pre)
            b = b if _is_view(b) else self.spill(b, pre)
            return replace(e, a=a, b=b, seed=seed)
        if isinstance(e, ir.Reduce):
            x = self.expr(e.x, pre)
            seed = self.expr(e.seed, pre) if e.seed is not None else None
            if _contains(x, (ir.Dot, ir.Reduce)):
                x = self.spill(x, pre)
            return replace(e, x=x, seed=seed)
        if isinstance(e, ir.Bin):
            return replace(e, a=self.expr(e.a, pre), b=self.expr(e.b, pre))
        if isinstance(e, (ir.Un, ir.Scale, ir.Transpose, ir.Reshape, ir.Broadcast)):
            x = self.expr(e.x, pre)
            if isinstance(e, (ir.Transpose, ir.Reshape, ir.Broadcast)) and _contains(x, (ir.Dot, ir.Reduce)):
                x = self.spill(x, pre)  # index adapters re-read their operand per element
            return replace(e, x=x)
        return e

    def spill(self, e: ir.Expr, pre: list) -> ir.Ref:
        name = self.fresh(e.shape)
        sl = _full_slices(e.shape)
        pre.append(ir.Compute(name, sl, e))
        return ir.Ref(tuple(e.shape), name, sl)

    def body(self, body) -> tuple:
        out = []
        for st in body:
            if isinstance(st, ir.Loop):
                out.append(replace(st, body=self.body(st.body)))
            elif isinstance(st, ir.Compute):
                pre: list = []
                e = self.expr(st.expr, pre)
                out.extend(pre)
                out.append(replace(st, expr=e))
            else:
                out.append(st)
        return tuple(out)


def _loop_points(loops, cap=1 << 16):
    """All assignments of the enclosing loop variables (bounded)."""
    if not loops:
        return [{}]
    n = _prod(e for _, e in loops)
    if n > cap:
        return None
    names = [v for v, _ in loops]
    return [dict(zip(names, p)) for p in itertools.product(*[range(e) for _, e in loops])]


def _walk_accesses(body, loops=()):
    """Yield (kind, buffer, slices, loops) for every access in program order."""
    for st in body:
        if isinstance(st, ir.Loop):
            yield from _walk_accesses(st.body, loops + ((st.var, st.extent),))
        elif isinstance(st, ir.Copy):
            yield ("r", st.src, st.src_slices, loops)
            yield ("w", st.dst, st.dst_slices, loops)
        else:
            for r in _refs(st.expr):
                yield ("r", r.buffer, r.slices, loops)
            yield ("w", st.dst, st.dst_slices, loops)


def _mark(arr, slices, envs, value=True):
    for env in envs:
        idx = tuple(slice(s.off.evaluate(env), s.off.evaluate(env) + s.length) for s in slices)
        arr[idx] = value


def _covered(arr, slices, envs) -> bool:
    for env in envs:
        idx = tuple(slice(s.off.evaluate(env), s.off.evaluate(env) + s.length) for s in slices)
        if not np.all(arr[idx]):
            return False
    return True


def _private_carried(kernel: ir.Kernel, private: dict) -> bool:
    """True if some private buffer may be read before this block point wrote it."""
    written = {n: np.zeros(s, dtype=bool) for n, s in private.items()}
    block_env = {v: 0 for v, _, _ in kernel.blocks}
    for kind, buf, slices, loops in _walk_accesses(kernel.body):
        if buf not in private:
            continue
        if any(v in block_env for s in slices for v in s.off.vars()):
            return True  # a private buffer indexed by the block point: keep the reference order
        envs = _loop_points(loops)
        if envs is None:
            return True
        envs = [dict(block_env, **e) for e in envs]
        if kind == "w":
            _mark(written[buf], slices, envs)
        elif not _covered(written[buf], slices, envs):
            return True
    return False


def _global_conflict(kernel: ir.Kernel, module: ir.Module, max_points=4096, max_elems=1 << 24) -> bool:
    """True if two block points of the kernel touch a Global element one of them writes."""
    points = _prod(e for _, _, e in kernel.blocks)
    if points <= 1:
        return False
    gl = {b.name: b.shape for b in module.buffers if b.scope == "Global"}
    acc = [a for a in _walk_accesses(kernel.body) if a[1] in gl]
    written = {buf for kind, buf, _, _ in acc if kind == "w"}
    if not written:
        return False
    if points > max_points or any(_prod(gl[b]) > max_elems for b in written):
        return _global_conflict_affine(kernel, acc, written)
    owner = {b: np.full(gl[b], -1, dtype=np.int64) for b in written}
    names = [v for v, _, _ in kernel.blocks]
    pts = list(itertools.product(*[range(e) for _, _, e in kernel.blocks]))
    for pi, p in enumerate(pts):
        benv = dict(zip(names, p))
        for kind, buf, slices, loops in acc:
            if kind != "w":
                continue
            envs = _loop_points(loops)
            if envs is None:
                return True
            for env in envs:
                env = dict(benv, **env)
                idx = tuple(slice(s.off.evaluate(env), s.off.evaluate(env) + s.length) for s in slices)
                region = owner[buf][idx]
                if np.any((region != -1) & (region != pi)):
                    return True
                region[...] = pi
    for pi, p in enumerate(pts):
        benv = dict(zip(names, p))
        for kind, buf, slices, loops in acc:
            if kind != "r" or buf not in written:
                continue
            envs = _loop_points(loops)
            if envs is None:
                return True
            for env in envs:
                env = dict(benv, **env)
                idx = tuple(slice(s.off.evaluate(env), s.off.evaluate(env) + s.length) for s in slices)
                region = owner[buf][idx]
                if np.any((region != -1) & (region != pi)):
                    return True
    return False


def _global_conflict_affine(kernel, acc, written) -> bool:
    """Sufficient independence test for large kernels: every write of a Global
    buffer has, for each block variable, a dimension whose offset moves by at
    least the slice length per step of that variable and does not depend on
    any loop variable; reads of written buffers must be exactly the writes."""
    bvars = [(v, e) for v, _, e in kernel.blocks if e > 1]
    writes = [(buf, sl) for kind, buf, sl, _ in acc if kind == "w"]
    for buf, sl in writes:
        for v, _ in bvars:
            ok = False
            for s in sl:
                c = s.off.coef(v)
                if abs(c) >= s.length and not (s.off.vars() - {b for b, _, _ in kernel.blocks}):
                    ok = True
            if not ok:
                return True
    wset = {(buf, tuple((s.off, s.length) for s in sl)) for buf, sl in writes}
    for kind, buf, sl, _ in acc:
        if kind == "r" and buf in written and (buf, tuple((s.off, s.length) for s in sl)) not in wset:
            return True
    return False


def prepare(module: ir.Module) -> _Prepared:
    private = {b.name: tuple(b.shape) for b in module.buffers if b.scope != "Global"}
    h = _Hoister()
    kernels = [replace(k, body=h.body(k.body)) for k in module.kernels]
    private.update(h.temps)
    stage = 0
    for k in kernels:
        for st in _statements(k.body):
            if _needs_stage(st):
                stage = max(stage, _prod(_dst_shape(st)))
    carried = any(_private_carried(k, private) for k in kernels)
    sequential = [carried or _global_conflict(k, module) for k in kernels]
    return _Prepared(module, kernels, private, stage, carried, sequential)


def _statements(body):
    for st in body:
        if isinstance(st, ir.Loop):
            yield from _statements(st.body)
        else:
            yield st


def _dst_shape(st) -> tuple:
    return tuple(s.length for s in st.dst_slices)


def _aligned_only(e: ir.Expr, dst: str, dst_slices, shape) -> bool:
    """Every read of `dst` in `e` touches exactly the element being written."""

    def go(n, elementwise: bool) -> bool:
        if isinstance(n, ir.Ref):
            if n.buffer != dst:
                return True
            return (elementwise and tuple(n.shape) == tuple(shape)
                    and tuple((s.off, s.length) for s in n.slices) == tuple((s.off, s.length) for s in dst_slices))
        if isinstance(n, ir.Bin):
            return go(n.a, elementwise and n.a.shape == n.shape) and go(n.b, elementwise and n.b.shape == n.shape)
        if isinstance(n, (ir.Un, ir.Scale)):
            return go(n.x, elementwise)
        if isinstance(n, ir.Dot):
            ok = go(n.a, False) and go(n.b, False)
            if n.seed is not None:
                ok = ok and go(n.seed, elementwise and tuple(n.seed.shape) == tuple(n.shape))
            return ok
        if isinstance(n, ir.Reduce):
            ok = go(n.x, False)
            if n.seed is not None:
                ok = ok and go(n.seed, elementwise and tuple(n.seed.shape) == tuple(n.shape))
            return ok
        if isinstance(n, (ir.Transpose, ir.Reshape, ir.Broadcast)):
            return go(n.x, False)
        return True

    return go(e, tuple(e.shape) == tuple(shape))


def _needs_stage(st) -> bool:
    if isinstance(st, ir.Copy):
        return st.src == st.dst
    return not _aligned_only(st.expr, st.dst, st.dst_slices, _dst_shape(st))


# ---------------------------------------------------------------------------
# Code generation


class _Gen:
    def __init__(self, prep: _Prepared, T: str):
        self.p = prep
        self.T = T
        self.lines: list[str] = []
        self.n = 0
        self.glob = {b.name: tuple(b.shape) for b in prep.module.buffers if b.scope == "Global"}

    def tmp(self, prefix="_v") -> str:
        self.n += 1
        return f"{prefix}{self.n}"

    def emit(self, line: str, depth: int):
        self.lines.append("  " * depth + line)

    # -- buffer addressing
    def addr(self, buf: str, slices, idx) -> str:
        shape = self.glob.get(buf) or self.p.private.get(buf)
        if shape is None:
            raise UnsupportedMA(f"unknown buffer {buf!r}")
        if len(slices) != len(shape):
            raise UnsupportedMA(f"buffer {buf!r}: {len(slices)} slices for rank {len(shape)}")
        st = _strides(shape)
        terms = []
        for s, i, stride in zip(slices, idx, st):
            off = _affine_c(s.off)
            pos = f"({off} + {i})" if i != "0" else off
            terms.append(f"(long long){pos}*{stride}LL" if stride != 1 else f"(long long){pos}")
        flat = " + ".join(terms) if terms else "0"
        name = ("g_" if buf in self.glob else "p_") + _cname(buf)
        return f"{name}[{flat}]"

    # -- expressions: returns a C expression (a temporary or a literal)
    def expr(self, e: ir.Expr, idx: list, d: int) -> str:
        T = self.T
        if isinstance(e, ir.Lit):
            return _lit(e.value, T)
        if isinstance(e, ir.Ref):
            lengths = tuple(s.length for s in e.slices)
            ridx = idx
            if tuple(lengths) != tuple(e.shape):  # a ref read through a reshape
                ridx = _unravel(_ravel(idx, e.shape), lengths)
            v = self.tmp()
            self.emit(f"const {T} {v} = {self.addr(e.buffer, e.slices, ridx)};", d)
            return v
        if isinstance(e, ir.Bin):
            a = self.expr(e.a, _bcast(idx, e.shape, e.a.shape), d)
            b = self.expr(e.b, _bcast(idx, e.shape, e.b.shape), d)
            v = self.tmp()
            if e.op == "add":
                rhs = f"{a} + {b}"
            elif e.op == "sub":
                rhs = f"{a} - {b}"
            elif e.op == "mul":
                rhs = f"{a} * {b}"
            elif e.op == "div":
                self.emit(f"if ({b} == ({T})0) atomicOr(err, 1);", d)
                rhs = f"{a} / {b}"
            elif e.op == "max":
                rhs = f"nt_max({a}, {b})"
            elif e.op == "min":
                rhs = f"nt_min({a}, {b})"
            else:
                raise UnsupportedMA(f"binary op {e.op!r}")
            self.emit(f"const {T} {v} = {rhs};", d)
            return v
        if isinstance(e, ir.Un):
            x = self.expr(e.x, idx, d)
            v = self.tmp()
            fn = {"exp": "exp", "exp2": "exp2", "log2": "log2"}.get(e.op)
            if e.op == "neg":
                rhs = f"-{x}"
            elif fn is not None:
                rhs = f"{fn}{'f' if T == 'float' else ''}({x})"
            else:
                raise UnsupportedMA(f"unary op {e.op!r}")
            self.emit(f"const {T} {v} = {rhs};", d)
            return v
        if isinstance(e, ir.Scale):
            if e.kind != "log2e":
                raise UnsupportedMA(f"scale {e.kind!r}")
            x = self.expr(e.x, idx, d)
            v = self.tmp()
            self.emit(f"const {T} {v} = {_lit(LOG2E_F64, T)} * {x};", d)
            return v
        if isinstance(e, ir.Dot):
            if len(e.a.shape) != 2 or len(e.b.shape) != 2 or len(e.shape) != 2:
                raise UnsupportedMA("dot of non-matrix tiles")
            K = int(e.a.shape[1])
            acc = self.tmp("_acc")
            if e.seed is not None:
                s = self.expr(e.seed, _bcast(idx, e.shape, e.seed.shape), d)
                self.emit(f"{T} {acc} = {s};", d)
            else:
                self.emit(f"{T} {acc} = ({T})0;", d)
            k = self.tmp("_k")
            self.emit(f"for (int {k} = 0; {k} < {K}; ++{k}) {{", d)
            a = self.expr(e.a, [idx[0], k], d + 1)
            b = self.expr(e.b, [k, idx[1]], d + 1)
            self.emit(f"{acc} = {acc} + {a} * {b};", d + 1)
            self.emit("}", d)
            return acc
        if isinstance(e, ir.Reduce):
            xs = tuple(int(s) for s in e.x.shape)
            axes = tuple(int(a) % len(xs) for a in e.axes)
            keep = [i for i in range(len(xs)) if i not in axes]
            red_shape = [xs[a] for a in axes]
            R = _prod(red_shape)
            if R == 0:
                raise UnsupportedMA("reduction over an empty axis")
            op = {"sum": "{a} + {b}", "prod": "{a} * {b}", "max": "nt_max({a}, {b})",
                  "min": "nt_min({a}, {b})"}.get(e.op)
            if op is None:
                raise UnsupportedMA(f"reduce op {e.op!r}")
            r = self.tmp("_r")

            def xidx(rvar):
                ri = _unravel(rvar, red_shape)
                full = ["0"] * len(xs)
                for pos, ax in enumerate(keep):
                    full[ax] = idx[pos]
                for pos, ax in enumerate(axes):
                    full[ax] = ri[pos]
                return full

            acc = self.tmp("_acc")
            if e.seed is not None:
                s = self.expr(e.seed, _bcast(idx, e.shape, e.seed.shape), d)
                self.emit(f"{T} {acc} = {s};", d)
                start = 0
            else:
                first = self.expr(e.x, xidx("0"), d)
                self.emit(f"{T} {acc} = {first};", d)
                start = 1
            if R > start:
                self.emit(f"for (int {r} = {start}; {r} < {R}; ++{r}) {{", d)
                x = self.expr(e.x, xidx(r), d + 1)
                self.emit(f"{acc} = {op.format(a=acc, b=x)};", d + 1)
                self.emit("}", d)
            return acc
        if isinstance(e, ir.Transpose):
            perm = tuple(e.perm)
            xi = ["0"] * len(perm)
            for i, p in enumerate(perm):
                xi[p] = idx[i]
            return self.expr(e.x, xi, d)
        if isinstance(e, ir.Reshape):
            return self.expr(e.x, _unravel(_ravel(idx, e.shape), e.x.shape), d)
        if isinstance(e, ir.Broadcast):
            return self.expr(e.x, _bcast(idx, e.shape, e.x.shape), d)
        raise UnsupportedMA(f"MA eval: unexpected node {type(e).__name__}")

    # -- statements
    def stmt(self, st, d: int):
        T = self.T
        if isinstance(st, ir.Loop):
            self.emit(f"for (int {st.var} = 0; {st.var} < {int(st.extent)}; ++{st.var}) {{", d)
            for s in st.body:
                self.stmt(s, d + 1)
            self.emit("}", d)
            return
        if isinstance(st, ir.Copy):
            src_shape = tuple(s.length for s in st.src_slices)
            expr = ir.Ref(src_shape, st.src, st.src_slices)
        else:
            expr = st.expr
        dshape = _dst_shape(st)
        ne = _prod(dshape)
        if _prod(expr.shape) != ne:
            raise UnsupportedMA(f"statement writing {st.dst!r}: {tuple(expr.shape)} does not fit {dshape}")
        staged = _needs_stage(st)
        e_ = self.tmp("_e")
        self.emit(f"for (int {e_} = threadIdx.x; {e_} < {ne}; {e_} += blockDim.x) {{", d)
        val = self.expr(expr, _unravel(e_, expr.shape), d + 1)
        if staged:
            self.emit(f"p___stage[{e_}] = {val};", d + 1)
        else:
            self.emit(f"{self.addr(st.dst, st.dst_slices, _unravel(e_, dshape))} = {val};", d + 1)
        self.emit("}", d)
        self.emit("__syncthreads();", d)
        if staged:
            self.emit(f"for (int {e_} = threadIdx.x; {e_} < {ne}; {e_} += blockDim.x)", d)
            self.emit(f"  {self.addr(st.dst, st.dst_slices, _unravel(e_, dshape))} = p___stage[{e_}];", d)
            self.emit("__syncthreads();", d)


def _cname(name: str) -> str:
    return "".join(c if c.isalnum() or c == "_" else "_" for c in name)


@dataclass
class KernelLaunch:
    entry: str
    points: int
    sequential: bool
    grid: int
    smem_bytes: int
    scratch_elems_per_block: int   # 0: private buffers in shared memory


@dataclass
class LoweredProgram:
    """CUDA source of an MA module plus its launch plan."""

    source: str
    precision: str
    ctype: str
    globals_: list                 # Global buffer names in kernel-parameter order
    launches: list                 # list[KernelLaunch]
    private_layout: dict           # name -> (offset elems, shape)
    private_elems: int
    carried: bool
    digest: str = ""
    realisation: dict = field(default_factory=dict)


def lower(module, precision: Optional[str] = None) -> LoweredProgram:
    """Lower an MA module to CUDA C (no device needed)."""
    mod = ir.as_module(module)
    prec = precision or mod.precision
    T = _ctype(prec)
    item = 4 if T == "float" else 8
    prep = prepare(mod)
    layout, off = {}, 0
    names = sorted(prep.private)
    for n in names:
        layout[n] = (off, prep.private[n])
        off += -(-_prod(prep.private[n]) // 4) * 4  # 16-byte aligned (fp32) / 32-byte (fp64)
    if prep.stage_elems:
        layout["__stage"] = (off, (prep.stage_elems,))
        off += -(-prep.stage_elems // 4) * 4
    private_elems = max(off, 4)
    in_smem = not prep.carried and private_elems * item <= SMEM_LIMIT
    glob = [b.name for b in mod.buffers if b.scope == "Global"]

    out = [
        "// generated by paper_2604_14825_b200.simt from an MA module (tilecc/ma/interp.py semantics)",
        "#include <math.h>",
        f"typedef {T} T;",
        "__device__ __forceinline__ T nt_max(T a, T b) { return (a >= b || a != a) ? a : b; }",
        "__device__ __forceinline__ T nt_min(T a, T b) { return (a <= b || a != a) ? a : b; }",
    ]
    launches = []
    for ki, (k, seq) in enumerate(zip(prep.kernels, prep.sequential)):
        g = _Gen(prep, T)
        points = _prod(e for _, _, e in k.blocks)
        entry = f"nt_ma_{ki}_{_cname(k.name)}"
        params = ", ".join(f"T* __restrict__ g_{_cname(n)}" for n in glob)
        out.append(f'extern "C" __global__ void __launch_bounds__({THREADS}) {entry}({params}, '
                   "T* __restrict__ scratch, long long scratch_stride, int* __restrict__ err) {")
        if in_smem:
            out.append("  extern __shared__ __align__(16) unsigned char smem_raw[];")
            out.append("  T* priv = reinterpret_cast<T*>(smem_raw);")
        else:
            out.append("  T* priv = scratch + (long long)blockIdx.x * scratch_stride;")
        for n, (o, _) in layout.items():
            out.append(f"  T* __restrict__ p_{_cname(n)} = priv + {o};")
        out.append(f"  for (long long bp = blockIdx.x; bp < {points}LL; bp += gridDim.x) {{")
        rem = "bp"
        blocks = list(k.blocks)
        for i, (var, _, ext) in enumerate(reversed(blocks)):
            last = i == len(blocks) - 1
            out.append(f"    const int {var} = (int)({rem}" + ("" if last else f" % {int(ext)}") + ");")
            if not last:
                nr = f"_bq{i}"
                out.append(f"    const long long {nr} = {rem} / {int(ext)};")
                rem = nr
        for st in k.body:
            g.stmt(st, 2)
        out.extend(g.lines)
        out.append("    __syncthreads();")
        out.append("  }")
        out.append("}")
        if seq:
            grid = 1
        else:
            grid = min(points, MAX_GRID)
            if not in_smem:
                grid = max(1, min(grid, SCRATCH_CAP // max(1, private_elems * item)))
        launches.append(KernelLaunch(entry, points, seq, grid, private_elems * item if in_smem else 0,
                                     0 if in_smem else private_elems))
    src = "\n".join(out) + "\n"
    digest = hashlib.sha256((src + " ".join(NVCC_FLAGS)).encode()).hexdigest()[:24]
    real = {"kernel": "simt", "precision": prec, "private_in_smem": in_smem, "carried": prep.carried,
            "sequential": [l.sequential for l in launches], "grid": [l.grid for l in launches]}
    return LoweredProgram(src, prec, T, glob, launches, layout, private_elems, prep.carried, digest, real)


# ---------------------------------------------------------------------------
# Compilation (nvcc, content-hash cache) and execution


_mem_cache: dict = {}
_cache_lock = threading.Lock()


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise UnsupportedMA("nvcc not found: generic MA programs are compiled at run time")


def compile_cubin(prog: LoweredProgram) -> str:
    """nvcc -> sm_100a cubin, cached under CACHE_DIR by content hash; returns the path."""
    os.makedirs(CACHE_DIR, exist_ok=True)
    path = os.path.join(CACHE_DIR, prog.digest + ".cubin")
    if os.path.exists(path):
        return path
    with tempfile.TemporaryDirectory() as td:
        cu = os.path.join(td, "ma.cu")
        with open(cu, "w") as f:
            f.write(prog.source)
        tmp_out = os.path.join(td, "ma.cubin")
        r = subprocess.run([_nvcc()] + NVCC_FLAGS + ["-o", tmp_out, cu], capture_output=True, text=True)
        if r.returncode != 0:
            raise UnsupportedMA(f"nvcc failed on the lowered MA program:\n{r.stderr[-4000:]}")
        tmp_final = path + f".{os.getpid()}.tmp"
        shutil.copyfile(tmp_out, tmp_final)
        os.replace(tmp_final, path)  # atomic for concurrent workers
    return path


class _Loaded:
    def __init__(self, prog: LoweredProgram):
        import ctypes as C

        from . import _lib

        self.prog = prog
        path = compile_cubin(prog)
        with open(path, "rb") as f:
            self.image = f.read()
        L = _lib.lib()
        h = C.c_void_p()
        buf = C.create_string_buffer(self.image, len(self.image))
        _lib.check(L.nt_module_load(buf, len(self.image), C.byref(h)), "nt_module_load")
        self.handle = h
        self.fns = []
        for ln in prog.launches:
            fn = C.c_void_p()
            _lib.check(L.nt_module_function(h, ln.entry.encode(), C.byref(fn)), "nt_module_function")
            self.fns.append(fn)


def load(prog: LoweredProgram) -> _Loaded:
    import torch

    key = (prog.digest, torch.cuda.current_device())
    with _cache_lock:
        hit = _mem_cache.get(key)
        if hit is None:
            hit = _Loaded(prog)
            _mem_cache[key] = hit
    return hit


_lower_cache: dict = {}


def lower_cached(module, precision=None) -> LoweredProgram:
    key = (id(module), precision)
    hit = _lower_cache.get(key)
    if hit is not None and hit[0] is module:
        return hit[1]
    prog = lower(module, precision)
    if len(_lower_cache) > 256:
        _lower_cache.clear()
    _lower_cache[key] = (module, prog)
    return prog


def execute(module, inputs: dict, precision: Optional[str] = None, stream=None, return_torch: bool = False):
    """Run an MA module with the SIMT lowering.

    Returns ``(buffers, info)``: every Global buffer (inputs as given, the
    rest computed on the device) and a dict with the device time and launch
    count.  Shape mismatches raise ``OutOfBounds`` (interp.py:111-112); a zero
    denominator raises ``DivisionByZero``.
    """
    import ctypes as C

    import torch

    from . import _lib

    mod = ir.as_module(module)
    prog = lower_cached(module, precision)
    if not torch.cuda.is_available():
        raise UnsupportedMA("no CUDA device: the B200 executor has no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float32 if prog.ctype == "float" else torch.float64
    ndt = np.float32 if prog.ctype == "float" else np.float64
    tensors = {}
    for b in mod.buffers:
        if b.scope != "Global":
            continue
        if b.is_input:
            if b.name not in inputs:
                raise OutOfBounds(f"input {b.name!r} missing")
            x = inputs[b.name]
            if isinstance(x, torch.Tensor):
                t = x.to(device=dev, dtype=tdt).contiguous().clone()
            else:
                arr = np.ascontiguousarray(np.asarray(x, dtype=ndt))
                t = torch.from_numpy(arr).to(dev)
            if tuple(t.shape) != tuple(b.shape):
                raise OutOfBounds(f"input {b.name!r}: wrong shape {tuple(t.shape)}")
            tensors[b.name] = t
        else:
            tensors[b.name] = torch.zeros(tuple(b.shape), dtype=tdt, device=dev)
    loaded = load(prog)
    L = _lib.lib()
    cur = torch.cuda.current_stream(dev)
    if stream is None or (stream if isinstance(stream, int) else stream.cuda_stream) == cur.cuda_stream:
        st = cur
    else:
        st = stream if not isinstance(stream, int) else torch.cuda.ExternalStream(stream, device=dev)
        st.wait_stream(cur)  # inputs, zeroed buffers and scratch were staged on the current stream
    st_handle = C.c_void_p(st.cuda_stream)
    max_grid = max(l.grid for l in prog.launches) if prog.launches else 1
    scratch_elems = max([l.scratch_elems_per_block * l.grid for l in prog.launches] + [1])
    if prog.carried:
        scratch_elems = max(scratch_elems, prog.private_elems)
    scratch = torch.zeros(scratch_elems, dtype=tdt, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    ptrs = [C.c_void_p(tensors[n].data_ptr()) for n in prog.globals_]
    sp = C.c_void_p(scratch.data_ptr())
    ep = C.c_void_p(err.data_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(st)
    for ln, fn in zip(prog.launches, loaded.fns):
        stride = C.c_longlong(0 if prog.carried else ln.scratch_elems_per_block)
        args = ptrs + [sp, stride, ep]
        arr = (C.c_void_p * len(args))(*[C.cast(C.pointer(a), C.c_void_p) for a in args])
        _lib.check(L.nt_launch(fn, ln.grid, THREADS, ln.smem_bytes, arr, st_handle), "nt_launch")
    ev1.record(st)
    if st is not cur:
        cur.wait_stream(st)  # outputs and the error flag are read on the current stream
    ev1.synchronize()
    if int(err.item()) & 1:
        raise DivisionByZero("tile divide")
    info = dict(prog.realisation, device_ms=ev0.elapsed_time(ev1), launches=len(prog.launches),
                digest=prog.digest, max_grid=max_grid)
    bufs = {}
    for b in mod.buffers:
        if b.scope != "Global":
            continue
        if b.is_input:
            bufs[b.name] = inputs[b.name]
        else:
            t = tensors[b.name]
            bufs[b.name] = t if return_torch else t.cpu().numpy()
    return bufs, info
