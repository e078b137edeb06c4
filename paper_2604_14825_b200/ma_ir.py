"""Mirror of the reference MA-tile IR (the input contract of the B200 backend).

The reference defines the MA-tile IR in ``tilecc/ma/ir.py:15-105`` (MARef,
MACopy, MACompute, MALoop, MAKernel, MAModule), tile expressions in
``tilecc/vr/ir.py:20-140`` (VSlice, VLit, VBin, VUn, VScale, VDot, VReduce,
VTranspose, VReshape, VBroadcast) and buffers in ``tilecc/scalar/ir.py:55-63``
(BufferDecl with a Scope).  This module restates those types as plain frozen
dataclasses so that the backend can consume an MA program

* live, from a ``tilecc`` ``MAModule`` object (``from_tilecc``; duck-typed on
  class names, so ``tilecc`` is never imported here), or
* serialised, from the stable JSON produced by ``to_json`` (used for the
  committed golden fixtures and on GPU boxes where ``tilecc`` is absent).

Slice offsets are kept as integer affine forms (``Affine``) -- the reference
evaluates them with ``to_affine(...).evaluate(env)`` (tilecc/ma/interp.py:151-157,
tilecc/exprs.py:186-190) -- plus the reference's canonical text of the offset
expression so ``emit_text`` reproduces ``emit_tile_text(..., "generic")``
(tilecc/ma/emit.py:32-147) byte for byte.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Optional, Union

SCOPES = ("Global", "Shared", "Register")


class UnsupportedMA(Exception):
    """Raised when an MA program has no B200 realisation (no CPU fallback)."""


# ---------------------------------------------------------------------------
# Index math


@dataclass(frozen=True)
class Affine:
    """sum(coef[v] * v) + const over block / loop variables (integers)."""

    coefs: tuple[tuple[str, int], ...]
    const: int = 0

    @staticmethod
    def make(coefs: dict, const: int = 0) -> "Affine":
        return Affine(tuple(sorted((k, int(v)) for k, v in coefs.items() if v)), int(const))

    def coef(self, var: str) -> int:
        for k, v in self.coefs:
            if k == var:
                return v
        return 0

    def vars(self) -> set:
        return {k for k, _ in self.coefs}

    def evaluate(self, env: dict) -> int:
        total = self.const
        for k, c in self.coefs:
            total += c * env[k]
        return total


@dataclass(frozen=True)
class Slice:
    off: Affine
    length: int
    text: str = ""  # reference's str(VSlice) (tilecc/vr/ir.py:25-27)

    def __str__(self):
        if self.text:
            return self.text
        return _default_slice_text(self.off, self.length)


def _default_slice_text(off: Affine, length: int) -> str:
    parts = []
    for k, c in off.coefs:
        parts.append(k if c == 1 else f"{c} * {k}")
    if off.const or not parts:
        parts.append(str(off.const))
    o = " + ".join(parts)
    return f"{o}:{o}+{length}" if o != "0" else f"0:{length}"


# ---------------------------------------------------------------------------
# Tile expressions


@dataclass(frozen=True)
class Expr:
    shape: tuple[int, ...]

    def children(self) -> tuple["Expr", ...]:
        return ()

    def walk(self):
        yield self
        for c in self.children():
            yield from c.walk()


@dataclass(frozen=True)
class Lit(Expr):
    value: float = 0.0


@dataclass(frozen=True)
class Ref(Expr):
    """MARef: tile-shaped read of a buffer slice (tilecc/ma/ir.py:15-21)."""

    buffer: str = ""
    slices: tuple[Slice, ...] = ()


@dataclass(frozen=True)
class Bin(Expr):
    op: str = "add"  # add sub mul div max min
    a: Expr = None
    b: Expr = None

    def children(self):
        return (self.a, self.b)


@dataclass(frozen=True)
class Un(Expr):
    op: str = "exp"  # exp exp2 log2 neg
    x: Expr = None

    def children(self):
        return (self.x,)


@dataclass(frozen=True)
class Scale(Expr):
    kind: str = "log2e"
    x: Expr = None

    def children(self):
        return (self.x,)


@dataclass(frozen=True)
class Dot(Expr):
    a: Expr = None
    b: Expr = None
    seed: Optional[Expr] = None

    def children(self):
        return (self.a, self.b) + ((self.seed,) if self.seed is not None else ())


@dataclass(frozen=True)
class Reduce(Expr):
    op: str = "sum"
    x: Expr = None
    axes: tuple[int, ...] = ()
    seed: Optional[Expr] = None

    def children(self):
        return (self.x,) + ((self.seed,) if self.seed is not None else ())


@dataclass(frozen=True)
class Transpose(Expr):
    x: Expr = None
    perm: tuple[int, ...] = (1, 0)

    def children(self):
        return (self.x,)


@dataclass(frozen=True)
class Reshape(Expr):
    x: Expr = None

    def children(self):
        return (self.x,)


@dataclass(frozen=True)
class Broadcast(Expr):
    x: Expr = None

    def children(self):
        return (self.x,)


# ---------------------------------------------------------------------------
# Statements, kernels, modules


@dataclass(frozen=True)
class Copy:
    dst: str
    dst_slices: tuple[Slice, ...]
    src: str
    src_slices: tuple[Slice, ...]


@dataclass(frozen=True)
class Compute:
    dst: str
    dst_slices: tuple[Slice, ...]
    expr: Expr


@dataclass(frozen=True)
class Loop:
    var: str
    extent: int
    body: tuple


Stmt = Union[Copy, Compute, Loop]


@dataclass(frozen=True)
class Buffer:
    name: str
    shape: tuple[int, ...]
    precision: str = "fp32"
    scope: str = "Global"
    is_input: bool = False
    is_output: bool = False


@dataclass(frozen=True)
class Kernel:
    name: str
    blocks: tuple[tuple[str, str, int], ...]
    body: tuple
    backend: str = "generic"
    params: tuple[tuple[str, int], ...] = ()

    def param(self, name: str, default: int) -> int:
        for k, v in self.params:
            if k == name:
                return v
        return default


@dataclass(frozen=True)
class Module:
    buffers: tuple[Buffer, ...]
    kernels: tuple[Kernel, ...]
    output: str
    precision: str = "fp32"

    def buffer(self, name: str) -> Buffer:
        for b in self.buffers:
            if b.name == name:
                return b
        raise UnsupportedMA(f"unknown buffer {name!r}")

    def inputs(self) -> list[Buffer]:
        return [b for b in self.buffers if b.is_input]


# ---------------------------------------------------------------------------
# Adapter from live tilecc objects (duck-typed; tilecc is not imported)


def _enum_value(x):
    return getattr(x, "value", x)


def _affine_from_tilecc(offset_expr) -> tuple[Affine, str]:
    """Follows tilecc/exprs.py:228-254 (`to_affine`) on the offset tree."""

    def go(e):
        cls = type(e).__name__
        if cls == "Const":
            v = float(e.value)
            if not v.is_integer():
                raise UnsupportedMA(f"non-integer slice offset constant {v}")
            return {}, int(v)
        if cls == "Var":
            return {e.name: 1}, 0
        if cls == "Un" and e.op == "neg":
            c, k = go(e.x)
            return {n: -v for n, v in c.items()}, -k
        if cls == "Bin":
            ca, ka = go(e.a)
            cb, kb = go(e.b)
            if e.op in ("add", "sub"):
                s = 1 if e.op == "add" else -1
                out = dict(ca)
                for n, v in cb.items():
                    out[n] = out.get(n, 0) + s * v
                return out, ka + s * kb
            if e.op == "mul":
                if not ca:
                    return {n: v * ka for n, v in cb.items()}, kb * ka
                if not cb:
                    return {n: v * kb for n, v in ca.items()}, ka * kb
        raise UnsupportedMA(f"non-affine slice offset {e!r}")

    coefs, const = go(offset_expr)
    return Affine.make(coefs, const), ""


def _slice_from_tilecc(s) -> Slice:
    off, _ = _affine_from_tilecc(s.offset)
    return Slice(off, int(s.length), str(s))


def _expr_from_tilecc(e) -> Expr:
    cls = type(e).__name__
    shape = tuple(int(d) for d in e.shape)
    if cls == "VLit":
        return Lit(shape, float(e.value))
    if cls == "MARef":
        return Ref(shape, e.buffer, tuple(_slice_from_tilecc(s) for s in e.slices))
    if cls == "VBin":
        return Bin(shape, e.op, _expr_from_tilecc(e.a), _expr_from_tilecc(e.b))
    if cls == "VUn":
        return Un(shape, e.op, _expr_from_tilecc(e.x))
    if cls == "VScale":
        return Scale(shape, e.kind, _expr_from_tilecc(e.x))
    if cls == "VDot":
        seed = _expr_from_tilecc(e.seed) if e.seed is not None else None
        return Dot(shape, _expr_from_tilecc(e.a), _expr_from_tilecc(e.b), seed)
    if cls == "VReduce":
        seed = _expr_from_tilecc(e.seed) if e.seed is not None else None
        return Reduce(shape, e.op, _expr_from_tilecc(e.x), tuple(e.axes), seed)
    if cls == "VTranspose":
        return Transpose(shape, _expr_from_tilecc(e.x), tuple(e.perm))
    if cls == "VReshape":
        return Reshape(shape, _expr_from_tilecc(e.x))
    if cls == "VBroadcast":
        return Broadcast(shape, _expr_from_tilecc(e.x))
    raise UnsupportedMA(f"unknown MA expression node {cls}")


def _body_from_tilecc(body) -> tuple:
    out = []
    for st in body:
        cls = type(st).__name__
        if cls == "MALoop":
            out.append(Loop(st.var, int(st.extent), _body_from_tilecc(st.body)))
        elif cls == "MACopy":
            out.append(Copy(st.dst, tuple(_slice_from_tilecc(s) for s in st.dst_slices),
                            st.src, tuple(_slice_from_tilecc(s) for s in st.src_slices)))
        elif cls == "MACompute":
            out.append(Compute(st.dst, tuple(_slice_from_tilecc(s) for s in st.dst_slices),
                               _expr_from_tilecc(st.expr)))
        else:
            raise UnsupportedMA(f"unknown MA statement {cls}")
    return tuple(out)


def from_tilecc(module) -> Module:
    """Convert a tilecc ``MAModule`` (tilecc/ma/ir.py:65-76) into a ``Module``."""
    if isinstance(module, Module):
        return module
    bufs = tuple(
        Buffer(b.name, tuple(int(d) for d in b.shape), _enum_value(b.precision),
               _enum_value(b.scope), bool(b.is_input), bool(b.is_output))
        for b in module.buffers
    )
    kernels = tuple(
        Kernel(k.name, tuple((v, a, int(e)) for v, a, e in k.blocks),
               _body_from_tilecc(k.body), k.backend,
               tuple((n, int(v)) for n, v in k.params))
        for k in module.kernels
    )
    return Module(bufs, kernels, module.output, _enum_value(module.precision))


def as_module(obj) -> Module:
    """Accept a Module, a tilecc MAModule, a JSON string/dict or a path."""
    if isinstance(obj, Module):
        return obj
    if isinstance(obj, (str, bytes)) and str(obj).lstrip().startswith("{"):
        return from_json(obj)
    if isinstance(obj, dict):
        return from_dict(obj)
    if hasattr(obj, "kernels") and hasattr(obj, "buffers"):
        return from_tilecc(obj)
    if isinstance(obj, str):
        with open(obj) as f:
            return from_json(f.read())
    raise UnsupportedMA(f"cannot interpret {type(obj).__name__} as an MA module")


# ---------------------------------------------------------------------------
# JSON (stable; version 1)


def _num(v: float):
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if math.isnan(v):
        return "nan"
    return v


def _unnum(v) -> float:
    if isinstance(v, str):
        return float(v)
    return float(v)


def _slice_to(s: Slice) -> dict:
    return {"coefs": {k: c for k, c in s.off.coefs}, "const": s.off.const,
            "len": s.length, "text": s.text}


def _slice_from(d: dict) -> Slice:
    return Slice(Affine.make(d["coefs"], d["const"]), int(d["len"]), d.get("text", ""))


def _expr_to(e: Expr) -> dict:
    d = {"_t": type(e).__name__, "shape": list(e.shape)}
    if isinstance(e, Lit):
        d["value"] = _num(e.value)
    elif isinstance(e, Ref):
        d["buffer"] = e.buffer
        d["slices"] = [_slice_to(s) for s in e.slices]
    elif isinstance(e, Bin):
        d.update(op=e.op, a=_expr_to(e.a), b=_expr_to(e.b))
    elif isinstance(e, Un):
        d.update(op=e.op, x=_expr_to(e.x))
    elif isinstance(e, Scale):
        d.update(kind=e.kind, x=_expr_to(e.x))
    elif isinstance(e, Dot):
        d.update(a=_expr_to(e.a), b=_expr_to(e.b),
                 seed=_expr_to(e.seed) if e.seed is not None else None)
    elif isinstance(e, Reduce):
        d.update(op=e.op, x=_expr_to(e.x), axes=list(e.axes),
                 seed=_expr_to(e.seed) if e.seed is not None else None)
    elif isinstance(e, Transpose):
        d.update(x=_expr_to(e.x), perm=list(e.perm))
    elif isinstance(e, (Reshape, Broadcast)):
        d.update(x=_expr_to(e.x))
    return d


def _expr_from(d: dict) -> Expr:
    t = d["_t"]
    shape = tuple(d["shape"])
    if t == "Lit":
        return Lit(shape, _unnum(d["value"]))
    if t == "Ref":
        return Ref(shape, d["buffer"], tuple(_slice_from(s) for s in d["slices"]))
    if t == "Bin":
        return Bin(shape, d["op"], _expr_from(d["a"]), _expr_from(d["b"]))
    if t == "Un":
        return Un(shape, d["op"], _expr_from(d["x"]))
    if t == "Scale":
        return Scale(shape, d["kind"], _expr_from(d["x"]))
    if t == "Dot":
        return Dot(shape, _expr_from(d["a"]), _expr_from(d["b"]),
                   _expr_from(d["seed"]) if d.get("seed") else None)
    if t == "Reduce":
        return Reduce(shape, d["op"], _expr_from(d["x"]), tuple(d["axes"]),
                      _expr_from(d["seed"]) if d.get("seed") else None)
    if t == "Transpose":
        return Transpose(shape, _expr_from(d["x"]), tuple(d["perm"]))
    if t == "Reshape":
        return Reshape(shape, _expr_from(d["x"]))
    if t == "Broadcast":
        return Broadcast(shape, _expr_from(d["x"]))
    raise UnsupportedMA(f"unknown expression tag {t!r}")


def _stmt_to(st) -> dict:
    if isinstance(st, Loop):
        return {"_t": "Loop", "var": st.var, "extent": st.extent,
                "body": [_stmt_to(s) for s in st.body]}
    if isinstance(st, Copy):
        return {"_t": "Copy", "dst": st.dst, "dst_slices": [_slice_to(s) for s in st.dst_slices],
                "src": st.src, "src_slices": [_slice_to(s) for s in st.src_slices]}
    return {"_t": "Compute", "dst": st.dst,
            "dst_slices": [_slice_to(s) for s in st.dst_slices], "expr": _expr_to(st.expr)}


def _stmt_from(d: dict):
    t = d["_t"]
    if t == "Loop":
        return Loop(d["var"], int(d["extent"]), tuple(_stmt_from(s) for s in d["body"]))
    if t == "Copy":
        return Copy(d["dst"], tuple(_slice_from(s) for s in d["dst_slices"]),
                    d["src"], tuple(_slice_from(s) for s in d["src_slices"]))
    if t == "Compute":
        return Compute(d["dst"], tuple(_slice_from(s) for s in d["dst_slices"]),
                       _expr_from(d["expr"]))
    raise UnsupportedMA(f"unknown statement tag {t!r}")


def to_dict(m: Module) -> dict:
    return {
        "version": 1,
        "kind": "ma-module",
        "precision": m.precision,
        "output": m.output,
        "buffers": [{"name": b.name, "shape": list(b.shape), "precision": b.precision,
                     "scope": b.scope, "is_input": b.is_input, "is_output": b.is_output}
                    for b in m.buffers],
        "kernels": [{"name": k.name, "blocks": [list(b) for b in k.blocks],
                     "backend": k.backend, "params": [list(p) for p in k.params],
                     "body": [_stmt_to(s) for s in k.body]} for k in m.kernels],
    }


def from_dict(d: dict) -> Module:
    if d.get("kind") != "ma-module" or d.get("version") != 1:
        raise UnsupportedMA("not a version-1 MA module document")
    bufs = tuple(Buffer(b["name"], tuple(b["shape"]), b["precision"], b["scope"],
                        bool(b["is_input"]), bool(b["is_output"])) for b in d["buffers"])
    kernels = tuple(Kernel(k["name"], tuple((v, a, int(e)) for v, a, e in k["blocks"]),
                           tuple(_stmt_from(s) for s in k["body"]), k["backend"],
                           tuple((n, int(v)) for n, v in k["params"])) for k in d["kernels"])
    return Module(bufs, kernels, d["output"], d["precision"])


def to_json(m: Module) -> str:
    return json.dumps(to_dict(m), sort_keys=True, separators=(",", ":"))


def from_json(text) -> Module:
    return from_dict(json.loads(text))


# ---------------------------------------------------------------------------
# Generic text emission (restates tilecc/ma/emit.py:32-147, flavor "generic")

_INFIX = {"add": "+", "sub": "-", "mul": "*", "div": "/"}
_PREC = {"add": 1, "sub": 1, "mul": 2, "div": 2}


def emit_text(m: Module) -> str:
    lines: list[str] = []
    for b in m.buffers:
        if b.scope == "Global":
            shape = ", ".join(str(d) for d in b.shape)
            kind = "in" if b.is_input else ("out" if b.is_output else "tmp")
            lines.append(f"# {kind} {b.name}[{m.precision}]({shape})")
    for k in m.kernels:
        params = " ".join(f"{n}={v}" for n, v in k.params)
        lines.append(f"def {k.name}({params}) [{k.backend}]:")
        for var, axis, extent in k.blocks:
            lines.append(f"  {var} = block(\"{axis}\", 0, {extent})")
        _emit_body(k.body, lines, 1)
    return "\n".join(lines) + "\n"


def _slices_text(slices) -> str:
    return ", ".join(str(s) for s in slices)


def _emit_body(body, lines, depth):
    pad = "  " * depth
    for st in body:
        if isinstance(st, Loop):
            lines.append(f"{pad}for {st.var} in range({st.extent}):")
            _emit_body(st.body, lines, depth + 1)
        elif isinstance(st, Copy):
            lines.append(f"{pad}{st.dst}[{_slices_text(st.dst_slices)}] = "
                         f"{st.src}[{_slices_text(st.src_slices)}]")
        else:
            lines.append(f"{pad}{st.dst}[{_slices_text(st.dst_slices)}] = {_emit_expr(st.expr, 0)}")


def _lit_text(v: float) -> str:
    if v == float("-inf"):
        return "-inf"
    if v == float("inf"):
        return "inf"
    return str(int(v)) if float(v).is_integer() else repr(v)


def _ident_seed(e, op) -> bool:
    if not isinstance(e, Lit):
        return False
    return {"sum": e.value == 0.0, "prod": e.value == 1.0,
            "max": e.value == float("-inf"), "min": e.value == float("inf")}[op]


def _emit_expr(e: Expr, prec: int) -> str:
    if isinstance(e, Lit):
        return f"tile({_lit_text(e.value)}, {list(e.shape)})"
    if isinstance(e, Ref):
        return f"{e.buffer}[{_slices_text(e.slices)}]"
    if isinstance(e, Bin):
        if e.op in ("max", "min"):
            fn = {"max": "maximum", "min": "minimum"}[e.op]
            return f"{fn}({_emit_expr(e.a, 0)}, {_emit_expr(e.b, 0)})"
        mine = _PREC[e.op]
        s = f"{_emit_expr(e.a, mine)} {_INFIX[e.op]} {_emit_expr(e.b, mine + 1)}"
        return f"({s})" if prec > mine else s
    if isinstance(e, Un):
        return f"{e.op}({_emit_expr(e.x, 0)})"
    if isinstance(e, Scale):
        return f"log2e * {_emit_expr(e.x, 3)}"
    if isinstance(e, Dot):
        seed = ""
        if e.seed is not None and not (isinstance(e.seed, Lit) and e.seed.value == 0.0):
            seed = f", acc={_emit_expr(e.seed, 0)}"
        return f"dot({_emit_expr(e.a, 0)}, {_emit_expr(e.b, 0)}{seed})"
    if isinstance(e, Reduce):
        ax = e.axes[0] if len(e.axes) == 1 else list(e.axes)
        seed = ""
        if e.seed is not None and not _ident_seed(e.seed, e.op):
            seed = f", init={_emit_expr(e.seed, 0)}"
        return f"{e.op}({_emit_expr(e.x, 0)}, axis={ax}{seed})"
    if isinstance(e, Transpose):
        if tuple(e.perm) == (1, 0):
            return f"{_emit_expr(e.x, 3)}.T"
        return f"transpose({_emit_expr(e.x, 0)}, {list(e.perm)})"
    if isinstance(e, Reshape):
        return f"reshape({_emit_expr(e.x, 0)}, {list(e.shape)})"
    if isinstance(e, Broadcast):
        return f"broadcast({_emit_expr(e.x, 0)}, {list(e.shape)})"
    raise UnsupportedMA(f"unknown node {type(e).__name__}")
