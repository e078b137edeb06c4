"""MA kernel -> typed KernelSpec (the front half of the MA -> sm_100a lowering).

The reference lowers VR to MA in ``lower_to_ma`` (tilecc/ma/lower.py:64-190)
and executes it with ``interpret_ma`` (tilecc/ma/interp.py:102-280).  The B200
backend instead *recognises* each ``MAKernel`` as an instance of a kernel
family with a hand-written sm_100a template and extracts every number the
template needs (tile sizes, head dim, scale constant, mask source, buffer
roles, warps/stages).  Unrecognised programs raise ``UnsupportedMA`` -- there
is no CPU fallback.

Recognition is semantic, not textual: the kernel body is evaluated
symbolically (a term algebra over input tiles, literals and the ops of
tilecc/vr/ir.py), carried accumulators (``*_acc`` register buffers, and
Global read-modify-write accumulators such as the GEMM chain's Y) are turned
into ``carry`` terms, and the resulting per-iteration update terms are matched
against the algebra each family computes.  That covers every structural
variant the auto-scheduler emits (staged or
unstaged operands, the scale applied to K, the mask added twice, dead
register copies) with one matcher per family.

Index math is checked exactly: every slice offset must be the affine form
``t * var`` (coefficient equal to the slice length, constant 0) over the block
or loop variable, and block/loop extents times tile must cover the buffer.
The GPU kernels' tiles are unions of consecutive MA tiles (see
``AttentionSpec.gpu_tiles``), visited in the MA's ascending order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

from . import ma_ir as ir
from .errors import UnsupportedMA

# ---------------------------------------------------------------------------
# Symbolic terms (hashable tuples)
#   ("tile", buf, ((coefs, const, len), ...))      Global input tile
#   ("lit", value)                                 literal tile (shape dropped)
#   ("bin", op, a, b) ("un", op, x) ("scale", x)
#   ("dot", a, b, seed|None) ("red", op, x, axes, seed|None)
#   ("T", x) ("reshape", x) ("bcast", x)
#   ("carry", buf)  value of a carried buffer at the top of a loop iteration
#   ("final", buf)  value of a carried buffer after the loop


def _sl(s: ir.Slice):
    return (s.off.coefs, s.off.const, s.length)


class _Sym:
    def __init__(self, module: ir.Module, kernel: ir.Kernel):
        self.m = module
        self.k = kernel
        self.scope = {b.name: b.scope for b in module.buffers}
        self.inputs = {b.name for b in module.buffers if b.is_input}
        self.shape = {b.name: tuple(b.shape) for b in module.buffers}

    def read(self, env, buf, slices):
        if buf in self.inputs:
            return ("tile", buf, tuple(_sl(s) for s in slices))
        if buf not in env:
            raise UnsupportedMA(f"read of {buf!r} before any write")
        val, wslices = env[buf]
        if self.scope[buf] != "Global":
            full = tuple(((), 0, d) for d in self.shape[buf])
            got = tuple(_sl(s) for s in slices)
            if got != full:
                raise UnsupportedMA(f"partial access of local buffer {buf!r}")
        elif tuple(_sl(s) for s in slices) != wslices:
            raise UnsupportedMA(f"read of {buf!r} at a different slice than written")
        return val

    def expr(self, env, e):
        if isinstance(e, ir.Lit):
            return ("lit", float(e.value))
        if isinstance(e, ir.Ref):
            return self.read(env, e.buffer, e.slices)
        if isinstance(e, ir.Bin):
            return ("bin", e.op, self.expr(env, e.a), self.expr(env, e.b))
        if isinstance(e, ir.Un):
            return ("un", e.op, self.expr(env, e.x))
        if isinstance(e, ir.Scale):
            if e.kind != "log2e":
                raise UnsupportedMA(f"scale kind {e.kind!r}")
            return ("scale", self.expr(env, e.x))
        if isinstance(e, ir.Dot):
            seed = self.expr(env, e.seed) if e.seed is not None else None
            if seed == ("lit", 0.0):
                seed = None
            return ("dot", self.expr(env, e.a), self.expr(env, e.b), seed)
        if isinstance(e, ir.Reduce):
            seed = self.expr(env, e.seed) if e.seed is not None else None
            return ("red", e.op, self.expr(env, e.x), tuple(e.axes), seed)
        if isinstance(e, ir.Transpose):
            if tuple(e.perm) != (1, 0):
                raise UnsupportedMA("non-2D transpose")
            return ("T", self.expr(env, e.x))
        if isinstance(e, ir.Reshape):
            return ("reshape", self.expr(env, e.x))
        if isinstance(e, ir.Broadcast):
            return ("bcast", self.expr(env, e.x))
        raise UnsupportedMA(f"node {type(e).__name__}")

    def run(self):
        """Returns (pre_env, loop or None, updates, post_env, stores)."""
        env: dict = {}
        loop = None
        updates: dict = {}
        stores: list = []
        body = self.k.body
        loops = [st for st in body if isinstance(st, ir.Loop)]
        if len(loops) > 1:
            raise UnsupportedMA("more than one sequential loop")
        pre_env = None
        for st in body:
            if isinstance(st, ir.Loop):
                loop = st
                if any(isinstance(x, ir.Loop) for x in st.body):
                    raise UnsupportedMA("nested sequential loops")
                pre_env = dict(env)
                written_in_loop = set()
                read_before_write = set()
                for x in st.body:
                    reads = []
                    if isinstance(x, ir.Copy):
                        reads = [x.src]
                    else:
                        reads = [n.buffer for n in x.expr.walk() if isinstance(n, ir.Ref)]
                    for r in reads:
                        if r not in written_in_loop and r not in self.inputs:
                            read_before_write.add(r)
                    written_in_loop.add(x.dst)
                carried = {b for b in read_before_write if b in written_in_loop}
                lenv = dict(env)
                for b in carried:
                    lenv[b] = (("carry", b), env[b][1] if b in env else None)
                for x in st.body:
                    self._stmt(lenv, x, stores=None)
                for b in carried:
                    updates[b] = lenv[b][0]
                self.carried = carried
                # after the loop: carried buffers hold their final value, per-iteration
                # temporaries are not observable any more
                env = {b: v for b, v in env.items()}
                for b in written_in_loop:
                    if b in carried:
                        env[b] = (("final", b), lenv[b][1])
                    else:
                        env[b] = (("last", b), lenv[b][1])
                continue
            self._stmt(env, st, stores)
        if loop is None:
            pre_env = env
            self.carried = set()
        return pre_env, loop, updates, env, stores

    def _stmt(self, env, st, stores):
        if isinstance(st, ir.Copy):
            val = self.read(env, st.src, st.src_slices)
        else:
            val = self.expr(env, st.expr)
        wsl = tuple(_sl(s) for s in st.dst_slices)
        env[st.dst] = (val, wsl)
        if stores is not None and self.scope[st.dst] == "Global":
            stores.append((st.dst, wsl, val))


# ---------------------------------------------------------------------------
# Specs


@dataclass(frozen=True)
class AttentionSpec:
    """softmax(Q (K c)^T [+ Mask]) V realised as the rolling-update MA kernel."""

    q: str
    k: str
    v: str
    o: str
    mask: Optional[str]
    n: int  # query rows (MA buffer extent)
    m: int  # key rows
    d: int  # head dim (QK reduction = PV output)
    dv: int
    block_m: int  # t0_i: MA block rows
    block_n: int  # t0_j: MA KV tile
    n_blocks: int
    n_iters: int
    block_var: str
    loop_var: str
    scale: Optional[float]  # c of K_s * c (None when the program has no scale)
    warps: int
    stages: int
    backend: str
    kind: str = "attention"

    # GPU realisation: 256-row work items (two 128-row tiles) -- or 128-row items
    # for small MA query tiles (attn_item_rows) -- x 128-row KV tiles
    GPU_BN = 128

    @property
    def gpu_bm(self) -> int:
        """Rows per GPU work item for the single-head MA program (outer grid 1)."""
        return attn_effective_rows(attn_item_rows(self.block_m), self.n, 1, d=self.d, m=self.m)

    def flops(self, causal: bool = False) -> float:
        """Megatron/FA convention: the two GEMMs only."""
        if causal:
            return 2.0 * self.d * self.n * (self.n + 1) if self.n == self.m else 4.0 * self.n * self.m * self.d / 2
        return 4.0 * self.n * self.m * self.d

    def gpu_tiles(self):
        """Exact map GPU tile -> the MA tiles it covers (index-math parity).

        Yields (cta, [MA block values], kv_tile, [MA loop values]) so tests can
        check that the union of the MA slices equals each GPU tile and that
        iteration order is ascending as in the MA's sequential loop.
        """
        bm = self.gpu_bm
        n_cta = math.ceil(self.n / bm)
        n_kv = math.ceil(self.m / self.GPU_BN)
        for c in range(n_cta):
            rows = (c * bm, min(self.n, (c + 1) * bm))
            blocks = [i for i in range(self.n_blocks)
                      if rows[0] <= i * self.block_m < rows[1]]
            for j in range(n_kv):
                cols = (j * self.GPU_BN, min(self.m, (j + 1) * self.GPU_BN))
                iters = [t for t in range(self.n_iters) if cols[0] <= t * self.block_n < cols[1]]
                yield c, blocks, j, iters


def attn_item_rows(ma_block_rows: int) -> int:
    """K1 query rows per work item requested for the MA's query tile t0_i (the
    scheduler's `t0_i` tunable, tilecc/autosched/scheduler.py:116-124): small MA tiles
    (t0_i <= 32) -> 128-row items (one query tile per CTA, two CTAs per SM);
    otherwise 0 = the library's choice (attn_effective_rows).  Both realise the same
    MA blocks exactly (unions of consecutive MA row tiles)."""
    return 128 if 0 < ma_block_rows <= 32 else 0


def attn_effective_rows(requested: int, n: int, batch_heads: int, sms: int = 148, d: int = 128,
                        m: Optional[int] = None) -> int:
    """The rows nt_attn_fwd uses (csrc/capi.cu attn_item_rows): an explicit 128/256,
    else 128 when 256-row items would leave more than half of the SMs idle or at
    head_dim 64 with <= 1024 keys (short items), else 256."""
    if requested in (128, 256):
        return requested
    if d == 64 and m is not None and m <= 1024:
        return 128
    return 128 if -(-n // 256) * batch_heads * 2 < sms else 256


@dataclass(frozen=True)
class GemmChainSpec:
    """Y = (X . W1) . W2 fused per row block."""

    x: str
    w1: str
    w2: str
    y: str
    n: int
    k: int
    f: int
    e: int
    block_m: int  # t0_i
    block_f: int  # F tile per loop iteration
    n_blocks: int
    n_iters: int
    warps: int
    stages: int
    backend: str
    kind: str = "gemm_chain"

    def flops(self) -> float:
        return 2.0 * self.n * self.k * self.f + 2.0 * self.n * self.f * self.e


# ---------------------------------------------------------------------------
# Matchers


def _is_tile(t, buf=None):
    return isinstance(t, tuple) and t and t[0] == "tile" and (buf is None or t[1] == buf)


def _tile_axis(t, axis):
    coefs, const, length = t[2][axis]
    return dict(coefs), const, length


def _check_dense(t, axis, var, length, extent, total, what):
    """Slice offset along `axis` must be `length * var` and cover `total` rows."""
    coefs, const, ln = _tile_axis(t, axis)
    if ln != length:
        raise UnsupportedMA(f"{what}: slice length {ln} != tile {length}")
    if var is None:
        if coefs or const != 0 or ln != total:
            raise UnsupportedMA(f"{what}: expected the full extent 0:{total}")
        return
    if const != 0 or set(coefs) != {var} or coefs[var] != length:
        raise UnsupportedMA(f"{what}: offset is not {length} * {var}")
    if extent * length != total:
        raise UnsupportedMA(f"{what}: {extent} x {length} does not cover {total}")


def _strip_scale(kt):
    """K tile possibly multiplied by a literal scale tile: returns (tile, c|None)."""
    if _is_tile(kt):
        return kt, None
    if kt[0] == "bin" and kt[1] == "mul":
        a, b = kt[2], kt[3]
        if _is_tile(a) and b[0] == "lit":
            return a, b[1]
        if _is_tile(b) and a[0] == "lit":
            return b, a[1]
    raise UnsupportedMA("K operand is not a (scaled) input tile")


def _rowbcast(t):
    if t[0] == "bcast" and t[1][0] == "reshape":
        return t[1][1]
    return None


def recognize_attention(module: ir.Module, kernel: ir.Kernel, sym: _Sym, pre, loop, upd, post, stores):
    if loop is None or len(sym.carried) < 3:
        raise UnsupportedMA("not an attention kernel (needs 3 carried accumulators)")
    # identify m (init -inf), l (init 0, 1-D), O (init 0, 2-D)
    m_acc = l_acc = o_acc = None
    for b in sym.carried:
        init = pre.get(b, (None,))[0]
        nd = len(sym.shape[b])
        if init == ("lit", float("-inf")) and nd == 1:
            m_acc = b
        elif init == ("lit", 0.0) and nd == 1:
            l_acc = b
        elif init == ("lit", 0.0) and nd == 2:
            o_acc = b
    if not (m_acc and l_acc and o_acc):
        raise UnsupportedMA("carried accumulators are not (m=-inf, l=0, O=0)")
    m_new = upd[m_acc]
    if not (m_new[0] == "red" and m_new[1] == "max" and m_new[3] == (1,) and m_new[4] == ("carry", m_acc)):
        raise UnsupportedMA("m update is not max(S', axis=1, init=m)")
    s_masked = m_new[2]
    mask_tile = None
    s = s_masked
    if s[0] == "bin" and s[1] == "add" and _is_tile(s[3]):
        s, mask_tile = s[2], s[3]
    # S = dot(...) * c: the post-sum scale spelling (schedulable with upstream.apply())
    post_scale = None
    if s[0] == "bin" and s[1] == "mul":
        if s[2][0] == "dot" and s[3][0] == "lit":
            s, post_scale = s[2], s[3][1]
        elif s[3][0] == "dot" and s[2][0] == "lit":
            s, post_scale = s[3], s[2][1]
    if s[0] != "dot" or s[3] is not None or s[2][0] != "T":
        raise UnsupportedMA("S is not dot(Q, K^T)")
    q_tile = s[1]
    k_tile, scale = _strip_scale(s[2][1])
    if post_scale is not None:
        scale = post_scale if scale is None else scale * post_scale
    if not _is_tile(q_tile):
        raise UnsupportedMA("Q operand is not an input tile")
    alpha = ("un", "exp2", ("scale", ("bin", "sub", ("carry", m_acc), m_new)))
    p_term = ("un", "exp2", ("scale", ("bin", "sub", s_masked, ("bcast", ("reshape", m_new)))))
    l_new = upd[l_acc]
    if l_new != ("red", "sum", p_term, (1,), ("bin", "mul", ("carry", l_acc), alpha)):
        raise UnsupportedMA("l update is not sum(P, init=l*alpha)")
    o_new = upd[o_acc]
    if not (o_new[0] == "dot" and o_new[1] == p_term and
            o_new[3] == ("bin", "mul", ("carry", o_acc), ("bcast", ("reshape", alpha)))):
        raise UnsupportedMA("O update is not dot(P, V, acc=O*alpha)")
    v_tile = o_new[2]
    if not _is_tile(v_tile):
        raise UnsupportedMA("V operand is not an input tile")
    # final store: O[...] = final(O) / bcast(reshape(final(l)))
    outs = [(b, w, v) for b, w, v in stores if b == module.output]
    if len(outs) != 1:
        raise UnsupportedMA("expected exactly one store of the output")
    _, o_slices, o_val = outs[0]
    if o_val != ("bin", "div", ("final", o_acc), ("bcast", ("reshape", ("final", l_acc)))):
        raise UnsupportedMA("epilogue is not O / l")

    # ---- index math
    if len(kernel.blocks) != 1:
        raise UnsupportedMA("attention kernel must have one block axis (runtime adds batch x head)")
    bvar, _axis, n_blocks = kernel.blocks[0]
    lvar, n_iters = loop.var, loop.extent
    q_buf, k_buf, v_buf = q_tile[1], k_tile[1], v_tile[1]
    n, d = sym.shape[q_buf]
    m, dk = sym.shape[k_buf]
    mv, dv = sym.shape[v_buf]
    if dk != d or mv != m:
        raise UnsupportedMA("Q/K/V shapes inconsistent")
    bm = _tile_axis(q_tile, 0)[2]
    bn = _tile_axis(k_tile, 0)[2]
    _check_dense(q_tile, 0, bvar, bm, n_blocks, n, "Q rows")
    _check_dense(q_tile, 1, None, d, 1, d, "Q cols")
    _check_dense(k_tile, 0, lvar, bn, n_iters, m, "K rows")
    _check_dense(k_tile, 1, None, d, 1, d, "K cols")
    _check_dense(v_tile, 0, lvar, bn, n_iters, m, "V rows")
    _check_dense(v_tile, 1, None, dv, 1, dv, "V cols")
    o_t = ("tile", module.output, o_slices)
    _check_dense(o_t, 0, bvar, bm, n_blocks, n, "O rows")
    _check_dense(o_t, 1, None, dv, 1, dv, "O cols")
    mask_buf = None
    if mask_tile is not None:
        mask_buf = mask_tile[1]
        if sym.shape[mask_buf] != (n, m):
            raise UnsupportedMA("Mask must be [N, M]")
        _check_dense(mask_tile, 0, bvar, bm, n_blocks, n, "Mask rows")
        _check_dense(mask_tile, 1, lvar, bn, n_iters, m, "Mask cols")
    if dv != d:
        raise UnsupportedMA("value head dim must equal the QK head dim")
    return AttentionSpec(q=q_buf, k=k_buf, v=v_buf, o=module.output, mask=mask_buf, n=n, m=m, d=d,
                         dv=dv, block_m=bm, block_n=bn, n_blocks=n_blocks, n_iters=n_iters,
                         block_var=bvar, loop_var=lvar, scale=scale,
                         warps=kernel.param("warps", 4), stages=kernel.param("stages", 2),
                         backend=kernel.backend)


def recognize_gemm_chain(module: ir.Module, kernel: ir.Kernel, sym: _Sym, pre, loop, upd, post, stores):
    if loop is None:
        raise UnsupportedMA("not a GEMM chain (no sequential loop)")
    y = module.output
    if y not in sym.carried:
        raise UnsupportedMA("output is not a loop-carried accumulator")
    if pre.get(y, (None,))[0] != ("lit", 0.0):
        raise UnsupportedMA("Y accumulator is not zero-initialised")
    y_new = upd[y]
    if not (y_new[0] == "dot" and y_new[3] == ("carry", y)):
        raise UnsupportedMA("Y update is not dot(T, W2, acc=Y)")
    t_term, w2_tile = y_new[1], y_new[2]
    if not (t_term[0] == "dot" and t_term[3] is None and _is_tile(t_term[1]) and _is_tile(t_term[2])):
        raise UnsupportedMA("T is not dot(X, W1)")
    x_tile, w1_tile = t_term[1], t_term[2]
    if not _is_tile(w2_tile):
        raise UnsupportedMA("W2 operand is not an input tile")
    # the last Global value of Y must be the final accumulator
    if post.get(y, (None,))[0] != ("final", y):
        raise UnsupportedMA("Y is not written back every iteration")
    bvar, _axis, n_blocks = kernel.blocks[0]
    lvar, n_iters = loop.var, loop.extent
    n, k = sym.shape[x_tile[1]]
    k2, f = sym.shape[w1_tile[1]]
    f2, e = sym.shape[w2_tile[1]]
    if k2 != k or f2 != f or sym.shape[y] != (n, e):
        raise UnsupportedMA("GEMM chain shapes inconsistent")
    bm = _tile_axis(x_tile, 0)[2]
    bf = _tile_axis(w1_tile, 1)[2]
    _check_dense(x_tile, 0, bvar, bm, n_blocks, n, "X rows")
    _check_dense(x_tile, 1, None, k, 1, k, "X cols")
    _check_dense(w1_tile, 0, None, k, 1, k, "W1 rows")
    _check_dense(w1_tile, 1, lvar, bf, n_iters, f, "W1 cols")
    _check_dense(w2_tile, 0, lvar, bf, n_iters, f, "W2 rows")
    _check_dense(w2_tile, 1, None, e, 1, e, "W2 cols")
    return GemmChainSpec(x=x_tile[1], w1=w1_tile[1], w2=w2_tile[1], y=y, n=n, k=k, f=f, e=e,
                         block_m=bm, block_f=bf, n_blocks=n_blocks, n_iters=n_iters,
                         warps=kernel.param("warps", 4), stages=kernel.param("stages", 2),
                         backend=kernel.backend)


FAMILIES = (recognize_attention, recognize_gemm_chain)


def recognize_kernel(module, kernel):
    sym = _Sym(module, kernel)
    pre, loop, upd, post, stores = sym.run()
    errors = []
    for fam in FAMILIES:
        try:
            return fam(module, kernel, sym, pre, loop, upd, post, stores)
        except UnsupportedMA as e:
            errors.append(f"{fam.__name__}: {e}")
    raise UnsupportedMA(f"kernel {kernel.name!r} matches no sm_100a family: " + "; ".join(errors))


def recognize(module) -> list:
    """Recognise every kernel of an MA module (tilecc MAModule, Module or JSON)."""
    module = ir.as_module(module)
    if module.precision not in ("fp32",):
        raise UnsupportedMA(f"precision {module.precision!r} has no device realisation "
                            "(bf16 operands, fp32 accumulation)")
    return [recognize_kernel(module, k) for k in module.kernels]
