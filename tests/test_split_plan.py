"""K1 split-KV planning on the host (no GPU): the C planner's workspace size, restated.

The planner (csrc/capi.cu attn_split_plan) cuts few, long attention work items
into KV ranges; the kernel maps a unit index to (item, KV range) through a
prefix table over m-block positions (csrc/attn_fwd.cuh attn_unit).  Restated
here: the workspace size must match the C library's, and the units must cover
every (item, KV tile) exactly once.
"""

import ctypes
import math

import pytest

from paper_2604_14825_b200 import _lib

SMS = 148  # the library's SM count without a device


def _args(B, Hq, Hkv, N, M, D, mask):
    a = _lib.AttnArgs()
    a.batch, a.heads_q, a.heads_kv, a.seq_q, a.seq_kv, a.head_dim = B, Hq, Hkv, N, M, D
    a.mask_kind = mask
    return a


def _rows(B, Hq, N, D=128, M=None):
    """Library choice of query rows per work item (capi.cu attn_item_rows, item_rows = 0)."""
    if D == 64 and M is not None and M <= 1024:
        return 128
    return 128 if (N + 255) // 256 * B * Hq * 2 < SMS else 256


def _nkv(mb, N, M, causal, off=0, rows=256):
    total = (M + 127) // 128
    if not causal:
        return total
    last_q = min(mb * rows + rows - 1, N - 1) + off
    return max(min(total, last_q // 128 + 1), 1)


def _makespan(nk_lpt, BH, s, ctas):
    """Greedy schedule of the units (LPT order) over `ctas` CTAs, one extra step per unit."""
    import heapq
    free = [0.0] * ctas
    end = 0.0
    for n in nk_lpt:
        nc = (n + s - 1) // s if n > s else 1
        for c in range(nc):
            for _ in range(BH):
                t = heapq.heappop(free) + min(s, n - c * s) + 1.0
                heapq.heappush(free, t)
                end = max(end, t)
    return end


def _plan(B, Hq, N, M, D, causal):
    """Restatement of attn_split_plan: (kv_split, n_units, workspace bytes)."""
    rows = _rows(B, Hq, N, D, M)
    nmb = (N + rows - 1) // rows
    BH = B * Hq
    nk = [_nkv(mb, N, M, causal, rows=rows) for mb in range(nmb)]
    total = sum(nk) * BH
    avg = total / (SMS * (2 if rows == 128 else 1))
    mx = max(nk)
    if nmb > 384 or mx <= 2.0 * avg:
        return 0, nmb * BH, 0
    s_min = max(4, (mx + 31) // 32)
    S = max(math.ceil(avg / 0.9), s_min)
    ctas = SMS * (2 if rows == 128 else 1)
    best = None
    for s in range(max(s_min, int(0.8 * avg)), max(s_min, math.ceil(1.3 * avg)) + 1):
        m = _makespan(nk[::-1] if causal else nk, BH, s, ctas)
        if best is None or m < best - 1e-9:
            best, S = m, s
    if S >= mx:
        return 0, nmb * BH, 0
    units = sum((n + S - 1) // S for n in nk) * BH
    prefix = ((nmb + 1) * 4 + 255) // 256 * 256
    ml = (units * rows * 8 + 255) // 256 * 256
    return S, units, prefix + ml + units * rows * D * 2  # bf16 partials


def _units(B, Hq, N, M, causal, S, D=128):
    """Restatement of the kernel's unit map: unit -> (b*Hq + hq, m-block, first tile, tiles)."""
    rows = _rows(B, Hq, N, D, M)
    nmb = (N + rows - 1) // rows
    BH = B * Hq
    prefix = [0]
    for i in range(nmb):
        mb = nmb - 1 - i if causal else i
        prefix.append(prefix[-1] + (_nkv(mb, N, M, causal, rows=rows) + S - 1) // S * BH)
    out = []
    for w in range(prefix[-1]):
        lo = max(i for i in range(nmb) if prefix[i] <= w)
        r = w - prefix[lo]
        c, bh = divmod(r, BH)
        mb = nmb - 1 - lo if causal else lo
        n_full = _nkv(mb, N, M, causal, rows=rows)
        out.append((bh, mb, c * S, min(S, n_full - c * S)))
    return out


@pytest.mark.parametrize("B,Hq,Hkv,N,M,D,causal", [
    (1, 4, 1, 8192, 8192, 128, True),     # one kv-group at 8K: split
    (1, 32, 8, 8192, 8192, 128, True),    # the full headline grid: never split
    (1, 2, 2, 4096, 4096, 128, False),    # few long non-causal items: split
    (1, 2, 1, 3000, 3000, 64, True),
    (2, 1, 1, 2048, 5000, 64, False),
    (32, 12, 12, 512, 512, 64, False),    # BERT: not split
    (1, 1, 1, 256, 256, 64, False),       # attn256: one item, nothing to gain
])
def test_split_plan_matches_library_and_covers_every_tile(B, Hq, Hkv, N, M, D, causal):
    mask = _lib.NT_MASK_CAUSAL if causal else _lib.NT_MASK_NONE
    got = int(_lib.lib().nt_attn_workspace_bytes(ctypes.byref(_args(B, Hq, Hkv, N, M, D, mask))))
    S, units, bytes_ = _plan(B, Hq, N, M, D, causal)
    assert got == bytes_
    if S == 0:
        return
    cover = {}
    for bh, mb, lo, n in _units(B, Hq, N, M, causal, S, D):
        assert 1 <= n <= S
        for j in range(lo, lo + n):
            cover[(bh, mb, j)] = cover.get((bh, mb, j), 0) + 1
    rows = _rows(B, Hq, N, D, M)
    nmb = (N + rows - 1) // rows
    want = {(bh, mb, j) for bh in range(B * Hq) for mb in range(nmb)
            for j in range(_nkv(mb, N, M, causal, rows=rows))}
    assert set(cover) == want and all(v == 1 for v in cover.values())
    assert len(_units(B, Hq, N, M, causal, S, D)) == units


def test_tensor_masks_are_never_split():
    a = _args(1, 1, 1, 4096, 4096, 64, _lib.NT_MASK_TENSOR)
    assert int(_lib.lib().nt_attn_workspace_bytes(ctypes.byref(a))) == 0
