"""Batch x head sharding of the operator over GPUs (north-star subsystem 4).

The compiled unit is the 2-D single-head MA program (the reference cannot
express heads/GQA at realistic sizes), so multi-GPU execution
partitions the runtime's outer grid: independent (batch, kv-head) groups --
a GQA group keeps its q-heads and their shared K/V on one rank, so every rank
reads only its own K/V.  There is no data-path collective; NCCL is used only
to gather the outputs.  One process per GPU.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    b0: int
    b1: int
    h0: int  # kv-head range
    h1: int
    axis: str  # "batch" | "kv_head" | "none"

    def q_heads(self, q_per_kv: int) -> tuple[int, int]:
        return self.h0 * q_per_kv, self.h1 * q_per_kv


def plan_shard(batch: int, heads_kv: int, world: int, rank: int) -> Shard:
    """Contiguous equal split of the (batch, kv-head) groups: batch first, else kv heads."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if world == 1:
        return Shard(0, batch, 0, heads_kv, "none")
    if batch % world == 0:
        n = batch // world
        return Shard(rank * n, (rank + 1) * n, 0, heads_kv, "batch")
    if heads_kv % world == 0:
        n = heads_kv // world
        return Shard(0, batch, rank * n, (rank + 1) * n, "kv_head")
    raise ValueError(f"cannot split batch={batch} x kv_heads={heads_kv} evenly over {world} ranks")


@dataclass(frozen=True)
class RowShard:
    r0: int
    r1: int


def plan_row_shard(rows: int, world: int, rank: int, align: int = 128) -> RowShard:
    """Rows of X (and Y) of the GEMM chain for this rank.

    The MA's block variable i0 walks row tiles of X independently (Appendix B.4),
    so a rank owns a contiguous run of whole row tiles: ``align``-row units split
    as evenly as possible, the first ``units % world`` ranks taking one extra.
    W1 and W2 are replicated; Y rows are all-gathered.
    """
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    units = -(-rows // align)
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return RowShard(min(rows, u0 * align), min(rows, u1 * align))


def gather_rows(local, rows: int, world: int, dist=None, group=None, align: int = 128):
    """All-gather per-rank Y row blocks (uneven shards padded to the largest) into [rows, E]."""
    import torch

    if world == 1:
        return local
    if dist is None:
        import torch.distributed as dist
    shards = [plan_row_shard(rows, world, r, align) for r in range(world)]
    cap = max(s.r1 - s.r0 for s in shards)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    stacked = torch.empty((world,) + tuple(pad.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(stacked, pad, group=group)
    else:
        parts = list(stacked.unbind(0))
        dist.all_gather(parts, pad, group=group)
        stacked = torch.stack(parts, 0)
    return torch.cat([stacked[r, : s.r1 - s.r0] for r, s in enumerate(shards)], 0)


def gather_output(local, world: int, shard: Shard, dist=None, group=None):
    """All-gather per-rank O shards [b, hq, n, d] into the full [B, Hq, N, D] tensor.

    With NCCL this is one all_gather_into_tensor over NVLink; the result is
    re-assembled along the sharded axis (batch or heads).
    """
    import torch

    if world == 1:
        return local
    if dist is None:
        import torch.distributed as dist
    local = local.contiguous()
    stacked = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(stacked, local, group=group)
    else:
        parts = list(stacked.unbind(0))
        dist.all_gather(parts, local, group=group)
        stacked = torch.stack(parts, 0)
    return assemble(stacked, shard.axis)


def assemble(stacked, axis: str):
    """[world, b, hq, n, d] per-rank O shards (rank order) -> the full [B, Hq, N, D] tensor."""
    world, b, hq = stacked.shape[:3]
    if axis in ("batch", "none"):
        return stacked.reshape((world * b,) + tuple(stacked.shape[2:]))
    # kv_head: [world, B, hq_local, N, D] -> [B, world * hq_local, N, D]
    return stacked.permute(1, 0, 2, 3, 4).reshape(b, world * hq, *stacked.shape[3:])


def assemble_rows(parts, rows: int, align: int = 128):
    """Per-rank Y row blocks (rank order, unpadded) -> [rows, E]; checks the row plan."""
    import torch

    world = len(parts)
    for r, p in enumerate(parts):
        s = plan_row_shard(rows, world, r, align)
        if p.shape[0] != s.r1 - s.r0:
            raise ValueError(f"rank {r}: {p.shape[0]} rows, plan says {s.r1 - s.r0}")
    return torch.cat(list(parts), 0)
