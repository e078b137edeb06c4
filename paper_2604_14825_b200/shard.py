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
    if shard.axis == "batch":
        return stacked.reshape((world * local.shape[0],) + tuple(local.shape[1:]))
    # kv_head: [world, B, hq_local, N, D] -> [B, world * hq_local, N, D]
    return stacked.permute(1, 0, 2, 3, 4).reshape(local.shape[0], world * local.shape[1], *local.shape[2:])
