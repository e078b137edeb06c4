"""Multi-GPU host logic on CPU: world_size-2 gloo, shards + gather == the full oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_14825_b200.shard import plan_shard


def test_plan_shard_partitions_every_group_exactly_once():
    for B, Hkv in [(1, 8), (32, 12), (64, 8), (4, 2)]:
        for world in (1, 2, 4, 8):
            try:
                shards = [plan_shard(B, Hkv, world, r) for r in range(world)]
            except ValueError:
                assert B % world and Hkv % world
                continue
            seen = set()
            for s in shards:
                for b in range(s.b0, s.b1):
                    for h in range(s.h0, s.h1):
                        assert (b, h) not in seen
                        seen.add((b, h))
            assert seen == {(b, h) for b in range(B) for h in range(Hkv)}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, Hq, Hkv, N, D, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import reference_math
    from paper_2604_14825_b200.shard import gather_output, plan_shard

    g = np.random.default_rng(0)
    q = g.standard_normal((B, Hq, N, D))
    k = g.standard_normal((B, Hkv, N, D))
    v = g.standard_normal((B, Hkv, N, D))
    sh = plan_shard(B, Hkv, world, rank)
    qh0, qh1 = sh.q_heads(Hq // Hkv)
    local = reference_math.attention_batched_fp64(q[sh.b0:sh.b1, qh0:qh1], k[sh.b0:sh.b1, sh.h0:sh.h1],
                                                  v[sh.b0:sh.b1, sh.h0:sh.h1], 0.125, True)
    full = gather_output(torch.from_numpy(local), world, sh)
    if rank == 0:
        ref = reference_math.attention_batched_fp64(q, k, v, 0.125, True)
        np.save(out_path, np.abs(full.numpy() - ref).max())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B,Hq,Hkv", [(2, 4, 2), (1, 8, 2)])
def test_gloo_world2_sharded_attention_equals_full(tmp_path, B, Hq, Hkv):
    out = str(tmp_path / "err.npy")
    mp.spawn(_worker, args=(2, _free_port(), B, Hq, Hkv, 64, 16, out), nprocs=2, join=True)
    assert float(np.load(out)) == 0.0


def test_plan_row_shard_covers_rows_in_whole_tiles():
    from paper_2604_14825_b200.shard import plan_row_shard
    for rows in (1, 127, 128, 300, 4096, 4100):
        for world in (1, 2, 3, 4, 8):
            sh = [plan_row_shard(rows, world, r) for r in range(world)]
            assert sh[0].r0 == 0 and sh[-1].r1 == rows
            for a, b in zip(sh, sh[1:]):
                assert a.r1 == b.r0
            for s in sh[:-1]:
                assert s.r0 % 128 == 0 and s.r1 % 128 == 0 or s.r1 == rows
            sizes = [s.r1 - s.r0 for s in sh]
            assert max(sizes) - min(sizes) <= 2 * 128  # whole 128-row tiles, ragged last tile


def _chain_worker(rank, world, port, rows, K, F, E, out_path):
    """Row-sharded (X.W1).W2: each rank its X rows, Y rows gathered."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_14825_b200.shard import gather_rows, plan_row_shard

    g = np.random.default_rng(1)
    x = g.standard_normal((rows, K))
    w1 = g.standard_normal((K, F)) / np.sqrt(K)
    w2 = g.standard_normal((F, E)) / np.sqrt(F)
    sh = plan_row_shard(rows, world, rank)
    local = (x[sh.r0:sh.r1] @ w1) @ w2
    full = gather_rows(torch.from_numpy(local), rows, world)
    if rank == 0:
        np.save(out_path, np.abs(full.numpy() - (x @ w1) @ w2).max() if full.shape == (rows, E) else np.inf)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("rows", [256, 300])
def test_gloo_world2_row_sharded_chain_equals_full(tmp_path, rows):
    out = str(tmp_path / "err.npy")
    mp.spawn(_chain_worker, args=(2, _free_port(), rows, 32, 48, 16, out), nprocs=2, join=True)
    assert float(np.load(out)) < 1e-12
