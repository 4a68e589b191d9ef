"""Sharding and the deterministic NCCL-style norm, exercised with gloo on CPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_11665_b200 import shard


def test_shard_range_covers_everything():
    for total in (1, 7, 4096, 2**21):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                e0, c = shard.shard_range(total, r, world)
                seen.append((e0, c))
            assert seen[0][0] == 0
            for (a, ca), (b, _) in zip(seen, seen[1:]):
                assert a + ca == b
            assert seen[-1][0] + seen[-1][1] == total


def test_tree_sum_matches_definition():
    x = np.random.default_rng(0).standard_normal(64)
    t = torch.from_numpy(x)
    ref = x.copy()
    while ref.size > 1:
        ref = ref[0::2] + ref[1::2]
    assert shard.tree_sum(t).item() == ref[0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, block, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(123)
    sumsq_all = torch.from_numpy(rng.uniform(0, 1, total))
    e0, cnt = shard.shard_range(total, rank, world)
    local = sumsq_all[e0:e0 + cnt].contiguous()
    det = shard.global_norm(local, block=block)
    red = shard.global_norm(local, block=block, allreduce=True)
    if rank == 0:
        out.put((det, red))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_global_norm_is_world_size_invariant(world):
    total, block = 4096 * 8, 4096
    ref = shard.global_norm(torch.from_numpy(np.random.default_rng(123).uniform(0, 1, total)),
                            block=block)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), total, block, q), nprocs=world, join=True)
    det, red = q.get()
    assert det == ref  # bitwise: fixed block partials + fixed global tree
    assert abs(red - ref) <= 1e-14 * ref


def test_job_block_and_block_shard():
    assert shard.job_block(2**21) == 4096
    assert shard.job_block(3 * 1024) == 1024
    assert shard.job_block(7) == 1
    for total, world in ((2**21, 3), (2**21, 6), (4096 * 5, 4), (12, 8)):
        b = shard.job_block(total)
        spans = [shard.block_shard(total, r, world, b) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][0] + spans[-1][1] == total
        for (a, ca), (c, _) in zip(spans, spans[1:]):
            assert a + ca == c and a % b == 0 and ca % b == 0


def _worker_uneven(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = torch.from_numpy(np.random.default_rng(7).uniform(0, 1, total))
    block = shard.job_block(total)
    e0, cnt = shard.block_shard(total, rank, world, block)
    local = x[e0:e0 + cnt].contiguous()
    a = float(shard.global_norm_tensor(local, block=block, total=total))
    b = shard.global_norm(local, block=block)  # counts exchanged instead of derived
    if rank == 0:
        out.put((a, b))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_global_norm_uneven_block_shards(world):
    # 5 blocks of 1024 over 2 or 3 ranks: unequal block counts per rank
    total = 5 * 1024
    ref = shard.global_norm(torch.from_numpy(np.random.default_rng(7).uniform(0, 1, total)),
                            block=shard.job_block(total))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_worker_uneven, args=(world, _free_port(), total, q), nprocs=world, join=True)
    a, b = q.get()
    assert a == ref and b == ref
