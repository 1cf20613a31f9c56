"""Head sharding: partition math and the optional all-gather, on CPU with the
gloo backend at world_size 2 (the CUDA operator is replaced by a head-local GQA stand-in, so
this checks exactly the host logic the multi-GPU path adds)."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_22575_b200.shard import head_shard, sharded_attention


def test_head_shard_partition():
    for world in (1, 2, 4, 8):
        shards = [head_shard(32, 8, world, r) for r in range(world)]
        assert [s.q_lo for s in shards] == [r * 32 // world for r in range(world)]
        assert shards[-1].q_hi == 32 and shards[-1].kv_hi == 8
        for s in shards:
            assert s.hq == 4 * s.hkv  # whole GQA groups
            assert s.q_lo == 4 * s.kv_lo
    with pytest.raises(ValueError):
        head_shard(32, 8, 3, 0)
    with pytest.raises(ValueError):
        head_shard(30, 8, 2, 0)


def fake_op(q, k, v, cfg):
    """Head-local stand-in for s2o_attention: out[:, h] = q[:, h] * 2 + v[:, h // group]."""
    group = q.shape[1] // k.shape[1]
    return q * 2 + v.repeat_interleave(group, dim=1)


def _worker(rank, world, port, q, k, v, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = sharded_attention(q, k, v, None, world, rank, allgather=False, op=fake_op)
        full = sharded_attention(q, k, v, None, world, rank, allgather=True, op=fake_op)
        result[rank] = (local.clone(), full.contiguous().clone())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("z", [1, 2])
def test_sharded_allgather_world2(z):
    torch.manual_seed(0)
    q = torch.randn(z, 8, 16, 4)
    k = torch.randn(z, 2, 16, 4)
    v = torch.randn(z, 2, 16, 4)
    want = fake_op(q, k, v, None)
    world = 2
    with mp.Manager() as mgr:
        result = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), q, k, v, result), nprocs=world, join=True)
        res = dict(result)
    for r in range(world):
        local, full = res[r]
        s = head_shard(8, 2, world, r)
        torch.testing.assert_close(local, want[:, s.q_lo:s.q_hi], rtol=0, atol=0)
        torch.testing.assert_close(full, want, rtol=0, atol=0)
