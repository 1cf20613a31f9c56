"""Multi-GPU head sharding for the S2O operator.

Every (q head, segment, query tile) of S2O is independent and plans are per q head, so heads
partition across ranks with no exchange on the data path. Rank r of `world` owns a contiguous
range of whole GQA groups: kv heads [r*Hkv/world, (r+1)*Hkv/world) and the q heads that read
them. The only collective is the optional all-gather that returns the full output to every
rank (NCCL all_gather_into_tensor over NVLink on B200; gloo in the CPU tests).

The reference has no multi-device code (its parallelism is a std::thread fork over (z, h)
slices, proj/src/parallel.cpp:25-66); this module is the B200 counterpart of that fork.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_lo: int
    kv_hi: int
    q_lo: int
    q_hi: int

    @property
    def hkv(self) -> int:
        return self.kv_hi - self.kv_lo

    @property
    def hq(self) -> int:
        return self.q_hi - self.q_lo


def head_shard(hq: int, hkv: int, world: int, rank: int) -> HeadShard:
    """Contiguous GQA-group partition of the heads for `rank` (whole groups per rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must satisfy 0 <= rank < world")
    if hq % hkv != 0:
        raise ValueError("Q/K/V dims must match")
    if hkv % world != 0:
        raise ValueError(f"{hkv} kv heads do not split evenly over {world} ranks")
    group = hq // hkv
    per = hkv // world
    kv_lo, kv_hi = rank * per, (rank + 1) * per
    return HeadShard(rank, world, kv_lo, kv_hi, kv_lo * group, kv_hi * group)


def shard_inputs(q, k, v, shard: HeadShard):
    """Views of [Z, H, L, D] tensors restricted to the shard's heads (no copies)."""
    return (q[:, shard.q_lo:shard.q_hi], k[:, shard.kv_lo:shard.kv_hi], v[:, shard.kv_lo:shard.kv_hi])


def gather_heads(out_local, world: int, group=None):
    """All-gather head shards [Z, Hq/world, L, D] into [Z, Hq, L, D] on every rank.

    One all_gather_into_tensor of the contiguous shard buffers (rank-major == head-major
    when Z == 1), then a head-axis view for Z > 1."""
    import torch
    import torch.distributed as dist

    z, h, l, d = out_local.shape
    local = out_local.transpose(0, 1).contiguous()  # [H/world, Z, L, D]: rank-major == head-major
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * h, z, l, d), dtype=out_local.dtype, device=out_local.device)
        dist.all_gather_into_tensor(full, local, group=group)
    else:  # gloo (CPU tests)
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local, group=group)
        full = torch.cat(parts, 0)
    return full.transpose(0, 1)


def sharded_attention(q, k, v, cfg, world: int, rank: int, allgather: bool = False, group=None, op=None):
    """S2O attention on this rank's head shard; optionally all-gather the full output.

    q/k/v are the FULL [Z, H, L, D] tensors (or any objects supporting head slicing); `op`
    defaults to the CUDA operator (paper_2602_22575_b200.s2o_attention) and is injectable so
    the partition/assembly logic is testable on CPU."""
    z, hq, l, d = q.shape
    hkv = k.shape[1]
    shard = head_shard(hq, hkv, world, rank)
    qs, ks, vs = shard_inputs(q, k, v, shard)
    if op is None:
        from .s2o import s2o_attention

        out = s2o_attention(qs, ks, vs, cfg, want_plan=False).out
    else:
        out = op(qs, ks, vs, cfg)
    if allgather:
        return gather_heads(out, world, group)
    return out
