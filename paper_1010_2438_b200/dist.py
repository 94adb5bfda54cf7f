"""Multi-GPU sharding of a run.

Trajectories are independent and the RNG is keyed by the global trajectory
id, so rank r of N runs replicas [r*R, (r+1)*R) of every point
(cwc_sim_opts.replica_offset / replicas_total) and produces exactly the
trajectories an unsharded run would.  The only exchange step is the merge of
the exact integer moments: one all-reduce (sum) over torch.distributed --
NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests.

sumsq is a 128-bit (lo, hi) pair; a plain 64-bit sum of the lo words would
drop carries, so it travels as four 32-bit limbs held in int64 (exact for up
to 2^31 ranks) and is carry-propagated after the reduce.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_replicas_per_rank: int, rank: int):
    """(replica_offset, replicas_total) for weak scaling: every rank runs
    n_replicas_per_rank replicas of every point."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    return rank * n_replicas_per_rank, world * n_replicas_per_rank


def _limbs(sumsq_pairs: torch.Tensor) -> torch.Tensor:
    """[..., 2] int64 (lo, hi as raw u64 bits) -> [..., 4] int64 32-bit limbs."""
    lo = sumsq_pairs[..., 0]
    hi = sumsq_pairs[..., 1]
    m = 0xFFFFFFFF
    return torch.stack([lo & m, (lo >> 32) & m, hi & m, (hi >> 32) & m], dim=-1)


def _from_limbs(limbs: torch.Tensor) -> torch.Tensor:
    """Carry-propagate summed 32-bit limbs back into (lo, hi) u64 bit pairs."""
    m = 0xFFFFFFFF
    l0, l1, l2, l3 = limbs.unbind(-1)
    c = l0 >> 32
    w0 = l0 & m
    l1 = l1 + c
    c = l1 >> 32
    w1 = l1 & m
    l2 = l2 + c
    c = l2 >> 32
    w2 = l2 & m
    w3 = (l3 + c) & m
    lo = w0 | (w1 << 32)
    hi = w2 | (w3 << 32)
    return torch.stack([lo, hi], dim=-1)


def allreduce_stats(count: torch.Tensor, sum_: torch.Tensor, sumsq: torch.Tensor, group=None):
    """In-place exact merge of per-rank moments (count, sum int64; sumsq
    [..., 2] int64 holding u64 words).  No-op without an initialised group."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return count, sum_, sumsq
    limbs = _limbs(sumsq)
    flat = torch.cat([count.reshape(-1), sum_.reshape(-1), limbs.reshape(-1)])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    n = count.numel()
    count.copy_(flat[:n].view_as(count))
    sum_.copy_(flat[n:2 * n].view_as(sum_))
    sumsq.copy_(_from_limbs(flat[2 * n:].view(limbs.shape)))
    return count, sum_, sumsq
