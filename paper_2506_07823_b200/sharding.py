"""Batch sharding over ranks: one process per GPU, each rank owns its
own instances and solves them with no collective on the hot path; one all-gather of the first
controls and the step statistics after the timed region, and the max-over-ranks device time.

Plumbing only (torch.distributed, NCCL on GPUs, gloo in the CPU tests): no arithmetic of the method.
bench.py and tests/test_sharding_gloo.py both call these functions.
"""
from __future__ import annotations

import torch

STAT_KEYS = ("cost", "theta", "alpha", "accepted", "info")


def shard(per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: rank r owns instances [r * per_rank, (r + 1) * per_rank) of the global batch
    (its inputs are regenerated from the instance seeds, so nothing is scattered)."""
    return rank * per_rank, per_rank


def pack_results(u0: torch.Tensor, stats: dict) -> torch.Tensor:
    """[B][12 + 5] rows: u_0 followed by (cost, theta, alpha, accepted, info) in u_0's dtype
    (accepted and info are small integers, exact in f32/f64)."""
    cols = [stats[k].to(u0.dtype).reshape(-1, 1) for k in STAT_KEYS]
    return torch.cat([u0.reshape(u0.shape[0], -1)] + cols, 1).contiguous()


def gather_results(packed: torch.Tensor, world: int, dist=None) -> torch.Tensor:
    """The one collective of the sharded path: all_gather_into_tensor of every rank's packed rows
    (rank-major, i.e. global instance order)."""
    if world == 1:
        return packed
    out = torch.empty((world * packed.shape[0],) + tuple(packed.shape[1:]), dtype=packed.dtype,
                      device=packed.device)
    dist.all_gather_into_tensor(out, packed)
    return out


def max_over_ranks(ms: float, world: int, device, dist=None) -> float:
    """Timing rule: the job's time is the slowest rank's device time."""
    if world == 1:
        return float(ms)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
