"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) for a6.

Sharding: every rank holds a contiguous block of source
nodes of each unit.  Schedules and packs are per node and need no communication
(each node "runs independently"); the only exchange is the receive-load
reduction of a6: partial R / R_e / column sums / totals are SUM-reduced and the
send-side maxima MAX-reduced across ranks before rails_eval_finalize.
"""
from __future__ import annotations

from typing import Callable


def shard_nodes(M: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous node block (d0, nd) of `rank`; blocks differ by at most one node."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if world > M:
        raise ValueError(f"cannot split {M} nodes over {world} ranks")
    base, extra = divmod(M, world)
    d0 = rank * base + min(rank, extra)
    nd = base + (1 if rank < extra else 0)
    return d0, nd


def weak_units(world: int, units_per_gpu_factor: int = 1) -> int:
    """Weak scaling: U = world units, so each rank holds M/world nodes of each of
    `world` units -- M (unit, node) schedules per GPU regardless of world size."""
    return world * units_per_gpu_factor


def make_reduce(group=None) -> Callable:
    """a6 hook for pipeline.*.step: SUM the partial sums, MAX the partial maxima."""
    import torch.distributed as dist

    def reduce(red_sum, red_max):
        dist.all_reduce(red_sum, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(red_max, op=dist.ReduceOp.MAX, group=group)

    return reduce
