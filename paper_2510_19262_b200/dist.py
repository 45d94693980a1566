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
    """a6 hook for pipeline.*.step: SUM the partial sums, MAX the partial maxima.

    NCCL reduces the device tensors in place.  Under gloo (the CPU tests; test
    processes sharing one GPU, where NCCL refuses duplicate devices -- fine here, no
    kernel waits on another rank) device tensors are staged through host copies."""
    import torch.distributed as dist

    staged = dist.get_backend(group) == "gloo"

    def reduce(red_sum, red_max):
        if staged and red_sum.is_cuda:
            s, m = red_sum.cpu(), red_max.cpu()
            dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
            red_sum.copy_(s)
            red_max.copy_(m)
            return
        dist.all_reduce(red_sum, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(red_max, op=dist.ReduceOp.MAX, group=group)

    return reduce


def check_not_capturing(what: str):
    """The peer-memory exchanges count calls on the host (gen, passed by value to the
    kernel): a CUDA-graph replay would reuse the captured gen and parity, so the flag
    waits would pass at once and read stale or half-written partials.  Refuse."""
    import torch
    if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
        raise RuntimeError(f"{what} cannot be captured into a CUDA graph: its call counter "
                           "lives on the host (include/rails.h)")


class PeerFinalize:
    """a6 + finalize fused over NVLink peer memory (rails_eval_finalize_peer).

    Collective setup: each rank allocates an exchange buffer exported by CUDA IPC,
    the handles are all-gathered once (torch.distributed object collective), and
    every rank maps the others' buffers.  Each call then runs ONE kernel per rank:
    push partials to every rank, flag, wait, reduce, finalize -- no NCCL call in
    the step.  Used as the `reduce` hook of the pipelines (they call .finalize)."""

    def __init__(self, tp, U: int, device, group=None):
        import torch
        import torch.distributed as dist
        from . import rails
        self.dist, self.group, self.tp, self.U = dist, group, tp, U
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world > rails.PEER_MAX:
            raise ValueError(f"peer finalize supports up to {rails.PEER_MAX} GPUs")
        n = rails.peer_buffer_bytes(tp, U, self.world)
        self.own_ptr, handle, view = rails.ipc_alloc(n)
        view.zero_()
        torch.cuda.synchronize(device)
        objs = [None] * self.world
        dist.all_gather_object(objs, (handle, torch.device(device).index), group=group)
        self.opened = []
        self.bufs = []
        self.error = None
        try:  # every rank reaches the barrier below even if its mapping fails
            for _, di in objs:
                if di != torch.device(device).index:
                    rails.enable_peer_access(di)
            for q, (h, _) in enumerate(objs):
                if q == self.rank:
                    self.bufs.append(self.own_ptr)
                else:
                    ptr = rails.ipc_open(h)
                    self.opened.append(ptr)
                    self.bufs.append(ptr)
        except Exception as exc:  # noqa: BLE001 -- surfaced through .ok()
            self.error = str(exc)
        self.gen = 0
        dist.barrier(group=group)

    def ok(self) -> bool:
        """True on every rank iff every rank mapped every peer (collective; an object
        collective, so it works under NCCL and gloo alike)."""
        flags = [None] * self.world
        self.dist.all_gather_object(flags, self.error is None, group=self.group)
        return all(flags)

    def finalize(self, red_sum, red_max, out, stream=None):
        from . import rails
        check_not_capturing("PeerFinalize.finalize")
        self.gen += 1
        rails.eval_finalize_peer(self.tp, self.U, red_sum, red_max, self.rank, self.world,
                                 self.gen, self.bufs, out=out, stream=stream)

    def __call__(self, red_sum, red_max):  # pragma: no cover - use .finalize
        raise RuntimeError("PeerFinalize reduces inside the finalize kernel; call .finalize")

    def close(self):
        import torch
        from . import rails
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)
        for ptr in self.opened:
            rails.ipc_close(ptr)
        self.opened = []
        self.dist.barrier(group=self.group)
        rails.ipc_free(self.own_ptr)
        self.own_ptr = None
