"""One pass of the whole hot path (all SURVEY section 8(a) rows) over preallocated buffers.

Routing configs (C1, C3, C4):  a1-a5 (histogram, then the fused LPT schedule + eval
+ rail offsets, + finalize when this call holds every node) -> [a6 cross-rank
reduction + finalize] -> a7 pack.
Matrix configs (C2, C5):       a2-a5 fused -> [a6 + finalize].

Only buffer management and call sequencing live here; every step is a C-ABI call
into librails.so (``rails.py``).  ``reduce`` is the a6 hook: a callable taking
(red_sum, red_max) int64 tensors and all-reducing them (SUM, MAX) across the ranks
that hold different source nodes of the same units (torch.distributed / NCCL).
"""
from __future__ import annotations

import contextlib
from typing import Callable

import torch

from . import rails


def _nvtx(on: bool, name: str):
    """NVTX range around one phase (seen by nsys / ncu range filters) when enabled."""
    return torch.cuda.nvtx.range(name) if on else contextlib.nullcontext()


class RoutingPipeline:
    def __init__(self, M: int, N: int, T: int, k: int, row_bytes: int, chunk_bytes: int,
                 U: int, d0: int, nd: int, n_inst: int, device, R2: float = 5.0e10,
                 ecmp_seed: int = 0x9E3779B97F4A7C15, out_cap: int | None = None,
                 nvtx: bool = False):
        self.tp = rails.topo(M, N, chunk_bytes, R2, 0.0, ecmp_seed)
        self.sh = rails.shard(U, d0, nd)
        self.M, self.N, self.T, self.k, self.RB, self.C = M, N, T, k, row_bytes, chunk_bytes
        self.U, self.d0, self.nd = U, d0, nd
        dev = torch.device(device)
        G = M * N
        self.counts = torch.empty((U, nd, N, G), dtype=torch.int32, device=dev)
        self.msg = torch.empty((U, nd, N, G), dtype=torch.int64, device=dev)
        self.rank = torch.empty((U, nd, N, T, k), dtype=torch.int32, device=dev)
        self.sched = rails.Schedule.empty(self.tp, self.sh, dev)
        self.ws = rails.new_workspace(self.tp, self.sh, dev)
        self.ev = rails.EvalOut.empty(self.tp, self.sh, dev)
        self.final = rails.empty_final(U, dev)
        self.rail_base = torch.empty((U, nd, N), dtype=torch.int64, device=dev)
        self.total = torch.empty(1, dtype=torch.int64, device=dev)
        self.holds_all = d0 == 0 and nd == M  # the fused kernel can finalize the units
        self.nvtx = nvtx
        self._calls = {}
        # every remote (t,s) copy is at most one row: a tight upper bound needing no sync
        cap = out_cap if out_cap is not None else U * nd * N * T * k * row_bytes
        self.out = torch.empty(cap, dtype=torch.uint8, device=dev)

    def _bound(self, key, make):
        """Marshal a call's arguments once per set of input buffers (`key`: their data
        pointers), reuse it every step."""
        b = self._calls.get(key)
        if b is None:
            b = self._calls[key] = make()
        return b

    def schedule_part(self, topk: torch.Tensor, lut: torch.Tensor, stream=None):
        """a1-a5 (rails_histogram_schedule_eval): the histogram, then one kernel for
        schedule, eval, rail offsets (and the finalize when this pipeline holds every
        node of its units), launched with PDL behind the histogram."""
        call = self._bound(("sched", topk.data_ptr(), lut.data_ptr(), lut.numel()),
                           lambda: rails.bind_histogram_schedule_eval(
                               self.tp, self.sh, topk, lut, self.RB,
                               (self.counts, self.msg, self.rank), self.sched, self.ev, self.ws,
                               final=self.final if self.holds_all else None,
                               rail_base=self.rail_base, rail_total=self.total))
        with _nvtx(self.nvtx, "a1-a5 histogram+schedule+eval"):
            call(stream)

    def finalize_part(self, reduce: Callable | None = None, stream=None):
        """a6 + finalize for pipelines holding a subset of the nodes (no-op otherwise:
        the fused kernel already finalized)."""
        if reduce is None and self.holds_all:
            return
        with _nvtx(self.nvtx, "a6 exchange + finalize"):
            if reduce is None:
                rails.eval_finalize(self.tp, self.U, self.ev.red_sum, self.ev.red_max,
                                    out=self.final, stream=stream)
            elif hasattr(reduce, "finalize"):  # fused a6 + finalize over peer memory
                reduce.finalize(self.ev.red_sum, self.ev.red_max, self.final, stream=stream)
            else:
                reduce(self.ev.red_sum, self.ev.red_max)
                rails.eval_finalize(self.tp, self.U, self.ev.red_sum, self.ev.red_max,
                                    out=self.final, stream=stream)

    def pack_part(self, topk, lut, x, stream=None):
        pk = self._bound(("pack", x.data_ptr(), topk.data_ptr(), lut.data_ptr(), lut.numel()),
                         lambda: rails.bind_pack(self.tp, self.sh, self.T, self.k, x, topk, lut,
                                                 self.rank, self.msg, self.RB, self.sched,
                                                 self.rail_base, self.out))
        with _nvtx(self.nvtx, "a7 pack"):
            pk(stream)

    def step(self, topk, lut, x, reduce: Callable | None = None, stream=None):
        self.schedule_part(topk, lut, stream)
        self.finalize_part(reduce, stream)
        self.pack_part(topk, lut, x, stream)


class MatrixPipeline:
    """Schedule + eval for D^(1) byte matrices msg [U][nd][N][G] (no routing, no pack)."""

    def __init__(self, M: int, N: int, chunk_bytes: int, U: int, d0: int, nd: int, device,
                 R2: float = 5.0e10, ecmp_seed: int = 0x9E3779B97F4A7C15):
        self.tp = rails.topo(M, N, chunk_bytes, R2, 0.0, ecmp_seed)
        self.sh = rails.shard(U, d0, nd)
        self.U = U
        dev = torch.device(device)
        self.sched = rails.Schedule.empty(self.tp, self.sh, dev)
        self.ws = rails.new_workspace(self.tp, self.sh, dev)
        self.ev = rails.EvalOut.empty(self.tp, self.sh, dev)
        self.final = rails.empty_final(U, dev)
        self.holds_all = d0 == 0 and nd == M
        self._calls = {}

    def step(self, msg: torch.Tensor, reduce: Callable | None = None, stream=None):
        fin = self.final if (self.holds_all and reduce is None) else None
        key = (msg.data_ptr(), fin is not None)
        b = self._calls.get(key)
        if b is None:
            b = self._calls[key] = rails.bind_schedule_eval(self.tp, self.sh, msg, self.sched,
                                                            self.ev, self.ws, final=fin)
        b(stream)
        if fin is not None:
            return
        if reduce is not None and hasattr(reduce, "finalize"):  # fused a6 + finalize
            reduce.finalize(self.ev.red_sum, self.ev.red_max, self.final, stream=stream)
            return
        if reduce is not None:
            reduce(self.ev.red_sum, self.ev.red_max)
        rails.eval_finalize(self.tp, self.U, self.ev.red_sum, self.ev.red_max, out=self.final,
                            stream=stream)


class GraphStep:
    """A pipeline step captured once into a CUDA graph and replayed.

    Every call the step makes is an asynchronous C-ABI launch on the capturing
    stream with preallocated buffers (no host synchronisation, no allocation), so
    `pipe.step(*args)` captures as is; replaying it re-runs the whole hot path with
    one graph launch instead of ~8 host launches.  Inputs are read from the tensors
    passed at capture time: refill them in place (tensor.copy_) between replays.
    The a6 hook must be graph-safe: an NCCL all-reduce is (NCCL's own graph
    support); the peer-memory finalize is NOT -- its call counter lives on the host,
    so a replay would reuse the captured counter and read stale partials -- and it
    raises if called during capture (dist.check_not_capturing)."""

    def __init__(self, step: Callable, *args, warmup: int = 2):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):  # warm: lazy init (function attributes, modules)
                step(*args)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            step(*args)
        torch.cuda.synchronize()

    def __call__(self):
        self.graph.replay()
