"""NEXT f2: one RailS node spread over the P GPUs of a box, rail buffers on their
owner GPUs, pack fused with the intra-node NVLink hop (include/rails.h, f2 block).

Rank p (one process per GPU) holds source GPUs g0 = p*ng .. g0+ng-1 of the node
(ng = N / P) and owns rails p*ng .. p*ng+ng-1: NIC j hangs off GPU j, so
rail j's send buffer lives in GPU j's HBM.  One step:
  1. rails_histogram_gpus on the local rows                         (kernel)
  2. rails_gather_rows_peer: the node's msg_bytes rows (N*G*8 B/unit) are stored
     into every rank's node table over NVLink, flagged and awaited   (kernel)
  3. rails_lpt_schedule of the whole node, identical on every rank    (kernels)
  4. rails_rail_offsets_owner + rails_pack_owner: each chunk piece is stored
     straight into the owner's buffer through a peer-mapped pointer   (kernel)
  5. rails_peer_barrier orders every rank's pack before any consumer (kernel).
exchange="nccl" keeps the NCCL all-gather / all-reduce for steps 2 and 5.
Peer mapping: CUDA IPC handles exported/imported by librails (rails_ipc_*), each
rank mapping the peers' buffers under its own device.
"""
from __future__ import annotations

import torch

from . import rails
from .dist import check_not_capturing


def _enable_peer_access(dev: int, peers):
    torch.cuda.set_device(dev)
    for q in peers:
        if q != dev:
            rails.enable_peer_access(q)


class RailOwnerNode:
    def __init__(self, M: int, N: int, T: int, k: int, row_bytes: int, chunk_bytes: int, U: int,
                 d: int, n_inst: int, group=None, R2: float = 5.0e10, exchange: str = "peer"):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.p = dist.get_rank(group)
        if N % self.P:
            raise ValueError(f"N={N} rails must divide over {self.P} GPUs")
        self.ng = N // self.P
        self.g0 = self.p * self.ng
        self.M, self.N, self.T, self.k, self.RB, self.C, self.U, self.d = (
            M, N, T, k, row_bytes, chunk_bytes, U, d)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        dev = self.dev
        G = M * N
        self.tp = rails.topo(M, N, chunk_bytes, R2)
        self.sh = rails.shard(U, d, 1)
        self.counts = torch.empty((U, 1, self.ng, G), dtype=torch.int32, device=dev)
        self.msg_loc = torch.empty((U, 1, self.ng, G), dtype=torch.int64, device=dev)
        self.rank_loc = torch.empty((U, 1, self.ng, T, k), dtype=torch.int32, device=dev)
        self.exchange = exchange
        if exchange not in ("peer", "nccl"):
            raise ValueError("exchange must be 'peer' or 'nccl'")
        self.msg_node = torch.empty((U, 1, N, G), dtype=torch.int64, device=dev)
        self.sched = rails.Schedule.empty(self.tp, self.sh, dev)
        self.ws = rails.new_workspace(self.tp, self.sh, dev)
        self.rail_base = torch.empty((U, 1, N), dtype=torch.int64, device=dev)
        self.rail_total = torch.empty(N, dtype=torch.int64, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        # Theorem 4 / LPT: a rail's load per unit is at most mean + w_max <=
        # T*k*RB + C (all N GPUs' rows spread over N rails, chunks <= C)
        self.cap = U * (T * k * row_bytes + chunk_bytes)
        self.cap = (self.cap + 255) // 256 * 256
        # own rail buffers in this GPU's HBM, exported by CUDA IPC; the other ranks
        # map them under their own device so their pack kernels store over NVLink
        self.own_ptr, handle, self.buf = rails.ipc_alloc(self.ng * self.cap)
        # exchange buffer (flags + node-wide msg table) for the NVLink row gather
        xb, moff = rails.owner_exchange_layout(self.tp, U, self.P)
        self.xown, xhandle, xview = rails.ipc_alloc(xb)
        xview.zero_()
        torch.cuda.synchronize(dev)
        if exchange == "peer":
            self.msg_node = xview[moff:moff + U * N * G * 8].view(torch.int64).view(U, 1, N, G)
        self.gen = 0
        objs = [None] * self.P
        dist.all_gather_object(objs, (handle, dev.index, xhandle), group=group)
        _enable_peer_access(dev.index, [o[1] for o in objs])
        bases = []
        self.xbufs = []
        self.opened = []
        for q, (h, _, xh) in enumerate(objs):
            if q == self.p:
                bases.append(self.own_ptr)
                self.xbufs.append(self.xown)
            else:
                ptr = rails.ipc_open(h)
                self.opened.append(ptr)
                bases.append(ptr)
                xp = rails.ipc_open(xh)
                self.opened.append(xp)
                self.xbufs.append(xp)
        self.rail_ptrs = [bases[j // self.ng] + (j % self.ng) * self.cap for j in range(N)]
        self.rail_caps = [self.cap] * N
        dist.barrier(group=group)

    def close(self):
        """Unmap the peers' buffers, then free this rank's own (collective)."""
        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)
        for ptr in self.opened:
            rails.ipc_close(ptr)
        self.opened = []
        self.dist.barrier(group=self.group)
        rails.ipc_free(self.own_ptr)
        rails.ipc_free(self.xown)
        self.own_ptr = None
        self.xown = None

    def own_rail(self, j: int) -> torch.Tensor:
        """This rank's buffer of rail j (must be owned here)."""
        assert j // self.ng == self.p
        o = (j % self.ng) * self.cap
        return self.buf[o:o + self.cap]

    def schedule_part(self, topk: torch.Tensor, lut: torch.Tensor):
        rails.histogram_gpus(self.tp, self.sh, self.g0, topk, lut, self.RB,
                             out=(self.counts, self.msg_loc, self.rank_loc))
        if self.exchange == "peer":
            check_not_capturing("RailOwnerNode (peer exchange)")
        self.gen += 1
        if self.exchange == "peer":
            rails.gather_rows_peer(self.tp, self.U, self.g0, self.ng, self.msg_loc, self.p,
                                   self.P, self.gen, self.xbufs)
        else:
            for u in range(self.U):
                self.dist.all_gather_into_tensor(self.msg_node[u, 0], self.msg_loc[u, 0],
                                                 group=self.group)
        rails.lpt_schedule(self.tp, self.sh, self.msg_node, out=self.sched, workspace=self.ws)
        rails.rail_offsets_owner(self.tp, self.sh, self.sched.send_load, self.rail_base,
                                 self.rail_total)

    def pack_part(self, topk: torch.Tensor, lut: torch.Tensor, x: torch.Tensor):
        rails.pack_owner(self.tp, self.sh, self.g0, self.T, self.k, x, topk, lut, self.rank_loc,
                         self.msg_node, self.RB, self.sched, self.rail_base, self.rail_ptrs,
                         self.rail_caps)

    def fence(self):
        # every rank's pack precedes this barrier on its stream, so its completion
        # anywhere orders all peer writes before later consumers
        if self.exchange == "peer":
            rails.peer_barrier(self.p, self.P, self.gen, self.xbufs)
        else:
            self.dist.all_reduce(self.flag, group=self.group)

    def step(self, topk: torch.Tensor, lut: torch.Tensor, x: torch.Tensor):
        self.schedule_part(topk, lut)
        self.pack_part(topk, lut, x)
        self.fence()
