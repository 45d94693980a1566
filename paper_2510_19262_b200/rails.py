"""ctypes binding of include/rails.h -- argument marshalling only.

Every function here has the name of a C entry point (without the ``rails_``
prefix), checks tensor dtypes/devices/shapes, passes ``tensor.data_ptr()`` and the
current CUDA stream, and raises :class:`RailsError` on a nonzero return code.  All
computation happens in librails.so's sm_100a kernels; there is no CPU fallback:
loading fails loudly when the library is missing, and calls require CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librails.so")

RAILS_OK, RAILS_EINVAL, RAILS_ERANGE, RAILS_ENOSPC, RAILS_EOVERFLOW, RAILS_ECUDA = 0, -1, -2, -3, -4, -5
RAILS_ETIMEDOUT = -6
_NAMES = {-1: "EINVAL", -2: "ERANGE", -3: "ENOSPC", -4: "EOVERFLOW", -5: "ECUDA", -6: "ETIMEDOUT"}
RED_MAX_LEN = 4


def red_sum_len(M: int, N: int) -> int:
    return 3 * M * N + M + 2


class RailsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"RAILS_{_NAMES.get(code, code)}: {msg}")
        self.code = code


class Topo(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("N", ctypes.c_int32), ("chunk_bytes", ctypes.c_int64),
                ("R2", ctypes.c_double), ("R1", ctypes.c_double), ("ecmp_seed", ctypes.c_uint64)]


class Fabric(ctypes.Structure):
    _fields_ = [("S", ctypes.c_int32), ("R1", ctypes.c_double), ("Rs", ctypes.c_double)]


class Shard(ctypes.Structure):
    _fields_ = [("U", ctypes.c_int32), ("d0", ctypes.c_int32), ("nd", ctypes.c_int32)]


class _Sched(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("full_base", "rem_rail", "rem_off", "send_load", "n_full", "n_rem")]


class _Eval(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("S", "S_e", "S_u", "mse", "nmse", "red_sum", "red_max")]


_FINAL_FIELDS = ("maxload", "maxload_e", "maxload_u", "total", "rowmax", "colmax", "T", "T_e",
                 "T_u", "T_star", "busbw", "busbw_e", "busbw_u")
_FINAL_FLOAT = ("T", "T_e", "T_u", "T_star", "busbw", "busbw_e", "busbw_u")


class _Final(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in _FINAL_FIELDS]


PEER_MAX = 8


class Peer(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("gen", ctypes.c_uint32),
                ("buf", ctypes.c_void_p * PEER_MAX)]


_lib = None


def lib():
    """Load librails.so (raises if it has not been built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        PT, PS = ctypes.POINTER(Topo), ctypes.POINTER(Shard)
        L.rails_histogram.argtypes = [PT, PS, i32, i32, P, P, i32, i64, P, P, P, P]
        L.rails_schedule_workspace.argtypes = [PT, PS, ctypes.POINTER(sz)]
        L.rails_lpt_schedule.argtypes = [PT, PS, P, ctypes.POINTER(_Sched), P, sz, P]
        L.rails_lpt_schedule_qp.argtypes = [PT, PS, P, ctypes.POINTER(_Sched), i32, P, P, sz, P]
        L.rails_lpt_schedule_qp.restype = ctypes.c_int
        PF = ctypes.POINTER(Fabric)
        L.rails_flowsim_plan.argtypes = [PT, PF, i32, P, P, P, P]
        L.rails_flowsim_plan.restype = ctypes.c_int
        L.rails_flowsim_workspace.argtypes = [PT, PF, i32, i64, i64, ctypes.POINTER(sz)]
        L.rails_flowsim_workspace.restype = ctypes.c_int
        L.rails_flowsim.argtypes = [PT, PF, i32, P, P, i64, i64, P, sz, P, P, P, P]
        L.rails_flowsim.restype = ctypes.c_int
        L.rails_assign_workspace.argtypes = [i32, i64, ctypes.POINTER(sz)]
        L.rails_lpt_assign.argtypes = [i32, i32, P, i64, P, P, P, P, P, sz, P]
        L.rails_eval.argtypes = [PT, PS, P, ctypes.POINTER(_Sched), ctypes.POINTER(_Eval), P]
        L.rails_eval_finalize.argtypes = [PT, i32, P, P, ctypes.POINTER(_Final), P]
        L.rails_schedule_eval.argtypes = [PT, PS, P, ctypes.POINTER(_Sched),
                                          ctypes.POINTER(_Eval), ctypes.POINTER(_Final), P, P, P,
                                          sz, P]
        L.rails_schedule_eval.restype = ctypes.c_int
        L.rails_histogram_schedule_eval.argtypes = [PT, PS, i32, i32, P, P, i32, i64, P, P, P,
                                                    ctypes.POINTER(_Sched),
                                                    ctypes.POINTER(_Eval),
                                                    ctypes.POINTER(_Final), P, P, P, sz, P]
        L.rails_histogram_schedule_eval.restype = ctypes.c_int
        L.rails_peer_buffer_bytes.argtypes = [PT, i32, i32, ctypes.POINTER(sz)]
        L.rails_peer_buffer_bytes.restype = ctypes.c_int
        L.rails_eval_finalize_peer.argtypes = [PT, i32, P, P, ctypes.POINTER(Peer),
                                               ctypes.POINTER(_Final), P]
        L.rails_eval_finalize_peer.restype = ctypes.c_int
        L.rails_owner_exchange_layout.argtypes = [PT, i32, i32, ctypes.POINTER(sz),
                                                  ctypes.POINTER(sz)]
        L.rails_owner_exchange_layout.restype = ctypes.c_int
        L.rails_gather_rows_peer.argtypes = [PT, i32, i32, i32, P, ctypes.POINTER(Peer), P]
        L.rails_gather_rows_peer.restype = ctypes.c_int
        L.rails_peer_barrier.argtypes = [ctypes.POINTER(Peer), P]
        L.rails_peer_barrier.restype = ctypes.c_int
        L.rails_eval_finalize_peer_local.argtypes = [PT, i32, P, P, ctypes.POINTER(Peer),
                                                     P, P]
        L.rails_gather_rows_peer_local.argtypes = [PT, i32, i32, P, ctypes.POINTER(Peer), P]
        L.rails_peer_barrier_local.argtypes = [ctypes.POINTER(Peer), P]
        for n in ("rails_eval_finalize_peer_local", "rails_gather_rows_peer_local",
                  "rails_peer_barrier_local"):
            getattr(L, n).restype = ctypes.c_int
        L.rails_rail_offsets.argtypes = [PT, PS, P, P, P, P]
        L.rails_pack.argtypes = [PT, PS, i32, i32, P, P, P, i32, P, P, i64,
                                 ctypes.POINTER(_Sched), P, P, i64, P]
        L.rails_histogram_gpus.argtypes = [PT, PS, i32, i32, i32, i32, P, P, i32, i64, P, P, P, P]
        L.rails_rail_offsets_owner.argtypes = [PT, PS, P, P, P, P]
        L.rails_pack_owner.argtypes = [PT, PS, i32, i32, i32, i32, P, P, P, i32, P, P, i64,
                                       ctypes.POINTER(_Sched), P, P, P, P]
        L.rails_transpose_traffic.argtypes = [PT, i32, P, P, P]
        L.rails_recv_offsets.argtypes = [PT, i32, P, P, P, P]
        L.rails_pack_combine.argtypes = [PT, PS, i64, i64, P, P, P, P, ctypes.POINTER(_Sched), P,
                                         P, i64, P]
        L.rails_unpack_combine.argtypes = [PT, PS, i32, i32, P, P, i32, P, P, P, i64, P, P,
                                           ctypes.POINTER(_Sched), P, P, P, i64, P]
        for n in ("rails_transpose_traffic", "rails_recv_offsets", "rails_pack_combine",
                  "rails_unpack_combine"):
            getattr(L, n).restype = ctypes.c_int
        L.rails_ipc_alloc.argtypes = [i64, ctypes.POINTER(ctypes.c_void_p), P]
        L.rails_ipc_open.argtypes = [P, ctypes.POINTER(ctypes.c_void_p)]
        L.rails_ipc_close.argtypes = [P]
        L.rails_ipc_free.argtypes = [P]
        for n in ("rails_ipc_alloc", "rails_ipc_open", "rails_ipc_close", "rails_ipc_free"):
            getattr(L, n).restype = ctypes.c_int
        L.rails_enable_peer_access.argtypes = [i32]
        for n in ("rails_histogram_gpus", "rails_rail_offsets_owner", "rails_pack_owner",
                  "rails_enable_peer_access"):
            getattr(L, n).restype = ctypes.c_int
        L.rails_check.argtypes = [P]
        L.rails_last_error.restype = ctypes.c_char_p
        L.rails_launch_count.argtypes = [i32]
        L.rails_launch_count.restype = i64
        L.rails_version.restype = i32
        for n in ("rails_histogram", "rails_schedule_workspace", "rails_lpt_schedule",
                  "rails_assign_workspace", "rails_lpt_assign", "rails_eval",
                  "rails_eval_finalize", "rails_rail_offsets", "rails_pack", "rails_check"):
            getattr(L, n).restype = ctypes.c_int
        _lib = L
    return _lib


def _ok(rc: int):
    if rc != RAILS_OK:
        raise RailsError(rc, lib().rails_last_error().decode())


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None, dtype=None, what="tensor"):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{what} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def topo(M: int, N: int, chunk_bytes: int, R2: float = 5.0e10, R1: float = 0.0,
         ecmp_seed: int = 0x9E3779B97F4A7C15) -> Topo:
    return Topo(M, N, chunk_bytes, R2, R1, ecmp_seed)


def shard(U: int, d0: int, nd: int) -> Shard:
    return Shard(U, d0, nd)


# ---------------------------------------------------------------- a1
def histogram(tp: Topo, sh: Shard, topk: torch.Tensor, lut: torch.Tensor, row_bytes: int,
              with_rank: bool = True, out=None, stream=None):
    """topk int32 [U][nd][N][T][k] -> (counts int32, msg_bytes int64 [U][nd][N][G], rank)."""
    U, nd, N, T, k = topk.shape
    G = tp.M * tp.N
    assert (U, nd, N) == (sh.U, sh.nd, tp.N), "topk shape must be [U][nd][N][T][k]"
    dev = topk.device
    if out is None:
        counts = torch.empty((U, nd, N, G), dtype=torch.int32, device=dev)
        msg = torch.empty((U, nd, N, G), dtype=torch.int64, device=dev)
        rank = torch.empty((U, nd, N, T, k), dtype=torch.int32, device=dev) if with_rank else None
    else:
        counts, msg, rank = out
    _ok(lib().rails_histogram(ctypes.byref(tp), ctypes.byref(sh), T, k,
                              _ptr(topk, torch.int32, "topk"), _ptr(lut, torch.int32, "lut"),
                              lut.numel(), row_bytes, _ptr(counts, torch.int32, "counts"),
                              _ptr(msg, torch.int64, "msg"), _ptr(rank, torch.int32, "rank"),
                              _stream(stream)))
    return counts, msg, rank


# ---------------------------------------------------------------- a2-a4
@dataclass
class Schedule:
    full_base: torch.Tensor  # int64 [U][nd][N][G]
    rem_rail: torch.Tensor   # int8  [U][nd][N][G]
    rem_off: torch.Tensor    # int64 [U][nd][N][G]
    send_load: torch.Tensor  # int64 [U][nd][N]
    n_full: torch.Tensor     # int64 [U][nd]
    n_rem: torch.Tensor      # int32 [U][nd]

    @staticmethod
    def empty(tp: Topo, sh: Shard, device) -> "Schedule":
        U, nd, N, G = sh.U, sh.nd, tp.N, tp.M * tp.N
        z = dict(device=device)
        return Schedule(torch.empty((U, nd, N, G), dtype=torch.int64, **z),
                        torch.empty((U, nd, N, G), dtype=torch.int8, **z),
                        torch.empty((U, nd, N, G), dtype=torch.int64, **z),
                        torch.empty((U, nd, N), dtype=torch.int64, **z),
                        torch.empty((U, nd), dtype=torch.int64, **z),
                        torch.empty((U, nd), dtype=torch.int32, **z))

    def c(self) -> _Sched:
        return _Sched(_ptr(self.full_base, torch.int64, "full_base"),
                      _ptr(self.rem_rail, torch.int8, "rem_rail"),
                      _ptr(self.rem_off, torch.int64, "rem_off"),
                      _ptr(self.send_load, torch.int64, "send_load"),
                      _ptr(self.n_full, torch.int64, "n_full"),
                      _ptr(self.n_rem, torch.int32, "n_rem"))


def schedule_workspace(tp: Topo, sh: Shard) -> int:
    n = ctypes.c_size_t(0)
    _ok(lib().rails_schedule_workspace(ctypes.byref(tp), ctypes.byref(sh), ctypes.byref(n)))
    return int(n.value)


def new_workspace(tp: Topo, sh: Shard, device) -> torch.Tensor:
    """Schedule workspace, zero-filled once as rails_schedule_eval requires (the
    kernels leave it zeroed)."""
    return torch.zeros(schedule_workspace(tp, sh), dtype=torch.uint8, device=device)


def lpt_schedule(tp: Topo, sh: Shard, msg: torch.Tensor, out: Schedule | None = None,
                 workspace: torch.Tensor | None = None, stream=None) -> Schedule:
    if out is None:
        out = Schedule.empty(tp, sh, msg.device)
    if workspace is None:
        workspace = new_workspace(tp, sh, msg.device)
    cs = out.c()
    _ok(lib().rails_lpt_schedule(ctypes.byref(tp), ctypes.byref(sh), _ptr(msg, torch.int64, "msg"),
                                 ctypes.byref(cs), _ptr(workspace, torch.uint8, "workspace"),
                                 workspace.numel(), _stream(stream)))
    return out


def lpt_schedule_qp(tp: Topo, sh: Shard, msg: torch.Tensor, qps_per_rail: int,
                    out: Schedule | None = None, rem_qp: torch.Tensor | None = None,
                    workspace: torch.Tensor | None = None, stream=None):
    """rails_lpt_schedule_qp (NEXT f2): the schedule plus rem_qp int32 [U][nd][N][G]."""
    if out is None:
        out = Schedule.empty(tp, sh, msg.device)
    if rem_qp is None:
        rem_qp = torch.empty(out.rem_rail.shape, dtype=torch.int32, device=msg.device)
    if workspace is None:
        workspace = new_workspace(tp, sh, msg.device)
    cs = out.c()
    _ok(lib().rails_lpt_schedule_qp(ctypes.byref(tp), ctypes.byref(sh),
                                    _ptr(msg, torch.int64, "msg"), ctypes.byref(cs),
                                    int(qps_per_rail), _ptr(rem_qp, torch.int32, "rem_qp"),
                                    _ptr(workspace, torch.uint8, "workspace"), workspace.numel(),
                                    _stream(stream)))
    return out, rem_qp


def lpt_assign(N: int, seg_off: torch.Tensor, w: torch.Tensor, stream=None):
    """Generic atomic-flow LPT: returns (rail int32 [F], off int64 [F], load int64 [n_seg][N])."""
    n_seg = seg_off.numel() - 1
    F = w.numel()
    dev = w.device
    n = ctypes.c_size_t(0)
    _ok(lib().rails_assign_workspace(n_seg, F, ctypes.byref(n)))
    ws = torch.empty(int(n.value), dtype=torch.uint8, device=dev)
    rail = torch.empty(F, dtype=torch.int32, device=dev)
    off = torch.empty(F, dtype=torch.int64, device=dev)
    load = torch.empty((n_seg, N), dtype=torch.int64, device=dev)
    _ok(lib().rails_lpt_assign(N, n_seg, _ptr(seg_off, torch.int64, "seg_off"), F,
                               _ptr(w, torch.int64, "w"), _ptr(rail), _ptr(off), _ptr(load),
                               _ptr(ws), ws.numel(), _stream(stream)))
    return rail, off, load


# ---------------------------------------------------------------- a5
@dataclass
class EvalOut:
    S: torch.Tensor        # int64 [U][nd][N]
    S_e: torch.Tensor      # int64 [U][nd][N]
    S_u: torch.Tensor      # int64 [U][nd][N]
    mse: torch.Tensor      # float64 [U][nd]
    nmse: torch.Tensor     # float64 [U][nd]
    red_sum: torch.Tensor  # int64 [U][3MN+M+2]
    red_max: torch.Tensor  # int64 [U][4]

    @staticmethod
    def empty(tp: Topo, sh: Shard, device) -> "EvalOut":
        U, nd, N = sh.U, sh.nd, tp.N
        z = dict(device=device)
        return EvalOut(torch.empty((U, nd, N), dtype=torch.int64, **z),
                       torch.empty((U, nd, N), dtype=torch.int64, **z),
                       torch.empty((U, nd, N), dtype=torch.int64, **z),
                       torch.empty((U, nd), dtype=torch.float64, **z),
                       torch.empty((U, nd), dtype=torch.float64, **z),
                       torch.empty((U, red_sum_len(tp.M, N)), dtype=torch.int64, **z),
                       torch.empty((U, RED_MAX_LEN), dtype=torch.int64, **z))

    def c(self) -> _Eval:
        return _Eval(_ptr(self.S, torch.int64), _ptr(self.S_e, torch.int64),
                     _ptr(self.S_u, torch.int64), _ptr(self.mse, torch.float64),
                     _ptr(self.nmse, torch.float64), _ptr(self.red_sum, torch.int64),
                     _ptr(self.red_max, torch.int64))

    def R(self, M: int, N: int) -> torch.Tensor:
        return self.red_sum[:, :M * N].view(-1, M, N)

    def R_e(self, M: int, N: int) -> torch.Tensor:
        return self.red_sum[:, M * N:2 * M * N].view(-1, M, N)

    def R_u(self, M: int, N: int) -> torch.Tensor:
        return self.red_sum[:, 2 * M * N:3 * M * N].view(-1, M, N)

    def colsum(self, M: int, N: int) -> torch.Tensor:
        return self.red_sum[:, 3 * M * N:3 * M * N + M]


def eval(tp: Topo, sh: Shard, msg: torch.Tensor, sched: Schedule, out: EvalOut | None = None,
         stream=None) -> EvalOut:  # noqa: A001 - the C entry point is rails_eval
    if out is None:
        out = EvalOut.empty(tp, sh, msg.device)
    cs, ce = sched.c(), out.c()
    _ok(lib().rails_eval(ctypes.byref(tp), ctypes.byref(sh), _ptr(msg, torch.int64, "msg"),
                         ctypes.byref(cs), ctypes.byref(ce), _stream(stream)))
    return out


def empty_final(U: int, device) -> dict:
    f = {}
    for n in _FINAL_FIELDS:
        dt = torch.float64 if n in _FINAL_FLOAT else torch.int64
        f[n] = torch.empty(U, dtype=dt, device=device)
    return f


def eval_finalize(tp: Topo, U: int, red_sum: torch.Tensor, red_max: torch.Tensor,
                  out: dict | None = None, stream=None) -> dict:
    if out is None:
        out = empty_final(U, red_sum.device)
    cf = _Final(*[_ptr(out[n]) for n in _FINAL_FIELDS])
    _ok(lib().rails_eval_finalize(ctypes.byref(tp), U, _ptr(red_sum, torch.int64, "red_sum"),
                                  _ptr(red_max, torch.int64, "red_max"), ctypes.byref(cf),
                                  _stream(stream)))
    return out


def schedule_eval(tp: Topo, sh: Shard, msg: torch.Tensor, sched: Schedule, ev: EvalOut,
                  workspace: torch.Tensor, final: dict | None = None,
                  rail_base: torch.Tensor | None = None, rail_total: torch.Tensor | None = None,
                  stream=None):
    """a2-a5 fused (rails_schedule_eval): schedule + evaluation of the shard's nodes in
    one kernel, plus the per-unit finalize when the shard holds every node (`final`)
    and the rail offsets (`rail_base`, `rail_total`).  `workspace` must come from
    new_workspace()."""
    cs, ce = sched.c(), ev.c()
    cf = _Final(*[_ptr(final[n]) for n in _FINAL_FIELDS]) if final is not None else None
    _ok(lib().rails_schedule_eval(ctypes.byref(tp), ctypes.byref(sh),
                                  _ptr(msg, torch.int64, "msg"), ctypes.byref(cs),
                                  ctypes.byref(ce), ctypes.byref(cf) if cf is not None else None,
                                  _ptr(rail_base, torch.int64, "rail_base"),
                                  _ptr(rail_total, torch.int64, "rail_total"),
                                  _ptr(workspace, torch.uint8, "workspace"), workspace.numel(),
                                  _stream(stream)))


def peer_buffer_bytes(tp: Topo, U: int, world: int) -> int:
    n = ctypes.c_size_t(0)
    _ok(lib().rails_peer_buffer_bytes(ctypes.byref(tp), U, world, ctypes.byref(n)))
    return int(n.value)


def eval_finalize_peer(tp: Topo, U: int, red_sum: torch.Tensor, red_max: torch.Tensor,
                       rank: int, world: int, gen: int, bufs: list, out: dict | None = None,
                       stream=None) -> dict:
    """a6 + finalize in one kernel over NVLink peer memory (rails_eval_finalize_peer)."""
    if out is None:
        out = empty_final(U, red_sum.device)
    cf = _Final(*[_ptr(out[n]) for n in _FINAL_FIELDS])
    pr = Peer(rank, world, gen)
    for i, b in enumerate(bufs):
        pr.buf[i] = b
    _ok(lib().rails_eval_finalize_peer(ctypes.byref(tp), U, _ptr(red_sum, torch.int64, "red_sum"),
                                       _ptr(red_max, torch.int64, "red_max"), ctypes.byref(pr),
                                       ctypes.byref(cf), _stream(stream)))
    return out


def _peer(rank: int, world: int, gen: int, bufs) -> Peer:
    pr = Peer(rank, world, gen)
    for i, b in enumerate(bufs):
        pr.buf[i] = b
    return pr


def owner_exchange_layout(tp: Topo, U: int, world: int) -> tuple[int, int]:
    """(bytes, msg_offset) of a rail-owner rank's exchange buffer."""
    n, off = ctypes.c_size_t(0), ctypes.c_size_t(0)
    _ok(lib().rails_owner_exchange_layout(ctypes.byref(tp), U, world, ctypes.byref(n),
                                          ctypes.byref(off)))
    return int(n.value), int(off.value)


def gather_rows_peer(tp: Topo, U: int, g0: int, ng: int, msg_loc: torch.Tensor, rank: int,
                     world: int, gen: int, bufs, stream=None):
    _ok(lib().rails_gather_rows_peer(ctypes.byref(tp), U, g0, ng,
                                     _ptr(msg_loc, torch.int64, "msg_loc"),
                                     ctypes.byref(_peer(rank, world, gen, bufs)), _stream(stream)))


def peer_barrier(rank: int, world: int, gen: int, bufs, stream=None):
    _ok(lib().rails_peer_barrier(ctypes.byref(_peer(rank, world, gen, bufs)), _stream(stream)))


# -- every rank driven by this process on one device (one cooperative launch each)
def _ptr_array(ts, dtype, what):
    return (ctypes.c_void_p * len(ts))(*[_ptr(t, dtype, what).value for t in ts])


def eval_finalize_peer_local(tp: Topo, U: int, red_sums: list, red_maxs: list, gen: int,
                             bufs: list, outs: list, stream=None):
    """rails_eval_finalize_peer_local: rank p = (red_sums[p], red_maxs[p], outs[p])."""
    world = len(red_sums)
    finals = (_Final * world)(*[_Final(*[_ptr(o[n]) for n in _FINAL_FIELDS]) for o in outs])
    _ok(lib().rails_eval_finalize_peer_local(
        ctypes.byref(tp), U, _ptr_array(red_sums, torch.int64, "red_sum"),
        _ptr_array(red_maxs, torch.int64, "red_max"), ctypes.byref(_peer(0, world, gen, bufs)),
        finals, _stream(stream)))


def gather_rows_peer_local(tp: Topo, U: int, ng: int, msg_locs: list, gen: int, bufs,
                           stream=None):
    world = len(msg_locs)
    _ok(lib().rails_gather_rows_peer_local(ctypes.byref(tp), U, ng,
                                           _ptr_array(msg_locs, torch.int64, "msg_loc"),
                                           ctypes.byref(_peer(0, world, gen, bufs)),
                                           _stream(stream)))


def peer_barrier_local(world: int, gen: int, bufs, stream=None):
    _ok(lib().rails_peer_barrier_local(ctypes.byref(_peer(0, world, gen, bufs)),
                                       _stream(stream)))


# ---------------------------------------------------------------- a7
def rail_offsets(tp: Topo, sh: Shard, send_load: torch.Tensor, rail_base=None, total=None,
                 stream=None):
    if rail_base is None:
        rail_base = torch.empty_like(send_load)
    if total is None:
        total = torch.empty(1, dtype=torch.int64, device=send_load.device)
    _ok(lib().rails_rail_offsets(ctypes.byref(tp), ctypes.byref(sh),
                                 _ptr(send_load, torch.int64, "send_load"),
                                 _ptr(rail_base, torch.int64, "rail_base"),
                                 _ptr(total, torch.int64, "total"), _stream(stream)))
    return rail_base, total


def pack(tp: Topo, sh: Shard, T: int, k: int, x: torch.Tensor, topk: torch.Tensor,
         lut: torch.Tensor, rank: torch.Tensor, msg: torch.Tensor, row_bytes: int,
         sched: Schedule, rail_base: torch.Tensor, out: torch.Tensor, stream=None):
    cs = sched.c()
    _ok(lib().rails_pack(ctypes.byref(tp), ctypes.byref(sh), T, k, _ptr(x, None, "x"),
                         _ptr(topk, torch.int32, "topk"), _ptr(lut, torch.int32, "lut"),
                         lut.numel(), _ptr(rank, torch.int32, "rank"),
                         _ptr(msg, torch.int64, "msg"), row_bytes, ctypes.byref(cs),
                         _ptr(rail_base, torch.int64, "rail_base"), _ptr(out, None, "out"),
                         out.numel() * out.element_size(), _stream(stream)))


# ---------------------------------------------------------------- bound calls
class Bound:
    """One C entry point with its arguments marshalled ONCE (the pipelines call the
    same buffers every step): calling it appends the current CUDA stream and checks
    the return code.  Keeps the ctypes structs and tensors alive."""

    def __init__(self, cfn, cargs, keep):
        self.cfn, self.cargs, self.keep = cfn, tuple(cargs), keep

    def __call__(self, stream=None):
        rc = self.cfn(*self.cargs, _stream(stream))
        if rc != RAILS_OK:
            _ok(rc)


def bind_histogram(tp: Topo, sh: Shard, topk, lut, row_bytes: int, out) -> Bound:
    U, nd, N, T, k = topk.shape
    counts, msg, rank = out
    return Bound(lib().rails_histogram,
                 [ctypes.byref(tp), ctypes.byref(sh), T, k, _ptr(topk, torch.int32, "topk"),
                  _ptr(lut, torch.int32, "lut"), lut.numel(), row_bytes,
                  _ptr(counts, torch.int32, "counts"), _ptr(msg, torch.int64, "msg"),
                  _ptr(rank, torch.int32, "rank")], (tp, sh, topk, lut, out))


def bind_schedule_eval(tp: Topo, sh: Shard, msg, sched: Schedule, ev: EvalOut, workspace,
                       final: dict | None = None, rail_base=None, rail_total=None) -> Bound:
    cs, ce = sched.c(), ev.c()
    cf = _Final(*[_ptr(final[n]) for n in _FINAL_FIELDS]) if final is not None else None
    return Bound(lib().rails_schedule_eval,
                 [ctypes.byref(tp), ctypes.byref(sh), _ptr(msg, torch.int64, "msg"),
                  ctypes.byref(cs), ctypes.byref(ce),
                  ctypes.byref(cf) if cf is not None else None,
                  _ptr(rail_base, torch.int64, "rail_base"),
                  _ptr(rail_total, torch.int64, "rail_total"),
                  _ptr(workspace, torch.uint8, "workspace"), workspace.numel()],
                 (tp, sh, msg, sched, ev, workspace, final, rail_base, rail_total, cs, ce, cf))


def bind_histogram_schedule_eval(tp: Topo, sh: Shard, topk, lut, row_bytes: int, hist_out,
                                 sched: Schedule, ev: EvalOut, workspace, final: dict | None = None,
                                 rail_base=None, rail_total=None) -> Bound:
    """a1-a5 fused (rails_histogram_schedule_eval), marshalled once."""
    U, nd, N, T, k = topk.shape
    counts, msg, rank = hist_out
    cs, ce = sched.c(), ev.c()
    cf = _Final(*[_ptr(final[n]) for n in _FINAL_FIELDS]) if final is not None else None
    return Bound(lib().rails_histogram_schedule_eval,
                 [ctypes.byref(tp), ctypes.byref(sh), T, k, _ptr(topk, torch.int32, "topk"),
                  _ptr(lut, torch.int32, "lut"), lut.numel(), row_bytes,
                  _ptr(counts, torch.int32, "counts"), _ptr(msg, torch.int64, "msg"),
                  _ptr(rank, torch.int32, "rank"), ctypes.byref(cs), ctypes.byref(ce),
                  ctypes.byref(cf) if cf is not None else None,
                  _ptr(rail_base, torch.int64, "rail_base"),
                  _ptr(rail_total, torch.int64, "rail_total"),
                  _ptr(workspace, torch.uint8, "workspace"), workspace.numel()],
                 (tp, sh, topk, lut, hist_out, sched, ev, workspace, final, rail_base, rail_total,
                  cs, ce, cf))


def bind_pack(tp: Topo, sh: Shard, T: int, k: int, x, topk, lut, rank, msg, row_bytes: int,
              sched: Schedule, rail_base, out) -> Bound:
    cs = sched.c()
    return Bound(lib().rails_pack,
                 [ctypes.byref(tp), ctypes.byref(sh), T, k, _ptr(x, None, "x"),
                  _ptr(topk, torch.int32, "topk"), _ptr(lut, torch.int32, "lut"), lut.numel(),
                  _ptr(rank, torch.int32, "rank"), _ptr(msg, torch.int64, "msg"), row_bytes,
                  ctypes.byref(cs), _ptr(rail_base, torch.int64, "rail_base"),
                  _ptr(out, None, "out"), out.numel() * out.element_size()],
                 (tp, sh, x, topk, lut, rank, msg, sched, rail_base, out, cs))


# ---------------------------------------------------------------- NEXT f1 (combine)
def transpose_traffic(tp: Topo, msg: torch.Tensor, out=None, stream=None):
    """Dispatch traffic [U][M][N][G] -> combine traffic (same shape, transposed GPUs)."""
    if out is None:
        out = torch.empty_like(msg)
    _ok(lib().rails_transpose_traffic(ctypes.byref(tp), msg.shape[0], _ptr(msg, torch.int64, "msg"),
                                      _ptr(out, torch.int64, "out"), _stream(stream)))
    return out


def recv_offsets(tp: Topo, counts: torch.Tensor, in_off=None, rows_in=None, stream=None):
    """Dispatch counts [U][M][N][G] -> in_off [U][G][G], rows_in [U][G]."""
    U = counts.shape[0]
    G = tp.M * tp.N
    if in_off is None:
        in_off = torch.empty((U, G, G), dtype=torch.int64, device=counts.device)
    if rows_in is None:
        rows_in = torch.empty((U, G), dtype=torch.int64, device=counts.device)
    _ok(lib().rails_recv_offsets(ctypes.byref(tp), U, _ptr(counts, torch.int32, "counts"),
                                 _ptr(in_off, torch.int64, "in_off"),
                                 _ptr(rows_in, torch.int64, "rows_in"), _stream(stream)))
    return in_off, rows_in


def pack_combine(tp: Topo, sh: Shard, row_bytes: int, y: torch.Tensor, in_off: torch.Tensor,
                 rows_in: torch.Tensor, msg_comb: torch.Tensor, sched: Schedule,
                 rail_base: torch.Tensor, out: torch.Tensor, stream=None):
    """y: bytes [U][nd][N][rows_cap][row_bytes] (any dtype view)."""
    rows_cap = y.shape[3]
    cs = sched.c()
    _ok(lib().rails_pack_combine(ctypes.byref(tp), ctypes.byref(sh), row_bytes, rows_cap,
                                 _ptr(y, None, "y"), _ptr(in_off, torch.int64, "in_off"),
                                 _ptr(rows_in, torch.int64, "rows_in"),
                                 _ptr(msg_comb, torch.int64, "msg_comb"), ctypes.byref(cs),
                                 _ptr(rail_base, torch.int64, "rail_base"), _ptr(out, None, "out"),
                                 out.numel() * out.element_size(), _stream(stream)))


def unpack_combine(tp: Topo, sh: Shard, T: int, k: int, topk: torch.Tensor, lut: torch.Tensor,
                   rank: torch.Tensor, w: torch.Tensor, y: torch.Tensor, in_off: torch.Tensor,
                   msg_comb_all: torch.Tensor, sched_all: Schedule, rail_base_all: torch.Tensor,
                   comb_out: torch.Tensor, row_bytes: int, out=None, stream=None):
    """-> float32 [U][nd][N][T][row_bytes/2]: top-k weighted expert outputs per token."""
    U, nd, N = sh.U, sh.nd, tp.N
    if out is None:
        out = torch.empty((U, nd, N, T, row_bytes // 2), dtype=torch.float32, device=topk.device)
    cs = sched_all.c()
    _ok(lib().rails_unpack_combine(ctypes.byref(tp), ctypes.byref(sh), T, k,
                                   _ptr(topk, torch.int32, "topk"), _ptr(lut, torch.int32, "lut"),
                                   lut.numel(), _ptr(rank, torch.int32, "rank"),
                                   _ptr(w, torch.float32, "w"), _ptr(y, None, "y"), y.shape[3],
                                   _ptr(in_off, torch.int64, "in_off"),
                                   _ptr(msg_comb_all, torch.int64, "msg_comb"), ctypes.byref(cs),
                                   _ptr(rail_base_all, torch.int64, "rail_base"),
                                   _ptr(comb_out, None, "comb_out"),
                                   _ptr(out, torch.float32, "out"), row_bytes, _stream(stream)))
    return out


# ---------------------------------------------------------------- NEXT f2 (rail owner)
def histogram_gpus(tp: Topo, sh: Shard, g0: int, topk: torch.Tensor, lut: torch.Tensor,
                   row_bytes: int, out=None, stream=None):
    """topk int32 [U][nd][ng][T][k] of source GPUs g0..g0+ng-1."""
    U, nd, ng, T, k = topk.shape
    G = tp.M * tp.N
    dev = topk.device
    if out is None:
        out = (torch.empty((U, nd, ng, G), dtype=torch.int32, device=dev),
               torch.empty((U, nd, ng, G), dtype=torch.int64, device=dev),
               torch.empty((U, nd, ng, T, k), dtype=torch.int32, device=dev))
    counts, msg, rank = out
    _ok(lib().rails_histogram_gpus(ctypes.byref(tp), ctypes.byref(sh), g0, ng, T, k,
                                   _ptr(topk, torch.int32, "topk"), _ptr(lut, torch.int32, "lut"),
                                   lut.numel(), row_bytes, _ptr(counts, torch.int32, "counts"),
                                   _ptr(msg, torch.int64, "msg"), _ptr(rank, torch.int32, "rank"),
                                   _stream(stream)))
    return counts, msg, rank


def rail_offsets_owner(tp: Topo, sh: Shard, send_load: torch.Tensor, rail_base=None,
                       rail_total=None, stream=None):
    if rail_base is None:
        rail_base = torch.empty_like(send_load)
    if rail_total is None:
        rail_total = torch.empty(tp.N, dtype=torch.int64, device=send_load.device)
    _ok(lib().rails_rail_offsets_owner(ctypes.byref(tp), ctypes.byref(sh),
                                       _ptr(send_load, torch.int64, "send_load"),
                                       _ptr(rail_base, torch.int64, "rail_base"),
                                       _ptr(rail_total, torch.int64, "rail_total"),
                                       _stream(stream)))
    return rail_base, rail_total


def pack_owner(tp: Topo, sh: Shard, g0: int, T: int, k: int, x: torch.Tensor,
               topk: torch.Tensor, lut: torch.Tensor, rank: torch.Tensor, msg_node: torch.Tensor,
               row_bytes: int, sched: Schedule, rail_base: torch.Tensor, rail_ptrs, rail_caps,
               stream=None):
    """rail_ptrs / rail_caps: python lists of N ints (device pointers, peer-mapped for
    rails owned by other GPUs) and capacities."""
    ng = topk.shape[2]
    N = tp.N
    ptrs = (ctypes.c_void_p * N)(*[ctypes.c_void_p(int(p)) for p in rail_ptrs])
    caps = (ctypes.c_int64 * N)(*[int(c) for c in rail_caps])
    cs = sched.c()
    _ok(lib().rails_pack_owner(ctypes.byref(tp), ctypes.byref(sh), g0, ng, T, k, _ptr(x, None, "x"),
                               _ptr(topk, torch.int32, "topk"), _ptr(lut, torch.int32, "lut"),
                               lut.numel(), _ptr(rank, torch.int32, "rank"),
                               _ptr(msg_node, torch.int64, "msg"), row_bytes, ctypes.byref(cs),
                               _ptr(rail_base, torch.int64, "rail_base"),
                               ctypes.cast(ptrs, ctypes.c_void_p), ctypes.cast(caps, ctypes.c_void_p),
                               _stream(stream)))


class _CudaArray:
    """__cuda_array_interface__ view of raw device bytes (for torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


def ipc_alloc(nbytes: int):
    """Owner side: (device pointer, 64-byte handle, uint8 tensor view)."""
    p = ctypes.c_void_p()
    h = ctypes.create_string_buffer(64)
    _ok(lib().rails_ipc_alloc(nbytes, ctypes.byref(p), h))
    view = torch.as_tensor(_CudaArray(p.value, nbytes), device="cuda")
    return p.value, bytes(h.raw), view


def ipc_open(handle: bytes) -> int:
    """Map another process's rail buffer for kernels of the current device."""
    p = ctypes.c_void_p()
    h = ctypes.create_string_buffer(handle, 64)
    _ok(lib().rails_ipc_open(h, ctypes.byref(p)))
    return p.value


def ipc_close(ptr: int):
    _ok(lib().rails_ipc_close(ctypes.c_void_p(ptr)))


def ipc_free(ptr: int):
    _ok(lib().rails_ipc_free(ctypes.c_void_p(ptr)))


def enable_peer_access(peer_device: int):
    """Let kernels on the current device load/store memory of `peer_device`."""
    _ok(lib().rails_enable_peer_access(peer_device))


# ---------------------------------------------------------------- misc
def check(stream=None):
    """Synchronise and raise on any device-side error recorded since the last check."""
    _ok(lib().rails_check(_stream(stream)))


def launch_count(reset: bool = False) -> int:
    return int(lib().rails_launch_count(1 if reset else 0))


def version() -> int:
    return int(lib().rails_version())


# ---------------------------------------------------------------- NEXT f4 (flowsim)
FS_POLICIES = {"lpt": 0, "uniform": 1, "ecmp": 2, "reps": 3, "minrtt": 4, "plb": 5}
FS_STATS = ("T", "total", "busbw", "cct_mean", "cct_p80", "cct_p95", "cct_p99",
            "max_pair_frac", "events", "flows")


def fabric(M: int, N: int, R2: float, S: int | None = None, R1: float | None = None,
           Rs: float | None = None) -> Fabric:
    """Defaults of R#35: S = N spines, R1 = 8*R2, Rs = M*R2/S."""
    S = N if S is None else S
    return Fabric(S, 8.0 * R2 if R1 is None else R1, M * R2 / S if Rs is None else Rs)


def fs_nlinks(M: int, N: int, S: int) -> int:
    return 2 * M * N * N + 2 * M * N + 2 * N * S


def flowsim(tp: Topo, fb: Fabric, policy: torch.Tensor, msg: torch.Tensor, stream=None):
    """rails_flowsim_plan + rails_flowsim: policy int32 [n_sim], msg int64
    [n_sim][M][N][G] (device).  Returns (msg_cct, link_bytes, stats) device tensors.
    The plan's flow totals are read back to size the workspace (one sync)."""
    n_sim = policy.numel()
    dev = msg.device
    tot = torch.empty((n_sim, 2), dtype=torch.int64, device=dev)
    _ok(lib().rails_flowsim_plan(ctypes.byref(tp), ctypes.byref(fb), n_sim,
                                 _ptr(policy, torch.int32, "policy"), _ptr(msg, torch.int64, "msg"),
                                 _ptr(tot), _stream(stream)))
    mx = tot.max(dim=0).values.cpu()
    capF, capS = max(int(mx[0]), 1), max(int(mx[1]), 1)
    n = ctypes.c_size_t(0)
    _ok(lib().rails_flowsim_workspace(ctypes.byref(tp), ctypes.byref(fb), n_sim, capF, capS,
                                      ctypes.byref(n)))
    ws = torch.empty(int(n.value), dtype=torch.uint8, device=dev)
    G = tp.M * tp.N
    cct = torch.empty((n_sim, tp.M, tp.N, G), dtype=torch.float64, device=dev)
    lb = torch.empty((n_sim, fs_nlinks(tp.M, tp.N, fb.S)), dtype=torch.float64, device=dev)
    st = torch.empty((n_sim, len(FS_STATS)), dtype=torch.float64, device=dev)
    _ok(lib().rails_flowsim(ctypes.byref(tp), ctypes.byref(fb), n_sim, _ptr(policy), _ptr(msg),
                            capF, capS, _ptr(ws), ws.numel(), _ptr(cct), _ptr(lb), _ptr(st),
                            _stream(stream)))
    return cct, lb, st
