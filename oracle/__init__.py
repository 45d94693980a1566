"""CPU oracle for the RailS hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_2510_19262_b200``) and never imports it.

The arithmetic lives in ``oracle.c`` (plain C, one function per paper step, each
citing the PAPER.md passage it follows) and ``flowsim.c`` (the NEXT f4 fluid
simulator: plain progressive filling and an event loop, R#35-R#39); this module only
marshals numpy arrays through ctypes and strings the per-node steps together in the
paper's order (Alg. 2).  ``brute.py`` holds the exhaustive optimum for
tiny inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "flowsim.c")]
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FP contraction: R#25)."""
    stale = not os.path.exists(_LIB) or any(
        os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS)
    if force or stale:
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
             "-o", _LIB] + _SRCS + ["-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64, u64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.orc_mix64.restype = u64
        L.orc_mix64.argtypes = [u64]
        L.orc_ecmp_rail.restype = i32
        L.orc_ecmp_rail.argtypes = [u64, i64, i64, i32]
        L.orc_histogram_node.restype = ctypes.c_int
        L.orc_histogram_node.argtypes = [i32, i32, i32, i32, i32, P, P, i32, i64, P, P, P]
        L.orc_chunk_count.restype = i64
        L.orc_chunk_count.argtypes = [i32, i64, P, i64]
        L.orc_split.restype = i64
        L.orc_split.argtypes = [i32, i64, P, i64, P, P, P, P]
        L.orc_lpt.restype = None
        L.orc_lpt.argtypes = [i64, i32, P, P, P, P, P]
        L.orc_compact.restype = None
        L.orc_compact.argtypes = [i32, i64, P, i64, i64, P, P, P, P, P, P, P, P, P, P, P]
        L.orc_mse.restype = dbl
        L.orc_mse.argtypes = [i32, P]
        L.orc_nmse.restype = dbl
        L.orc_nmse.argtypes = [i32, P]
        L.orc_eval.restype = None
        L.orc_eval.argtypes = [i32, i32, dbl, u64, P, i64, P, P, P, P, P, P, P, P, P, P, P, P]
        L.orc_pack_node.restype = ctypes.c_int
        L.orc_pack_node.argtypes = [i32, i32, i32, i32, i32, i64, i64, P, P, P, P, i64,
                                    P, P, P, P, P, P, P, P, i64]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


DEFAULT_ECMP_SEED = 0x9E3779B97F4A7C15  # R#14


# ------------------------------------------------------------------ scalars
def mix64(z: int) -> int:
    return int(lib().orc_mix64(z & 0xFFFFFFFFFFFFFFFF))


def ecmp_rail(seed: int, src: int, dst: int, N: int) -> int:
    return int(lib().orc_ecmp_rail(seed & 0xFFFFFFFFFFFFFFFF, src, dst, N))


def mse(loads) -> float:
    L = _c(loads, np.int64)
    return float(lib().orc_mse(len(L), _p(L)))


def nmse(loads) -> float:
    L = _c(loads, np.int64)
    return float(lib().orc_nmse(len(L), _p(L)))


# ------------------------------------------------------------------ steps
def histogram_node(M, N, d, T, k, topk_node, lut, row_bytes, with_rank=True):
    """a1 for node d: topk_node int32 [N][T][k] -> counts [N][G], msg [N][G], rank."""
    G = M * N
    topk_node = _c(topk_node, np.int32)
    lut = _c(lut, np.int32)
    counts = np.zeros((N, G), np.int32)
    msg = np.zeros((N, G), np.int64)
    rank = np.zeros((N, T, k), np.int32) if with_rank else None
    rc = lib().orc_histogram_node(M, N, d, T, k, _p(topk_node), _p(lut), len(lut), row_bytes,
                                  _p(counts), _p(msg), _p(rank) if with_rank else None)
    if rc != 0:
        raise ValueError("oracle histogram: routing id out of range")
    return counts, msg, rank


def split(msg_node, C):
    """a2: msg_node int64 [N][G] -> chunk arrays in emission order (g, h, c)."""
    msg_node = _c(msg_node, np.int64)
    N, G = msg_node.shape
    F = int(lib().orc_chunk_count(N, G, _p(msg_node), C))
    ch = dict(g=np.zeros(F, np.int32), h=np.zeros(F, np.int32),
              c=np.zeros(F, np.int64), size=np.zeros(F, np.int64))
    F2 = lib().orc_split(N, G, _p(msg_node), C, _p(ch["g"]), _p(ch["h"]), _p(ch["c"]),
                         _p(ch["size"]))
    assert F2 == F
    return ch


def lpt(w, N):
    """Alg. 2 steps 2-3 on weights given in tie-break order.
    Returns (order, rail, off, load)."""
    w = _c(w, np.int64)
    F = len(w)
    order = np.zeros(F, np.int64)
    rail = np.zeros(F, np.int32)
    off = np.zeros(F, np.int64)
    load = np.zeros(N, np.int64)
    lib().orc_lpt(F, N, _p(w), _p(order), _p(rail), _p(off), _p(load))
    return order, rail, off, load


def compact(msg_node, C, ch, rail, off):
    msg_node = _c(msg_node, np.int64)
    N, G = msg_node.shape
    F = len(ch["size"])
    full_base = np.zeros((N, G), np.int64)
    rem_rail = np.zeros((N, G), np.int8)
    rem_off = np.zeros((N, G), np.int64)
    n_full = np.zeros(1, np.int64)
    n_rem = np.zeros(1, np.int32)
    lib().orc_compact(N, G, _p(msg_node), C, F, _p(ch["g"]), _p(ch["h"]), _p(ch["c"]),
                      _p(ch["size"]), _p(rail), _p(off), _p(full_base), _p(rem_rail),
                      _p(rem_off), _p(n_full), _p(n_rem))
    return dict(full_base=full_base, rem_rail=rem_rail, rem_off=rem_off,
                n_full=int(n_full[0]), n_rem=int(n_rem[0]))


def schedule_node(msg_node, C):
    """a2-a4 for one node: chunks, LPT per chunk, compact schedule, LoadState."""
    msg_node = _c(msg_node, np.int64)
    N = msg_node.shape[0]
    ch = split(msg_node, C)
    order, rail, off, load = lpt(ch["size"], N)
    comp = compact(msg_node, C, ch, rail, off)
    return dict(chunks=ch, order=order, rail=rail, off=off, send_load=load, **comp)


def eval_unit(M, N, R2, ecmp_seed, msg_unit, ch_d, ch_h, ch_size, ch_rail):
    """a5 for one unit from an explicit per-chunk assignment (any policy)."""
    msg_unit = _c(msg_unit, np.int64)
    ch_d, ch_h = _c(ch_d, np.int32), _c(ch_h, np.int32)
    ch_size, ch_rail = _c(ch_size, np.int64), _c(ch_rail, np.int32)
    S = np.zeros((M, N), np.int64); R = np.zeros((M, N), np.int64)
    S_e = np.zeros((M, N), np.int64); R_e = np.zeros((M, N), np.int64)
    ints = np.zeros(6, np.int64); dbl = np.zeros(5, np.float64)
    ms = np.zeros(M, np.float64); nms = np.zeros(M, np.float64)
    lib().orc_eval(M, N, float(R2), ecmp_seed & 0xFFFFFFFFFFFFFFFF, _p(msg_unit), len(ch_size),
                   _p(ch_d), _p(ch_h), _p(ch_size), _p(ch_rail), _p(S), _p(R), _p(S_e), _p(R_e),
                   _p(ints), _p(dbl), _p(ms), _p(nms))
    return dict(S=S, R=R, S_e=S_e, R_e=R_e, maxload=int(ints[0]), maxload_e=int(ints[1]),
                total=int(ints[2]), rowmax=int(ints[3]), colmax=int(ints[4]),
                total_e=int(ints[5]), T=float(dbl[0]), T_e=float(dbl[1]),
                T_star=float(dbl[2]), busbw=float(dbl[3]), busbw_e=float(dbl[4]),
                mse=ms, nmse=nms)


def eval_uniform(M, N, R2, msg_unit):
    """The uniform split P* = 1/N (Theorem 3, R#41) of one unit msg_unit [M][N][G]."""
    L = lib()
    P = ctypes.c_void_p
    L.orc_eval_uniform.restype = None
    L.orc_eval_uniform.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, P, P, P, P, P]
    msg_unit = _c(msg_unit, np.int64)
    S_u = np.zeros((M, N), np.int64)
    R_u = np.zeros((M, N), np.int64)
    mx = np.zeros(1, np.int64)
    dbl = np.zeros(2, np.float64)
    L.orc_eval_uniform(M, N, float(R2), _p(msg_unit), _p(S_u), _p(R_u), _p(mx), _p(dbl))
    return dict(S_u=S_u, R_u=R_u, maxload_u=int(mx[0]), T_u=float(dbl[0]), busbw_u=float(dbl[1]))


def pack_node(M, N, d, T, k, row_bytes, C, x_node, topk_node, lut, msg_node, sched,
              rail_base, out_cap):
    """a7 for one node by definition; returns the output byte buffer."""
    x_node = _c(x_node, np.uint8)
    topk_node, lut = _c(topk_node, np.int32), _c(lut, np.int32)
    msg_node = _c(msg_node, np.int64)
    ch = sched["chunks"]
    rail_base = _c(rail_base, np.int64)
    out = np.zeros(int(out_cap), np.uint8)
    rc = lib().orc_pack_node(M, N, d, T, k, row_bytes, C, _p(x_node), _p(topk_node), _p(lut),
                             _p(msg_node), len(ch["size"]), _p(ch["g"]), _p(ch["h"]),
                             _p(ch["c"]), _p(ch["size"]), _p(_c(sched["rail"], np.int32)),
                             _p(_c(sched["off"], np.int64)), _p(rail_base), _p(out), out_cap)
    if rc != 0:
        raise RuntimeError(f"oracle pack failed rc={rc}")
    return out


# ------------------------------------------------------------------ whole unit
def run_unit_matrix(M, N, C, R2, ecmp_seed, msg_unit):
    """Schedule + eval one unit given D^(1) bytes msg_unit [M][N][G]."""
    msg_unit = _c(msg_unit, np.int64)
    scheds = []
    cd, chh, cs, cr = [], [], [], []
    for d in range(M):
        s = schedule_node(msg_unit[d], C)
        scheds.append(s)
        F = len(s["chunks"]["size"])
        cd.append(np.full(F, d, np.int32)); chh.append(s["chunks"]["h"])
        cs.append(s["chunks"]["size"]); cr.append(s["rail"])
    ev = eval_unit(M, N, R2, ecmp_seed, msg_unit, np.concatenate(cd), np.concatenate(chh),
                   np.concatenate(cs), np.concatenate(cr))
    ev.update(eval_uniform(M, N, R2, msg_unit))  # the uniform P* = 1/N baseline (R#41)
    return scheds, ev


def run_unit_routing(M, N, T, k, row_bytes, C, R2, ecmp_seed, topk_unit, lut):
    """Histogram + schedule + eval for one unit given routing topk_unit [M][N][T][k]."""
    G = M * N
    counts = np.zeros((M, N, G), np.int32)
    msg = np.zeros((M, N, G), np.int64)
    rank = np.zeros((M, N, T, k), np.int32)
    for d in range(M):
        counts[d], msg[d], rank[d] = histogram_node(M, N, d, T, k, topk_unit[d], lut, row_bytes)
    scheds, ev = run_unit_matrix(M, N, C, R2, ecmp_seed, msg)
    return dict(counts=counts, msg=msg, rank=rank, scheds=scheds, eval=ev)


# ------------------------------------------------------------------ NEXT f1 (combine)
def _sig_f1(L):
    P = ctypes.c_void_p
    i32, i64 = ctypes.c_int32, ctypes.c_int64
    L.orc_transpose.restype = None
    L.orc_transpose.argtypes = [i32, i32, P, P]
    L.orc_recv_offsets.restype = None
    L.orc_recv_offsets.argtypes = [i64, P, P]
    L.orc_pack_combine_node.restype = ctypes.c_int
    L.orc_pack_combine_node.argtypes = [i32, i32, i32, i64, i64, P, P, P, i64, P, P, P, P, P, P,
                                        P, P, i64]
    L.orc_unpack_combine.restype = ctypes.c_int
    L.orc_unpack_combine.argtypes = [i32, i32, i32, i32, i32, i32, i64, i64, P, P, P, P, P, P,
                                     P, P, P, P, P, P]


def transpose(M, N, msg_unit):
    """Combine traffic of one unit (R#28): [M][N][G] -> [M][N][G]."""
    L = lib(); _sig_f1(L)
    msg_unit = _c(msg_unit, np.int64)
    out = np.zeros_like(msg_unit)
    L.orc_transpose(M, N, _p(msg_unit), _p(out))
    return out


def recv_offsets(rows_in):
    """Exclusive prefix of one receiving GPU's incoming row counts (R#29)."""
    L = lib(); _sig_f1(L)
    rows_in = _c(rows_in, np.int64)
    out = np.zeros_like(rows_in)
    L.orc_recv_offsets(len(rows_in), _p(rows_in), _p(out))
    return out


def pack_combine_node(M, N, f, RB, C, y_node, in_off_node, msgc_node, sched, rail_base, out_cap):
    """Combine pack of sender node f (R#30).  y_node: list of N uint8 arrays [rows][RB];
    in_off_node: [N][G] (rows of GPU f*N+m); msgc_node: [N][G] combine bytes."""
    L = lib(); _sig_f1(L)
    ys = [_c(v, np.uint8) for v in y_node]
    yp = (ctypes.c_void_p * N)(*[v.ctypes.data for v in ys])
    in_off_node, msgc_node = _c(in_off_node, np.int64), _c(msgc_node, np.int64)
    ch = sched["chunks"]
    rail_base = _c(rail_base, np.int64)
    out = np.zeros(int(out_cap), np.uint8)
    rc = L.orc_pack_combine_node(M, N, f, RB, C, ctypes.cast(yp, ctypes.c_void_p), _p(in_off_node),
                                 _p(msgc_node), len(ch["size"]), _p(ch["g"]), _p(ch["h"]),
                                 _p(ch["c"]), _p(ch["size"]), _p(_c(sched["rail"], np.int32)),
                                 _p(_c(sched["off"], np.int64)), _p(rail_base), _p(out), out_cap)
    if rc != 0:
        raise RuntimeError(f"oracle combine pack failed rc={rc}")
    return out


def first_chunk_table(N, G, sched):
    """Index (emission order) of chunk 0 of every message of a node's chunk list."""
    ch = sched["chunks"]
    first = np.full((N, G), -1, np.int64)
    sel = ch["c"] == 0
    first[ch["g"][sel], ch["h"][sel]] = np.nonzero(sel)[0]
    return first


def unpack_combine(M, N, d, g, T, k, RB, C, topk_g, lut, rank_g, w_g, y_node_d, in_off_node_d,
                   rails_bytes, rail_bases, firsts, scheds):
    """Top-k weighted combine for GPU (d,g) by definition (R#31); float32 [T][RB/2].
    rails_bytes[f]: node f's combine rail buffer block; rail_bases[f]: [N] offsets
    of its rails; firsts[f]/scheds[f]: node f's combine chunk list lookup."""
    L = lib(); _sig_f1(L)
    H = RB // 2
    out = np.zeros((T, H), np.float32)
    topk_g, lut, rank_g = _c(topk_g, np.int32), _c(lut, np.int32), _c(rank_g, np.int32)
    w_g = _c(w_g, np.float32)
    yd = [_c(v, np.uint8) for v in y_node_d]
    yp = (ctypes.c_void_p * N)(*[v.ctypes.data for v in yd])
    in_off_node_d = _c(in_off_node_d, np.int64)
    keep = []

    def arr(lst, dtype):
        a = [_c(v, dtype) for v in lst]
        keep.append(a)
        return (ctypes.c_void_p * len(a))(*[v.ctypes.data for v in a])
    rp = arr(rails_bytes, np.uint8)
    rbp = arr(rail_bases, np.int64)
    fp = arr(firsts, np.int64)
    railp = arr([s["rail"] for s in scheds], np.int32)
    offp = arr([s["off"] for s in scheds], np.int64)
    cv = lambda x: ctypes.cast(x, ctypes.c_void_p)  # noqa: E731
    rc = L.orc_unpack_combine(M, N, d, g, T, k, RB, C, _p(topk_g), _p(lut), _p(rank_g), _p(w_g),
                              cv(yp), _p(in_off_node_d), cv(rp), cv(rbp), cv(fp), cv(railp),
                              cv(offp), _p(out))
    if rc != 0:
        raise RuntimeError(f"oracle unpack failed rc={rc}")
    return out


# ------------------------------------------------------------------ NEXT f2 (QP map)
def qp_map(order, rail, N, qps_per_rail):
    """Alg. 2 step 4 (R#34): per-rail round-robin QP index of every chunk,
    visiting chunks in assignment order (order from lpt())."""
    L = lib()
    L.orc_qp_map.restype = ctypes.c_int
    L.orc_qp_map.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_int64, ctypes.c_void_p]
    order = _c(order, np.int64)
    rail = _c(rail, np.int32)
    qp = np.zeros(len(order), np.int64)
    rc = L.orc_qp_map(len(order), N, _p(order), _p(rail), qps_per_rail, _p(qp))
    if rc != 0:
        raise ValueError(f"oracle qp_map rc={rc}")
    return qp


def rem_qp_node(msg_node, C, qps_per_rail, sched=None):
    """QP index of each message's remainder chunk, -1 if none: int64 [N][G]."""
    msg_node = _c(msg_node, np.int64)
    N, G = msg_node.shape
    s = schedule_node(msg_node, C) if sched is None else sched
    qp = qp_map(s["order"], s["rail"], N, qps_per_rail)
    ch = s["chunks"]
    out = np.full((N, G), -1, np.int64)
    for i in range(len(ch["size"])):
        if ch["size"][i] < C:
            out[ch["g"][i], ch["h"][i]] = qp[i]
    return out, qp


# ------------------------------------------------------------------ NEXT f4 (flowsim)
FS_POLICIES = {"lpt": 0, "uniform": 1, "ecmp": 2, "reps": 3, "minrtt": 4, "plb": 5}
FS_STATS = ("T", "total", "busbw", "cct_mean", "cct_p80", "cct_p95", "cct_p99",
            "max_pair_frac", "events", "flows")


def fs_nlinks(M, N, S):
    L = lib()
    L.orc_fs_nlinks.restype = ctypes.c_int64
    L.orc_fs_nlinks.argtypes = [ctypes.c_int32] * 3
    return int(L.orc_fs_nlinks(M, N, S))


def max_min(paths, w, cap):
    """Progressive-filling max-min rates (R#37) of subflows with link lists
    `paths` (each <= 4 links), share-weights `w`, link capacities `cap`."""
    L = lib()
    P = ctypes.c_void_p
    L.orc_max_min.restype = ctypes.c_int
    L.orc_max_min.argtypes = [ctypes.c_int64, P, P, P, ctypes.c_int64, P, P]
    n = len(paths)
    nl = np.array([len(p) for p in paths], np.int32)
    links = np.full((max(n, 1), 4), -1, np.int64)
    for i, p in enumerate(paths):
        links[i, :len(p)] = p
    w = _c(w, np.float64)
    cap = _c(cap, np.float64)
    rate = np.zeros(n, np.float64)
    rc = L.orc_max_min(n, _p(nl), _p(links), _p(w), len(cap), _p(cap), _p(rate))
    assert rc == 0
    return rate


def flowsim(M, N, S, R1, R2, Rs, C, policy, msg_unit, seed=None):
    """One all-to-all round through the fluid simulator (R#35-R#39).
    msg_unit int64 [M][N][G].  Returns dict(msg_cct [M][N][G], link_bytes [L],
    and the FS_STATS scalars)."""
    L = lib()
    P = ctypes.c_void_p
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    L.orc_flowsim.restype = ctypes.c_int
    L.orc_flowsim.argtypes = [i32, i32, i32, dbl, dbl, dbl, i64, ctypes.c_uint64, i32, P, P, P, P]
    pol = FS_POLICIES[policy] if isinstance(policy, str) else int(policy)
    msg_unit = _c(msg_unit, np.int64)
    G = M * N
    cct = np.zeros((M, N, G), np.float64)
    lb = np.zeros(fs_nlinks(M, N, S), np.float64)
    st = np.zeros(10, np.float64)
    rc = L.orc_flowsim(M, N, S, R1, R2, Rs, C, DEFAULT_ECMP_SEED if seed is None else seed, pol,
                       _p(msg_unit), _p(cct), _p(lb), _p(st))
    if rc != 0:
        raise ValueError(f"oracle flowsim rc={rc}")
    out = dict(msg_cct=cct, link_bytes=lb)
    out.update({k: float(v) for k, v in zip(FS_STATS, st)})
    return out
