"""CUDA path (through the C ABI) vs the CPU oracle, element by element (-m gpu).

Integers (counts, bytes, ranks, schedules, loads, packed bytes) must be bit-exact;
derived floats (T, T*, busbw, MSE) within 1e-6 relative (BASELINE.json), and the
max observed error is printed.  Inputs are seeded; sizes span several tiles plus
ragged tails and include the degenerate cases of the method.
"""
import hashlib

import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import (R2, SEED, compare_schedule, oracle_eval_from_scheds, random_msg, rel_err,
                     routing_inputs)

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import MatrixPipeline, RoutingPipeline

DEV = "cuda:0"
FLOAT_TOL = 1e-6
MAX_ERR = {"v": 0.0}


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    rails.check()


def _cmp_float(a, b, what):
    e = rel_err(float(a), float(b))
    MAX_ERR["v"] = max(MAX_ERR["v"], e)
    assert e <= FLOAT_TOL, f"{what}: gpu {a!r} oracle {b!r} rel {e:g}"


# ------------------------------------------------------------------ a1 histogram
@pytest.mark.parametrize("M,N,T,k,E,U,d0,nd", [
    (4, 4, 4096, 2, 8, 1, 0, 4),      # C1 shape
    (3, 5, 777, 3, 7, 2, 1, 2),       # ragged, N not a power of 2, shard
    (2, 1, 100, 1, 3, 1, 0, 2),       # N = 1, k = 1
    (9, 8, 333, 2, 8, 2, 3, 4),       # G = 72, multi-unit
    (64, 8, 513, 2, 8, 1, 60, 4),     # C3-sized bins (G = 512), ragged tokens
    (300, 8, 64, 2, 8, 1, 0, 2),      # G = 2400 -> 4-warp histogram variant
])
def test_histogram_parity(M, N, T, k, E, U, d0, nd):
    topk_all, lut = routing_inputs(M, N, T, k, E, 11, 0, U)
    topk = topk_all[:, d0:d0 + nd].contiguous()
    tp = rails.topo(M, N, 65536)
    sh = rails.shard(U, d0, nd)
    RB = 8192
    counts, msg, rank = rails.histogram(tp, sh, topk.to(DEV), lut.to(DEV), RB)
    counts, msg, rank = counts.cpu().numpy(), msg.cpu().numpy(), rank.cpu().numpy()
    for u in range(U):
        for dl in range(nd):
            c, m, r = oracle.histogram_node(M, N, d0 + dl, T, k, topk[u, dl].numpy(), lut.numpy(), RB)
            assert np.array_equal(counts[u, dl], c)
            assert np.array_equal(msg[u, dl], m)
            assert np.array_equal(rank[u, dl], r)


def test_histogram_range_error_flagged():
    M, N, T, k = 2, 2, 64, 2
    topk = torch.zeros((1, 2, N, T, k), dtype=torch.int32)
    topk[0, 1, 1, 7, 1] = 99  # instance id out of range
    lut = torch.tensor([0, 1, 2, 3], dtype=torch.int32)
    rails.histogram(rails.topo(M, N, 4096), rails.shard(1, 0, 2), topk.to(DEV), lut.to(DEV), 16)
    with pytest.raises(rails.RailsError) as ei:
        rails.check()
    assert ei.value.code == rails.RAILS_ERANGE
    rails.check()  # flag cleared


# ------------------------------------------------------------------ a2-a4 schedule
@pytest.mark.parametrize("M,N,C,U,d0,nd,p,hi,mult", [
    (4, 4, 65536, 2, 0, 4, 0.7, 500000, 1),
    (16, 8, 1 << 20, 2, 0, 16, 0.9, 30 << 20, 1),     # C2-like sizes
    (5, 3, 1000, 1, 0, 5, 0.5, 20000, 1),            # C not a power of two
    (6, 7, 16, 1, 2, 3, 0.3, 2000, 1),               # tiny chunks, many full chunks
    (3, 2, 1, 1, 0, 3, 0.5, 50, 1),                  # C = 1: no remainders
    (4, 8, 1 << 30, 1, 0, 4, 0.8, 100000, 1),        # C > every message: all remainders
    (70, 8, 32768, 1, 0, 3, 0.9, 300000, 1),         # NG = 4480 remainder sort
    (3, 4, 96, 1, 0, 3, 0.8, 10, 32),                # many equal sizes (ties)
    (2, 1, 4096, 3, 0, 2, 1.0, 100000, 1),           # N = 1
    (300, 8, 4096, 1, 0, 2, 0.9, 50000, 1),          # NG = 19200 > smem: global-scratch sort
    (6, 8, 1 << 24, 1, 0, 6, 0.8, 1 << 26, 1),       # 2^23 <= C < 2^26: warp relative-key chain
    (5, 16, 65536, 2, 0, 5, 0.6, 400000, 1),         # N = 16 register-network chain
    (40, 2, 8192, 30, 0, 40, 0.7, 100000, 1),        # N = 2, 1200 chains (thread chains)
    (3, 32, 65536, 2, 0, 3, 0.7, 400000, 1),         # N = 32: the maximum (one rail per lane)
    (4, 32, 4096, 1, 0, 4, 0.9, 40, 4096),           # N = 32, equal sizes (runs, ties)
])
def test_schedule_parity(M, N, C, U, d0, nd, p, hi, mult):
    rng = np.random.default_rng(M * 1000 + N * 10 + U)
    msg = random_msg(rng, U, M, N, p=p, hi=hi, mult=mult, nodes=range(d0, d0 + nd))
    tp = rails.topo(M, N, C)
    sh = rails.shard(U, d0, nd)
    s = rails.lpt_schedule(tp, sh, torch.from_numpy(msg).to(DEV))
    for u in range(U):
        for dl in range(nd):
            compare_schedule(s, u, dl, oracle.schedule_node(msg[u, dl], C), f"u{u} d{dl}")


@pytest.mark.parametrize("M,N,U,RB,C,outliers", [
    (64, 8, 1, 12288, 32768, 0),     # C4 rows: 7 remainder sizes, runs span batches
    (64, 8, 1, 8192, 32768, 6),      # C3 rows: 3 sizes, a few odd sizes break runs
    (40, 4, 2, 12288, 32768, 3),     # N = 4
    (30, 16, 1, 4096, 65536, 2),     # N = 16 (no 8-item cyclic group, run path only)
    (50, 2, 1, 3000, 32768, 4),      # N = 2, 11 sizes
    (40, 8, 32, 12288, 32768, 2),    # 1280 chains: thread-per-chain kernel
    (64, 8, 1, 0, 4096, 0),          # RB = 0: size depends on the destination only,
    (64, 4, 1, 0, 65536, 3),         # so aligned groups of N equal sizes (C5-like)
    (64, 2, 1, 0, 1 << 20, 0),       # -> the warp-scan window path
    (6, 32, 1, 8192, 32768, 2),      # N = 32 (the generic warp chain)
])
def test_schedule_parity_equal_runs(M, N, U, RB, C, outliers):
    # routing-like traffic (row multiples) makes long runs of equal remainder sizes:
    # the cyclic run path (lpt_run_cyclic) and its single-step transients
    rng = np.random.default_rng(M * 7 + N + U)
    G = M * N
    if RB:
        msg = rng.integers(0, 40, size=(U, M, N, G)).astype(np.int64) * RB
        msg *= rng.random((U, M, N, G)) < 0.9
    else:
        col = rng.integers(1, 1 << 24, size=(U, M, 1, G)).astype(np.int64)
        msg = np.repeat(col, N, axis=2)
        RB = 1
    for _ in range(outliers * U * M):
        u, d, g, h = (int(rng.integers(0, x)) for x in (U, M, N, G))
        msg[u, d, g, h] = int(rng.integers(1, 40 * RB))
    for d in range(M):
        msg[:, d, :, d * N:(d + 1) * N] = 0
    s = rails.lpt_schedule(rails.topo(M, N, C), rails.shard(U, 0, M), torch.from_numpy(msg).to(DEV))
    for u in range(U):
        for d in range(M):
            compare_schedule(s, u, d, oracle.schedule_node(msg[u, d], C), f"u{u} d{d}")


def test_schedule_general_path_large_chunks():
    # C >= 2^26 uses the 64-bit argmin chain
    rng = np.random.default_rng(5)
    M, N, C = 3, 4, 1 << 27
    msg = random_msg(rng, 1, M, N, p=0.9, hi=1 << 29)
    s = rails.lpt_schedule(rails.topo(M, N, C), rails.shard(1, 0, M), torch.from_numpy(msg).to(DEV))
    for d in range(M):
        compare_schedule(s, 0, d, oracle.schedule_node(msg[0, d], C), f"d{d}")


def test_schedule_all_zero_and_empty_nodes():
    M, N, C = 4, 4, 4096
    msg = np.zeros((2, M, N, M * N), np.int64)
    msg[1, 2, 3, 5] = 12345
    s = rails.lpt_schedule(rails.topo(M, N, C), rails.shard(2, 0, M), torch.from_numpy(msg).to(DEV))
    for u in range(2):
        for d in range(M):
            compare_schedule(s, u, d, oracle.schedule_node(msg[u, d], C))


def test_schedule_intra_node_bytes_flagged():
    M, N = 2, 2
    msg = np.zeros((1, M, N, M * N), np.int64)
    msg[0, 0, 0, 1] = 100  # node 0 -> its own GPU 1: not inter-domain (R#2)
    rails.lpt_schedule(rails.topo(M, N, 64), rails.shard(1, 0, M), torch.from_numpy(msg).to(DEV))
    with pytest.raises(rails.RailsError):
        rails.check()


@pytest.mark.parametrize("skew", ["receiver", "sender", "uniform"])
def test_schedule_eval_c2_reduced(skew):
    cfg = dict(gen.CONFIGS["c2"], skew=skew)
    U = 3
    msg = gen.d1_units(cfg, gen.config_seed(2), 0, U)
    M, N, C = cfg["M"], cfg["N"], cfg["C"]
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    for u in range(U):
        scheds = [oracle.schedule_node(msg[u, d], C) for d in range(M)]
        for d in range(M):
            compare_schedule(pipe.sched, u, d, scheds[d], f"u{u} d{d}")
        ev = oracle_eval_from_scheds(M, N, msg[u], scheds)
        _compare_eval(pipe, u, 0, M, M, N, ev)


# ------------------------------------------------------------------ generic LPT
def test_lpt_assign_parity():
    rng = np.random.default_rng(9)
    sets = [[5, 4, 3, 3, 2], [3, 3, 2, 2, 2], [7, 7, 6, 6, 5, 5, 4, 4, 4], [], [0, 0, 5],
            list(rng.integers(1, 10 ** 6, size=1000)), list(rng.integers(1, 4, size=333)),
            list(rng.integers(1, 1 << 40, size=77))]
    for N in (1, 2, 3, 8, 32):
        w = np.concatenate([np.asarray(s, np.int64) for s in sets])
        off = np.concatenate([[0], np.cumsum([len(s) for s in sets])]).astype(np.int64)
        rail, o, load = rails.lpt_assign(N, torch.from_numpy(off).to(DEV), torch.from_numpy(w).to(DEV))
        rail, o, load = rail.cpu().numpy(), o.cpu().numpy(), load.cpu().numpy()
        for i, s in enumerate(sets):
            _, r_o, o_o, l_o = oracle.lpt(np.asarray(s, np.int64), N)
            a, b = off[i], off[i + 1]
            assert np.array_equal(rail[a:b], r_o), (N, i)
            assert np.array_equal(o[a:b], o_o), (N, i)
            assert np.array_equal(load[i], l_o), (N, i)


# ------------------------------------------------------------------ a5 eval
def _compare_eval(pipe, u, d0, nd, M, N, ev):
    e = pipe.ev
    S = e.S[u].cpu().numpy()
    assert np.array_equal(S, ev["S"][d0:d0 + nd])
    assert np.array_equal(e.S_e[u].cpu().numpy(), ev["S_e"][d0:d0 + nd])
    assert np.array_equal(e.R(M, N)[u].cpu().numpy(), ev["R"])
    assert np.array_equal(e.R_e(M, N)[u].cpu().numpy(), ev["R_e"])
    # uniform P* = 1/N split (Theorem 3, R#41)
    assert np.array_equal(e.S_u[u].cpu().numpy(), ev["S_u"][d0:d0 + nd])
    assert np.array_equal(e.R_u(M, N)[u].cpu().numpy(), ev["R_u"])
    # send_load from the LPT chain equals S recomputed from the schedule
    assert np.array_equal(pipe.sched.send_load[u].cpu().numpy(), S)
    f = {k: v[u].item() for k, v in pipe.final.items()}
    for key in ("maxload", "maxload_e", "maxload_u", "total", "rowmax", "colmax"):
        assert f[key] == ev[key], key
    for key in ("T", "T_e", "T_u", "T_star", "busbw", "busbw_e", "busbw_u"):
        _cmp_float(f[key], ev[key], key)
    for dl in range(nd):
        _cmp_float(e.mse[u, dl].item(), ev["mse"][d0 + dl], "mse")
        _cmp_float(e.nmse[u, dl].item(), ev["nmse"][d0 + dl], "nmse")


@pytest.mark.parametrize("M,N,C,U", [(4, 4, 65536, 2), (7, 3, 1000, 1), (5, 8, 4096, 2),
                                     (2, 1, 64, 1), (33, 8, 32768, 1), (3, 32, 4096, 2)])
def test_eval_parity(M, N, C, U):
    rng = np.random.default_rng(M + N + C)
    msg = random_msg(rng, U, M, N, p=0.5, hi=300000)
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    for u in range(U):
        scheds = [oracle.schedule_node(msg[u, d], C) for d in range(M)]
        _compare_eval(pipe, u, 0, M, M, N, oracle_eval_from_scheds(M, N, msg[u], scheds))


@pytest.mark.parametrize("nsizes,rep", [(20, 40), (45, 40), (60, 32)])
def test_schedule_many_runs(nsizes, rep):
    """Remainders in runs of >= 32 equal sizes (the chain's deferred cyclic runs,
    lpt.cuh RunList): fewer and more runs than the fused kernel's run list holds
    (32; the rest are written inline), with odd sizes and full chunks around them.
    Schedule and eval both exact."""
    M, N, C = 32, 8, 1 << 16
    G = M * N
    rng = np.random.default_rng(nsizes * 1000 + rep)
    msg = np.zeros((1, M, N, G), np.int64)
    for d in range(M):
        sizes = rng.choice(np.arange(100, C - 1, 37), nsizes, replace=False)
        vals = np.repeat(sizes, rep) + C * rng.integers(0, 3, nsizes * rep)
        extra = rng.integers(1, 4 * C, 60)  # odd sizes between the runs
        vals = np.concatenate([vals, extra])
        slots = [(g, h) for g in range(N) for h in range(G) if h // N != d]
        pick = rng.choice(len(slots), len(vals), replace=False)
        for v, i in zip(vals, pick):
            g, h = slots[i]
            msg[0, d, g, h] = v
    pipe = MatrixPipeline(M, N, C, 1, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    scheds = [oracle.schedule_node(msg[0, d], C) for d in range(M)]
    for d in range(M):
        compare_schedule(pipe.sched, 0, d, scheds[d], f"d{d}")
    _compare_eval(pipe, 0, 0, M, M, N, oracle_eval_from_scheds(M, N, msg[0], scheds))
    s = rails.lpt_schedule(rails.topo(M, N, C), rails.shard(1, 0, M), torch.from_numpy(msg).to(DEV))
    for d in range(M):
        compare_schedule(s, 0, d, scheds[d], f"schedule-only d{d}")


def test_eval_no_traffic():
    M, N = 3, 2
    msg = np.zeros((1, M, N, M * N), np.int64)
    pipe = MatrixPipeline(M, N, 4096, 1, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    assert pipe.final["total"].item() == 0 and pipe.final["busbw"].item() == 0.0
    assert pipe.final["T"].item() == 0.0 and pipe.ev.nmse.abs().sum().item() == 0


def test_sharded_eval_equals_unsharded():
    # a6: partial red_sum (SUM) / red_max (MAX) over node shards == one-shot result
    rng = np.random.default_rng(21)
    M, N, C, U = 9, 4, 8192, 2
    msg = random_msg(rng, U, M, N, p=0.6, hi=100000)
    full = MatrixPipeline(M, N, C, U, 0, M, DEV)
    full.step(torch.from_numpy(msg).to(DEV))
    cuts = [0, 2, 7, 9]
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        p = MatrixPipeline(M, N, C, U, a, b - a, DEV)
        p.step(torch.from_numpy(msg[:, a:b].copy()).to(DEV))
        parts.append(p)
        assert torch.equal(p.sched.send_load, full.sched.send_load[:, a:b])
        assert torch.equal(p.sched.rem_off, full.sched.rem_off[:, a:b])
    rs = sum(p.ev.red_sum for p in parts)
    rm = torch.stack([p.ev.red_max for p in parts]).amax(0)
    assert torch.equal(rs, full.ev.red_sum) and torch.equal(rm, full.ev.red_max)
    fin = rails.eval_finalize(full.tp, U, rs.contiguous(), rm.contiguous())
    for k in fin:
        assert torch.equal(fin[k], full.final[k]), k


# ------------------------------------------------------------------ a7 pack
def _oracle_pack_check(pipe, topk, lut, x, u, dl, scheds_oracle=None):
    M, N, T, k, RB, C = pipe.M, pipe.N, pipe.T, pipe.k, pipe.RB, pipe.C
    d = pipe.d0 + dl
    c, m, r = oracle.histogram_node(M, N, d, T, k, topk[u, dl].numpy(), lut.numpy(), RB)
    s = oracle.schedule_node(m, C) if scheds_oracle is None else scheds_oracle
    base_all = pipe.rail_base[u, dl].cpu().numpy()
    start = int(base_all[0])
    L = s["send_load"]
    base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
    assert np.array_equal(base_all - start, base)
    want = oracle.pack_node(M, N, d, T, k, RB, C, x[u, dl].numpy().view(np.uint8), topk[u, dl].numpy(),
                            lut.numpy(), m, s, base, int(L.sum()))
    got = pipe.out[start:start + int(L.sum())].cpu().numpy()
    assert got.shape == want.shape
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"pack mismatch u{u} d{d}: {len(bad)} bytes differ, first at {bad[0]}")


@pytest.mark.parametrize("M,N,T,k,E,RB,C,U,d0,nd", [
    (4, 4, 512, 2, 8, 1024, 4096, 1, 0, 4),     # C >= RB, 2-piece path
    (3, 2, 300, 2, 4, 4096, 1024, 1, 0, 3),     # C < RB: multi-piece path
    (3, 5, 211, 3, 6, 48, 80, 2, 1, 2),         # C not a power of two, ragged T, 3 slots
    (2, 1, 100, 1, 3, 16, 16, 1, 0, 2),         # N = 1, smallest rows/chunks
    (5, 8, 128, 2, 8, 12288, 32768, 1, 0, 5),   # C4 row size (12 KiB) straddling 32 KiB
    (3, 2, 40, 2, 4, 20480, 8192, 1, 0, 3),     # rows > 16 KiB window, multi-piece
    (2, 32, 64, 4, 32, 256, 1024, 1, 0, 2),     # N = 32 rails (maximum), G = 64
    (4, 4, 1, 2, 8, 8192, 32768, 1, 0, 4),      # T = 1: one token row per GPU
    (3, 4, 2, 1, 8, 16, 4096, 2, 0, 3),         # T = 2, 16-byte rows, every message < C
])
def test_pack_parity(M, N, T, k, E, RB, C, U, d0, nd):
    topk_all, lut = routing_inputs(M, N, T, k, E, 7, 0, U)
    topk = topk_all[:, d0:d0 + nd].contiguous()
    x = torch.stack([gen.payload(M, N, T, RB, 3, u, d0, nd) for u in range(U)])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), DEV)
    pipe.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
    torch.cuda.synchronize()
    assert int(pipe.total.item()) == int(pipe.sched.send_load.sum().item())
    for u in range(U):
        for dl in range(nd):
            _oracle_pack_check(pipe, topk, lut, x, u, dl)


def test_pack_enospc_flagged():
    M, N, T, k, E, RB, C = 2, 2, 64, 2, 4, 256, 4096
    topk, lut = routing_inputs(M, N, T, k, E, 1, 0, 1)
    x = gen.payload(M, N, T, RB, 3, 0, 0, M)[None]
    pipe = RoutingPipeline(M, N, T, k, RB, C, 1, 0, M, lut.numel(), DEV, out_cap=1024)
    pipe.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
    with pytest.raises(rails.RailsError) as ei:
        rails.check()
    assert ei.value.code == rails.RAILS_ENOSPC


# ------------------------------------------------------------------ full configs
def _routing_full(cfg_name, U=None, sample_nodes=None, pack_nodes=(0,), seed_off=0,
                  eval_full=True, d0=0, nd=None):
    cfg = gen.CONFIGS[cfg_name]
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    U = cfg["U"] if U is None else U
    nd = M - d0 if nd is None else nd
    RB = cfg["H"] * 2
    seed = gen.config_seed(int(cfg_name[1])) + seed_off
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u, d0, nd, device=DEV) for u in range(U)])
    lut = gen.inst_lut(M, N, E).to(DEV)
    x = torch.empty((U, nd, N, T, RB // 8), dtype=torch.int64, device=DEV)
    for u in range(U):
        gen.payload(M, N, T, RB, seed, u, d0, nd, device=DEV, out=x[u])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), DEV)
    pipe.step(topk, lut, x)
    torch.cuda.synchronize()
    topk_c, lut_c = topk.cpu(), lut.cpu()
    for u in range(U):
        nodes = range(M) if sample_nodes is None else sample_nodes
        if eval_full:
            res = oracle.run_unit_routing(M, N, T, k, RB, C, R2, SEED, topk_c[u].numpy(), lut_c.numpy())
            assert np.array_equal(pipe.counts[u].cpu().numpy(), res["counts"])
            assert np.array_equal(pipe.msg[u].cpu().numpy(), res["msg"])
            assert np.array_equal(pipe.rank[u].cpu().numpy(), res["rank"])
            for d in nodes:
                compare_schedule(pipe.sched, u, d, res["scheds"][d], f"u{u} d{d}")
            _compare_eval(pipe, u, 0, M, M, N, res["eval"])
            scheds = res["scheds"]
        else:
            scheds = {}
            for d in nodes:
                dl = d - d0
                c, m, r = oracle.histogram_node(M, N, d, T, k, topk_c[u, dl].numpy(), lut_c.numpy(), RB)
                assert np.array_equal(pipe.msg[u, dl].cpu().numpy(), m)
                assert np.array_equal(pipe.rank[u, dl].cpu().numpy(), r)
                scheds[d] = oracle.schedule_node(m, C)
                compare_schedule(pipe.sched, u, dl, scheds[d], f"u{u} d{d}")
        for d in pack_nodes:
            xs = x[u:u + 1, d - d0:d - d0 + 1].cpu()
            _oracle_pack_check_node(pipe, topk_c, lut_c, xs, u, d, scheds[d])
    return pipe


def _oracle_pack_check_node(pipe, topk, lut, x_node, u, d, sched):
    M, N, T, k, RB, C = pipe.M, pipe.N, pipe.T, pipe.k, pipe.RB, pipe.C
    dl = d - pipe.d0
    _, m, _ = oracle.histogram_node(M, N, d, T, k, topk[u, dl].numpy(), lut.numpy(), RB)
    L = sched["send_load"]
    base_all = pipe.rail_base[u, dl].cpu().numpy()
    start = int(base_all[0])
    base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
    assert np.array_equal(base_all - start, base)
    want = oracle.pack_node(M, N, d, T, k, RB, C, x_node[0, 0].numpy().view(np.uint8),
                            topk[u, dl].numpy(), lut.numpy(), m, sched, base, int(L.sum()))
    got = pipe.out[start:start + int(L.sum())].cpu().numpy()
    assert hashlib.sha256(got.tobytes()).digest() == hashlib.sha256(want.tobytes()).digest(), \
        f"pack mismatch u{u} d{d}"


def test_config_c1_full():
    _routing_full("c1", pack_nodes=(0, 1, 2, 3))


@pytest.mark.slow
def test_config_c3_full_eval_sampled_pack():
    # BASELINE config 3 at full size in the launch configuration bench.py times;
    # oracle: every node's histogram/schedule/eval, pack on sampled nodes.
    _routing_full("c3", pack_nodes=(0, 37, 63))


@pytest.mark.slow
def test_config_c4_sampled_units():
    # config 4 (U=32 layers x 128 nodes, sharded over 8 GPUs): one GPU's shard of
    # the sharded launch -- 4 layers x 16 nodes (the per-rank block at P = 8);
    # oracle on sampled nodes (histogram, rank, schedule) and a sampled pack.
    _routing_full("c4", U=4, d0=64, nd=16, sample_nodes=(64, 70, 79), pack_nodes=(70,),
                  eval_full=False)


@pytest.mark.slow
@pytest.mark.parametrize("C", [4 << 10, 64 << 10, 1 << 20, 4 << 20])
def test_config_c5_sweep_sampled(C):
    cfg = gen.CONFIGS["c5"]
    M, N = cfg["M"], cfg["N"]
    msg = gen.d1_units(cfg, gen.config_seed(5), 0, 1)
    pipe = MatrixPipeline(M, N, C, 1, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    for d in (0, 100, 255):
        compare_schedule(pipe.sched, 0, d, oracle.schedule_node(msg[0, d], C), f"d{d}")
    if C >= (1 << 20):
        scheds = [oracle.schedule_node(msg[0, d], C) for d in range(M)]
        _compare_eval(pipe, 0, 0, M, M, N, oracle_eval_from_scheds(M, N, msg[0], scheds))
    else:
        # property at any size: sum S = sum R = total; T >= T*; send_load == S
        f = pipe.final
        assert f["T"].item() >= f["T_star"].item()
        assert int(pipe.ev.S.sum()) == int(msg.sum()) == f["total"].item()
        assert torch.equal(pipe.ev.S, pipe.sched.send_load)


@pytest.mark.parametrize("C", [4 << 10, 64 << 10])
def test_c5_family_small_chunks_full_eval(C):
    """C5's receiver-skew Zipf family at the small chunk sizes where the full-size
    sweep above only checks properties (the oracle materialises every chunk: 134 M at
    4 KiB and 256 nodes): the same generator on 32 nodes x 8 rails, 16 MiB per source
    GPU (32 K chunks per node at 4 KiB), schedule and evaluation exact for every node."""
    cfg = dict(gen.CONFIGS["c5"])
    cfg.update(M=32, V=16 << 20, C=C)
    M, N = cfg["M"], cfg["N"]
    msg = gen.d1_units(cfg, gen.config_seed(5), 0, 1)
    pipe = MatrixPipeline(M, N, C, 1, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    scheds = [oracle.schedule_node(msg[0, d], C) for d in range(M)]
    for d in range(M):
        compare_schedule(pipe.sched, 0, d, scheds[d], f"C{C} d{d}")
    _compare_eval(pipe, 0, 0, M, M, N, oracle_eval_from_scheds(M, N, msg[0], scheds))


def test_determinism_repeat():
    M, N, T, k, E, RB, C = 6, 4, 700, 2, 8, 2048, 8192
    topk, lut = routing_inputs(M, N, T, k, E, 5, 0, 2)
    x = torch.stack([gen.payload(M, N, T, RB, 5, u, 0, M) for u in range(2)])
    outs = []
    for _ in range(2):
        pipe = RoutingPipeline(M, N, T, k, RB, C, 2, 0, M, lut.numel(), DEV)
        pipe.out.zero_()
        pipe.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
        torch.cuda.synchronize()
        outs.append((pipe.rank.clone(), pipe.sched.rem_off.clone(), pipe.ev.red_sum.clone(),
                     pipe.out[:int(pipe.total.item())].clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_report_max_float_error():
    print(f"max relative float error observed vs oracle: {MAX_ERR['v']:.3g}")


@pytest.mark.parametrize("M,N,C,U,mult", [
    (40, 8, 32768, 4, 12288),     # 160 segments: fused per-node kernel, N = 8 network
    (40, 8, 32768, 12, 12288),    # 480 segments: k_chains (warp-staged chain)
    (5, 4, 65536, 2, 1),          # N = 4: generic redux chain (fused kernel)
    (5, 4, 65536, 80, 1),         # N = 4, 400 segments: generic chain of k_chains
    (30, 2, 4096, 3, 100),
    (6, 8, 1 << 24, 2, 1),        # C >= 2^23: generic chain on N = 8
    (6, 8, 1 << 24, 60, 1),       # ... in k_chains
    (3, 5, 1 << 27, 2, 1),        # C >= 2^26: 64-bit butterfly argmin
])
def test_schedule_parity_both_paths(M, N, C, U, mult):
    """rails_lpt_schedule picks the fused per-node kernel for few segments and the
    per-phase kernels (k_chains.cu) for more than 2 x the SM count; within each, the
    N = 8 sorted-register network or the generic chain by N and C.  All exact."""
    rng = np.random.default_rng(77 + U)
    msg = random_msg(rng, U, M, N, p=0.8, hi=40, mult=mult) if mult > 1 else \
        random_msg(rng, U, M, N, p=0.8, hi=min(4 * C, 1 << 40))
    s = rails.lpt_schedule(rails.topo(M, N, C), rails.shard(U, 0, M), torch.from_numpy(msg).to(DEV))
    for u in sorted(set([0, U - 1, U // 2])):
        for d in range(M):
            compare_schedule(s, u, d, oracle.schedule_node(msg[u, d], C), f"U{U} u{u} d{d}")


@pytest.mark.parametrize("M,N,T,k,E,RB,C,U,d0,nd", [
    (4, 4, 512, 2, 8, 1024, 4096, 1, 0, 4),     # rows <= 2 KiB: 4 vectors per lane
    (5, 8, 128, 2, 8, 8192, 32768, 1, 0, 5),    # 8 KiB rows: 16 vectors per lane
    (3, 4, 100, 2, 8, 4096, 1024, 2, 1, 2),     # C < RB: per-vector chunk lookup
    (3, 2, 64, 3, 6, 20480, 4096, 1, 0, 3),     # 20 KiB rows in 8 KiB windows, C < RB
])
def test_pack_parity_row_shapes(M, N, T, k, E, RB, C, U, d0, nd):
    topk_all, lut = routing_inputs(M, N, T, k, E, 7, 0, U)
    topk = topk_all[:, d0:d0 + nd].contiguous()
    x = torch.stack([gen.payload(M, N, T, RB, 3, u, d0, nd) for u in range(U)])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), DEV)
    pipe.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
    torch.cuda.synchronize()
    for u in range(U):
        for dl in range(nd):
            _oracle_pack_check(pipe, topk, lut, x, u, dl)


def _hist_check(M, N, T, k, E, U, nd, RB=4096, with_rank=True, seed=17, nodes=None):
    topk_all, lut = routing_inputs(M, N, T, k, E, seed, 0, U)
    topk = topk_all[:, 0:nd].contiguous()
    tp, sh = rails.topo(M, N, 65536), rails.shard(U, 0, nd)
    counts, msg, rank = rails.histogram(tp, sh, topk.to(DEV), lut.to(DEV), RB, with_rank=with_rank)
    for u in range(U):
        for dl in (range(nd) if nodes is None else nodes):
            c, m, r = oracle.histogram_node(M, N, dl, T, k, topk[u, dl].numpy(), lut.numpy(), RB)
            assert np.array_equal(counts[u, dl].cpu().numpy(), c), (M, N, T, u, dl)
            assert np.array_equal(msg[u, dl].cpu().numpy(), m), (M, N, T, u, dl)
            if with_rank:
                assert np.array_equal(rank[u, dl].cpu().numpy(), r), (M, N, T, u, dl)


@pytest.mark.parametrize("M,N,T,k,E,U,nd,with_rank", [
    (2, 2, 1000, 2, 4, 600, 2, True),       # G = 4: nearly every 32-id group collides
    (64, 8, 777, 2, 8, 5, 64, True),        # ragged last batch, shared LUT
    (128, 8, 300, 2, 8, 3, 128, False),     # no ranks
    (600, 8, 64, 2, 8, 1, 300, True),       # n_inst = 4800: LUT read through L1
    (4, 4, 1, 2, 8, 600, 4, True),          # T = 1: two entries per segment
    (8, 4, 5, 3, 8, 300, 8, True),          # T*k = 15 < 32: one partial group
])
def test_histogram_parity_batched(M, N, T, k, E, U, nd, with_rank):
    """>= 16 segments per SM: the warp-per-segment atomic-ranking kernel."""
    _hist_check(M, N, T, k, E, U, nd, with_rank=with_rank, nodes=[0, nd - 1])


@pytest.mark.parametrize("M,N,T,k,E,nd", [
    (2, 2, 1000, 2, 4, 2),        # G = 4: 16 warps per segment, collisions everywhere
    (64, 8, 777, 2, 8, 2),        # G = 512, 16 warps
    (3, 4, 4096, 4, 8, 2),
    (2, 4, 10000, 4, 8, 2),
    (300, 8, 500, 2, 8, 2),       # G = 2400: 4 warps (sub-histograms in 64 KiB)
    (1500, 8, 200, 2, 8, 1),      # G = 12000: 2 warps
    (5000, 4, 64, 2, 4, 1),       # G = 20000: 1 warp
    (4, 4, 1, 1, 8, 2),           # T*k = 1: 15 of the 16 warps have no entries
    (64, 8, 3, 2, 8, 2),          # T*k = 6, G = 512
    (16, 8, 37, 3, 8, 2),         # T*k = 111: ragged, fewer entries than 16 x 32
])
def test_histogram_parity_few_segments(M, N, T, k, E, nd):
    """Few segments: W warps per segment (by G), two passes, tag-trick ranks."""
    _hist_check(M, N, T, k, E, 1, nd)


def test_histogram_zero_tokens_rejected():
    """T = 0 is not a routing step (rails.h: T >= 1): EINVAL before any launch."""
    M, N = 2, 2
    topk = torch.zeros((1, 2, N, 0, 2), dtype=torch.int32, device=DEV)
    lut = torch.arange(4, dtype=torch.int32, device=DEV)
    with pytest.raises(rails.RailsError) as ei:
        rails.histogram(rails.topo(M, N, 4096), rails.shard(1, 0, 2), topk, lut, 16)
    assert ei.value.code == rails.RAILS_EINVAL


def test_histogram_parity_huge_segment():
    """T*k >= 2^24: ranks past the tag trick's 24 bits use the per-bit ballot match."""
    _hist_check(2, 1, (1 << 23) + 77, 2, 2, 1, 1, RB=16)



def test_graph_replay_matches_eager():
    # the whole routing step captured into a CUDA graph: replays give exactly the
    # eager step's schedule, evaluation and packed bytes (also after new inputs)
    from paper_2510_19262_b200.pipeline import GraphStep
    M, N, T, k, E, RB, C, U = 4, 4, 512, 2, 8, 1024, 4096, 2
    topk_all, lut = routing_inputs(M, N, T, k, E, 21, 0, U)
    x = torch.stack([gen.payload(M, N, T, RB, 5, u, 0, M) for u in range(U)]).to(DEV)
    topk = topk_all.to(DEV)
    lut = lut.to(DEV)
    eager = RoutingPipeline(M, N, T, k, RB, C, U, 0, M, lut.numel(), DEV)
    graphed = RoutingPipeline(M, N, T, k, RB, C, U, 0, M, lut.numel(), DEV)
    tk = topk.clone()
    g = GraphStep(graphed.step, tk, lut, x)
    for seed in (21, 22):
        new, _ = routing_inputs(M, N, T, k, E, seed, 0, U)
        tk.copy_(new.to(DEV))
        eager.step(tk, lut, x)
        graphed.out.zero_()
        g()
        torch.cuda.synchronize()
        assert torch.equal(eager.sched.rem_off, graphed.sched.rem_off)
        assert torch.equal(eager.sched.send_load, graphed.sched.send_load)
        for kk in eager.final:
            assert torch.equal(eager.final[kk], graphed.final[kk])
        n = int(eager.total.item())
        assert torch.equal(eager.out[:n], graphed.out[:n])
