"""Randomised parity sweep (-m gpu): seeded random topologies, chunk sizes, traffic
shapes and shards through schedule + eval (byte matrices) and histogram + schedule
+ pack (routing), each compared with the oracle -- bit-exact integers, floats within
1e-6.  Complements the hand-picked cases of test_gpu_parity.py with shapes nobody
chose (odd N, non-power-of-two C, ragged shards, equal-size runs, empty nodes)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import (compare_schedule, oracle_eval_from_scheds, random_msg, rel_err,
                     routing_inputs)

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import MatrixPipeline, RoutingPipeline

DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    rails.check()


def _matrix(rng, U, M, N):
    G = M * N
    kind = rng.integers(0, 4)
    if kind == 0:    # random sizes
        msg = rng.integers(1, int(rng.choice([50, 5000, 3_000_000])), size=(U, M, N, G))
    elif kind == 1:  # row multiples: long runs of equal remainders
        msg = rng.integers(0, 30, size=(U, M, N, G)) * int(rng.choice([48, 4096, 12288]))
    elif kind == 2:  # one size for everything
        msg = np.full((U, M, N, G), int(rng.integers(1, 100000)))
    else:            # sparse rows, some nodes silent
        msg = rng.integers(1, 1_000_000, size=(U, M, N, G)) * (rng.random((U, M, N, G)) < 0.1)
        msg[:, rng.integers(0, M)] = 0
    msg = msg * (rng.random((U, M, N, G)) < rng.uniform(0.3, 1.0))
    for d in range(M):
        msg[:, d, :, d * N:(d + 1) * N] = 0
    return msg.astype(np.int64)


@pytest.mark.parametrize("seed", range(32))
def test_fuzz_schedule_eval(seed):
    rng = np.random.default_rng(1000 + seed)
    M = int(rng.integers(2, 13))
    N = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 16]))
    C = int(rng.choice([1, 16, 100, 1000, 4096, 65536, 1 << 20, 12345]))
    U = int(rng.integers(1, 4))
    msg = _matrix(rng, U, M, N)
    d0 = int(rng.integers(0, M))
    nd = int(rng.integers(1, M - d0 + 1))
    tp, sh = rails.topo(M, N, C), rails.shard(U, d0, nd)
    s = rails.lpt_schedule(tp, sh, torch.from_numpy(msg[:, d0:d0 + nd].copy()).to(DEV))
    scheds = {}
    for u in range(U):
        for dl in range(nd):
            o = oracle.schedule_node(msg[u, d0 + dl], C)
            scheds[(u, dl)] = o
            compare_schedule(s, u, dl, o, f"seed{seed} u{u} d{d0 + dl}")
    # eval of whole units (all nodes) against the oracle
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    for u in range(U):
        ev = oracle_eval_from_scheds(M, N, msg[u], [oracle.schedule_node(msg[u, d], C)
                                                     for d in range(M)])
        assert int(pipe.final["maxload"][u]) == ev["maxload"]
        assert int(pipe.final["total"][u]) == ev["total"]
        for k in ("T", "T_star", "busbw", "T_e", "busbw_e"):
            assert rel_err(float(pipe.final[k][u]), ev[k]) <= 1e-6, (seed, k)


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_routing_pack(seed):
    from test_gpu_parity import _oracle_pack_check
    rng = np.random.default_rng(2000 + seed)
    M = int(rng.integers(2, 7))
    N = int(rng.choice([1, 2, 3, 4, 8]))
    E = int(rng.integers(max(2, N), 3 * N + 3))
    k = int(rng.integers(1, min(E, 4) + 1))
    T = int(rng.integers(1, 300))
    RB = 16 * int(rng.integers(1, 300))
    C = 16 * int(rng.integers(1, 2000))
    U = int(rng.integers(1, 3))
    topk_all, lut = routing_inputs(M, N, T, k, E, 50 + seed, 0, U)
    d0 = int(rng.integers(0, M))
    nd = int(rng.integers(1, M - d0 + 1))
    topk = topk_all[:, d0:d0 + nd].contiguous()
    x = torch.stack([gen.payload(M, N, T, RB, 9, u, d0, nd) for u in range(U)])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), DEV)
    pipe.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
    torch.cuda.synchronize()
    for u in range(U):
        for dl in range(nd):
            _oracle_pack_check(pipe, topk, lut, x, u, dl)


@pytest.mark.parametrize("C,mult", [(65536, 4096), (65536, 12288), (32768, 8192),
                                    (1 << 20, 3 << 14), (4096, 1), (65536, 1 << 15)])
def test_many_segments_narrow_digits(C, mult):
    """Message sizes on a granule (routing: multiples of the row size), so the
    remainder keys vary in a few bits only and the many-segment sort runs 1-8-bit
    digit passes over just those bits (radix.cuh radix_sort_narrow); with the
    expand pass inside the evaluation.  Exact against the oracle on sampled units."""
    rng = np.random.default_rng(C + mult)
    M, N = 4, 8
    U = 2 * 148 // M + 7  # > 2 x the SM count of segments: k_chains.cu
    msg = random_msg(rng, U, M, N, p=0.7, hi=40, mult=mult)
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    for u in rng.choice(U, size=4, replace=False):
        scheds = [oracle.schedule_node(msg[u, d], C) for d in range(M)]
        for d in range(M):
            compare_schedule(pipe.sched, u, d, scheds[d], f"C{C} mult{mult} u{u} d{d}")
        ev = oracle_eval_from_scheds(M, N, msg[u], scheds)
        assert np.array_equal(pipe.ev.S[u].cpu().numpy(), ev["S"])
        for k in ("maxload", "maxload_e", "maxload_u", "total"):
            assert int(pipe.final[k][u]) == ev[k], (C, mult, k)


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_many_segments(seed):
    """More (unit, node) segments than 2 x the SM count: the per-phase kernels of
    k_chains.cu schedule them and rails_eval's kernel evaluates them (the fused
    per-node kernel covers the few-segment shapes above) -- same outputs."""
    rng = np.random.default_rng(3000 + seed)
    M = int(rng.integers(2, 6))
    N = int(rng.choice([1, 3, 4, 8, 8, 8]))
    C = int(rng.choice([7, 100, 4096, 32768, 1 << 20]))
    U = int(rng.integers(320 // M + 1, 700 // M + 2))
    msg = _matrix(rng, U, M, N)
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    for u in rng.choice(U, size=6, replace=False):
        scheds = [oracle.schedule_node(msg[u, d], C) for d in range(M)]
        for d in range(M):
            compare_schedule(pipe.sched, u, d, scheds[d], f"seed{seed} u{u} d{d}")
        ev = oracle_eval_from_scheds(M, N, msg[u], scheds)
        assert np.array_equal(pipe.ev.S[u].cpu().numpy(), ev["S"])
        assert np.array_equal(pipe.ev.S_u[u].cpu().numpy(), ev["S_u"])
        for k in ("maxload", "maxload_e", "maxload_u", "total"):
            assert int(pipe.final[k][u]) == ev[k], (seed, k)
        for k in ("T", "T_star", "busbw", "T_e", "busbw_e", "T_u", "busbw_u"):
            assert rel_err(float(pipe.final[k][u]), ev[k]) <= 1e-6, (seed, k)
