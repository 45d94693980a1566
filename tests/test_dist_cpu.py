"""N > 1 host logic on CPU: world_size-2 gloo processes shard the nodes of each unit,
build their partial reduction buffers (from the oracle, standing in for the GPU
kernels that fill the same layout), all-reduce them with the same a6 hook the
GPU path uses, and must reproduce the unsharded buffers exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2510_19262_b200.dist import make_reduce, shard_nodes, weak_units

R2 = 5.0e10
SEED = oracle.DEFAULT_ECMP_SEED


def partial_buffers(msg_unit, M, N, C, d0, nd):
    """Layout of include/rails.h: red_sum = R[M][N], R_e[M][N], colsum[M], total,
    total_e; red_max = max S, max S_e, rowmax, 0 -- over nodes d0..d0+nd-1."""
    cd, chh, cs, cr = [], [], [], []
    sub = np.zeros_like(msg_unit)
    sub[d0:d0 + nd] = msg_unit[d0:d0 + nd]
    for d in range(d0, d0 + nd):
        s = oracle.schedule_node(msg_unit[d], C)
        F = len(s["chunks"]["size"])
        cd.append(np.full(F, d, np.int32)); chh.append(s["chunks"]["h"])
        cs.append(s["chunks"]["size"]); cr.append(s["rail"])
    ev = oracle.eval_unit(M, N, R2, SEED, sub, np.concatenate(cd), np.concatenate(chh),
                          np.concatenate(cs), np.concatenate(cr))
    col = sub.reshape(M, N, M, N).sum(axis=(0, 1, 3))
    rs = np.concatenate([ev["R"].ravel(), ev["R_e"].ravel(), col, [ev["total"], ev["total_e"]]])
    S, Se = ev["S"][d0:d0 + nd], ev["S_e"][d0:d0 + nd]
    rm = np.array([S.max(initial=0), Se.max(initial=0), S.sum(axis=1).max(initial=0), 0])
    return rs.astype(np.int64), rm.astype(np.int64)


def _worker(rank, world, port, msg, M, N, C, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    U = msg.shape[0]
    d0, nd = shard_nodes(M, rank, world)
    rs = torch.zeros((U, 2 * M * N + M + 2), dtype=torch.int64)
    rm = torch.zeros((U, 4), dtype=torch.int64)
    for u in range(U):
        a, b = partial_buffers(msg[u], M, N, C, d0, nd)
        rs[u] = torch.from_numpy(a)
        rm[u] = torch.from_numpy(b)
    make_reduce()(rs, rm)
    if rank == 0:
        q.put((rs.numpy(), rm.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_nodes_cover_exactly():
    for M in (2, 7, 64, 128):
        for world in (1, 2, 3, 4, 8):
            if world > M:
                continue
            blocks = [shard_nodes(M, r, world) for r in range(world)]
            covered = [d for d0, nd in blocks for d in range(d0, d0 + nd)]
            assert covered == list(range(M))
    assert weak_units(8) == 8


def test_gloo_two_ranks_reduce_matches_unsharded():
    rng = np.random.default_rng(3)
    M, N, C, U = 5, 3, 4096, 2
    G = M * N
    msg = rng.integers(1, 50000, size=(U, M, N, G)) * (rng.random((U, M, N, G)) < 0.6)
    for d in range(M):
        msg[:, d, :, d * N:(d + 1) * N] = 0
    msg = msg.astype(np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, msg, M, N, C, q)) for r in range(2)]
    for p in procs:
        p.start()
    rs, rm = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for u in range(U):
        a, b = partial_buffers(msg[u], M, N, C, 0, M)
        assert np.array_equal(rs[u], a)
        assert np.array_equal(rm[u], b)
