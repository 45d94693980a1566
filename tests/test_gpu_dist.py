"""Sharded GPU path with the real a6 reduction hook (-m gpu).

Two processes share cuda:0 (gloo carries the reduction of CUDA tensors through
the host; NCCL refuses two ranks on one GPU), each runs the CUDA pipeline on its
block of source nodes for U = 2 units, all-reduces with paper_2510_19262_b200.dist
.make_reduce, finalizes, and must reproduce the single-process results exactly.
The N>1 NCCL launch itself is exercised by bench.py under torchrun.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import gen

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, M, N, T, k, E, RB, C, U, q):
    import torch.distributed as dist

    from paper_2510_19262_b200.dist import make_reduce, shard_nodes
    from paper_2510_19262_b200.pipeline import RoutingPipeline
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = "cuda:0"
    d0, nd = shard_nodes(M, rank, world)
    seed = 77
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u, d0, nd, device=dev) for u in range(U)])
    lut = gen.inst_lut(M, N, E).to(dev)
    x = torch.stack([gen.payload(M, N, T, RB, seed, u, d0, nd, device=dev) for u in range(U)])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), dev)
    pipe.step(topk, lut, x, reduce=make_reduce())
    torch.cuda.synchronize()
    res = {kk: v.cpu().numpy() for kk, v in pipe.final.items()}
    res["send_load"] = pipe.sched.send_load.cpu().numpy()
    res["d0"] = d0
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_sharded_pipeline_matches_single():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2510_19262_b200.pipeline import RoutingPipeline
    M, N, T, k, E, RB, C, U = 6, 4, 300, 2, 8, 1024, 4096, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, N, T, k, E, RB, C, U, q))
             for r in range(2)]
    for p in procs:
        p.start()
    import queue
    import time
    got = {}
    t_end = time.time() + 300
    while len(got) < 2 and time.time() < t_end:
        try:
            r, res = q.get(timeout=5)
            got[r] = res
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert len(got) == 2, f"workers failed: exit codes {[p.exitcode for p in procs]}"
    dev = "cuda:0"
    seed = 77
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u, device=dev) for u in range(U)])
    lut = gen.inst_lut(M, N, E).to(dev)
    x = torch.stack([gen.payload(M, N, T, RB, seed, u, 0, M, device=dev) for u in range(U)])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, 0, M, lut.numel(), dev)
    pipe.step(topk, lut, x)
    torch.cuda.synchronize()
    for r in (0, 1):
        for key, v in pipe.final.items():
            assert np.array_equal(got[r][key], v.cpu().numpy()), (r, key)
        d0 = got[r]["d0"]
        nd = got[r]["send_load"].shape[1]
        assert np.array_equal(got[r]["send_load"], pipe.sched.send_load[:, d0:d0 + nd].cpu().numpy())
