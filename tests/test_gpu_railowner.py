"""NEXT f2 -- rail-owner pack fused with the intra-node NVLink hop (-m gpu, >= 2 GPUs).

P processes (one per GPU, NCCL) form one RailS node: each packs its own source GPUs'
rows into the rail buffers owned by the other GPUs through peer pointers.  Every
owned rail buffer must equal, byte for byte, the oracle's rail buffer of the node
(oracle.pack_node on all N source GPUs, by definition).  Skipped on 1-GPU boxes.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import gen

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import traceback
    try:
        _worker_body(rank, world, port, cfg, q)
    except BaseException:
        q.put((rank, ["EXC " + traceback.format_exc()]))
        raise


def _worker_body(rank, world, port, cfg, q):
    import torch.distributed as dist

    import oracle
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.railowner import RailOwnerNode
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    M, N, T, k, E, RB, C, U, d = (cfg[x] for x in "M N T k E RB C U d".split())
    dev = torch.device("cuda", rank)
    seed = 31
    topk_all = torch.stack([gen.routing(M, N, T, k, E, seed, u, d, 1) for u in range(U)])
    x_all = torch.stack([gen.payload(M, N, T, RB, seed, u, d, 1) for u in range(U)])
    lut = gen.inst_lut(M, N, E)
    node = RailOwnerNode(M, N, T, k, RB, C, U, d, lut.numel(), exchange=cfg.get("ex", "peer"))
    g0, ng = node.g0, node.ng
    topk = topk_all[:, :, g0:g0 + ng].contiguous().to(dev)
    x = x_all[:, :, g0:g0 + ng].contiguous().to(dev)
    node.buf.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    node.step(topk, lut.to(dev), x)
    node.buf.zero_()  # a second step re-gathers and re-packs (flags reused, gen 2)
    torch.cuda.synchronize()
    dist.barrier()
    node.step(topk, lut.to(dev), x)
    torch.cuda.synchronize()
    rails.check()
    errors = []
    for u in range(U):
        c, m, r = oracle.histogram_node(M, N, d, T, k, topk_all[u, 0].numpy(), lut.numpy(), RB)
        s = oracle.schedule_node(m, C)
        L = s["send_load"]
        base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
        want = oracle.pack_node(M, N, d, T, k, RB, C, x_all[u, 0].numpy().view(np.uint8),
                                topk_all[u, 0].numpy(), lut.numpy(), m, s, base, int(L.sum()))
        if not np.array_equal(node.sched.send_load[u, 0].cpu().numpy(), L):
            errors.append(f"u{u} send_load")
        rb = node.rail_base[u, 0].cpu().numpy()
        for j in range(g0, g0 + ng):
            got = node.own_rail(j)[int(rb[j]):int(rb[j]) + int(L[j])].cpu().numpy()
            if not np.array_equal(got, want[base[j]:base[j] + L[j]]):
                errors.append(f"u{u} rail{j}")
    q.put((rank, errors))
    node.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1),   # 2-piece path
    dict(M=3, N=4, T=128, k=2, E=6, RB=2048, C=1024, U=1, d=2),   # C < RB multi-piece
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1, ex="nccl"),  # NCCL exchange
    dict(M=3, N=4, T=100, k=2, E=8, RB=12288, C=32768, U=1, d=0),  # 12 KiB rows: windows
])
def test_railowner_pack_matches_oracle(cfg):
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if ngpu >= 4 and cfg["N"] % 4 == 0 else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res = {}
    t_end = time.time() + 600
    while len(res) < world and time.time() < t_end:
        try:
            r, errs = q.get(timeout=5)
            res[r] = errs
            if any(e.startswith("EXC") for e in errs):
                break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    for r, errs in res.items():
        assert not errs, (r, errs)
    assert len(res) == world, f"workers: exit codes {[p.exitcode for p in procs]}"
