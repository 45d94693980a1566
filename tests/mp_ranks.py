"""Run a multi-rank GPU test body as P spawned processes, one per GPU ("per_gpu":
rank r on cuda:r, process group over NCCL; CUDA-IPC mappings and NVLink stores).

Ranks whose kernels wait on each other's flags must never share one GPU as separate
processes (nothing guarantees their kernels run concurrently; on this driver it has
raised Xid 109): the single-GPU variants of the multi-rank tests play every rank in
one process with the *_local cooperative launches instead.  `placement` "shared"
(gloo, every rank on cuda:0) is only for bodies without cross-rank waits.
"""
from __future__ import annotations

import os
import queue
import socket
import time
import traceback

import torch
import torch.multiprocessing as mp


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(body, rank, world, port, placement, cfg, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dev_index = rank if placement == "per_gpu" else 0
        torch.cuda.set_device(dev_index)
        dev = torch.device("cuda", dev_index)
        if placement == "per_gpu":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        errors = body(rank, world, dev, cfg)
        q.put((rank, errors))
        dist.barrier()
        dist.destroy_process_group()
    except BaseException:
        q.put((rank, ["EXC " + traceback.format_exc()]))
        raise


def run_ranks(body, world: int, placement: str, cfg: dict, timeout_s: float = 900.0):
    """Spawn `world` ranks running body(rank, world, device, cfg) -> list of error
    strings; assert every rank reported and none reported an error.  A rendezvous
    port taken between picking it and binding it (EADDRINUSE) is retried on a new
    port."""
    for attempt in range(3):
        res, procs = _spawn(body, world, placement, cfg, timeout_s)
        taken = any("EADDRINUSE" in e for errs in res.values() for e in errs)
        if not taken or attempt == 2:
            break
    for r, errs in res.items():
        assert not errs, (placement, r, errs)
    assert len(res) == world, f"{placement}: workers exit codes {[p.exitcode for p in procs]}"


def _spawn(body, world, placement, cfg, timeout_s):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_entry, args=(body, r, world, port, placement, cfg, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    t_end = time.time() + timeout_s
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
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    return res, procs
