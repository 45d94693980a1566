"""a6 fused with the finalize over NVLink peer memory (-m gpu, >= 2 GPUs).

P processes (one per GPU) hold different source nodes of the same units.  The
fused rails_eval_finalize_peer (push partials to every rank, flag, wait, reduce,
finalize in one kernel) must give exactly what the NCCL all-reduce followed by
rails_eval_finalize gives -- reduced red_sum / red_max and every final output --
over several calls (the call counter `gen` reuses the flags), and the finalize of
a full unit must match the oracle's eval.  Skipped on 1-GPU boxes.
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
    from helpers import R2, SEED, oracle_eval_from_scheds
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.dist import PeerFinalize, make_reduce, shard_nodes
    from paper_2510_19262_b200.pipeline import MatrixPipeline
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    M, N, C, U = cfg["M"], cfg["N"], cfg["C"], cfg["U"]
    d0, nd = shard_nodes(M, rank, world)
    gcfg = dict(gen.CONFIGS["c2"], M=M, N=N, V=cfg["V"])
    msg_all = gen.d1_units(gcfg, gen.config_seed(2), 0, U)
    msg = torch.from_numpy(msg_all[:, d0:d0 + nd].copy()).to(dev)
    ref = MatrixPipeline(M, N, C, U, d0, nd, dev)
    fused = MatrixPipeline(M, N, C, U, d0, nd, dev)
    peer = PeerFinalize(fused.tp, U, dev)
    nccl = make_reduce()
    errors = []
    for it in range(3):  # gen 1, 2, 3
        ref.step(msg, nccl)
        fused.step(msg, peer)
        torch.cuda.synchronize()
        rails.check()
        if not torch.equal(ref.ev.red_sum, fused.ev.red_sum):
            errors.append(f"it{it} red_sum")
        if not torch.equal(ref.ev.red_max, fused.ev.red_max):
            errors.append(f"it{it} red_max")
        for kk in ref.final:
            if not torch.equal(ref.final[kk], fused.final[kk]):
                errors.append(f"it{it} {kk}")
    # back-to-back calls with no host synchronisation (double-buffered partials,
    # monotonic flags): still identical to the NCCL reference
    for _ in range(20):
        fused.step(msg, peer)
    torch.cuda.synchronize()
    rails.check()
    for kk in ref.final:
        if not torch.equal(ref.final[kk], fused.final[kk]):
            errors.append(f"back-to-back {kk}")
    # the fused result against the oracle's evaluation of the whole unit
    for u in range(U):
        scheds = [oracle.schedule_node(msg_all[u, d], C) for d in range(M)]
        ev = oracle_eval_from_scheds(M, N, msg_all[u], scheds)
        for kk in ("T", "T_star", "busbw"):
            got = float(fused.final[kk][u].item())
            want = float(ev[kk])
            if abs(got - want) > 1e-6 * max(abs(want), 1e-300):
                errors.append(f"u{u} {kk} {got} vs {want}")
    q.put((rank, errors))
    peer.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    dict(M=8, N=8, C=1 << 20, U=3, V=64 << 20),
    dict(M=5, N=4, C=65536, U=2, V=8 << 20),     # uneven node shards
])
def test_peer_finalize_matches_nccl_and_oracle(cfg):
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(ngpu, 4, cfg["M"])
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
