"""a6 fused with the finalize over peer memory (-m gpu, multi-rank).

P ranks hold different source nodes of the same units (each node
schedules independently; the receive loads need every source node).  The
fused peer finalize (push partials to every rank, flag, wait, reduce, finalize in
one kernel) must give exactly what the one-shot evaluation of all nodes gives --
the reduced red_sum / red_max and every final output -- over several calls (the
call counter `gen` reuses the flags), also back to back on CHANGING inputs with no
host synchronisation (the double-buffered partials), and every unit's finalize must
match the oracle's evaluation of the whole unit.

* test_peer_finalize_local_ranks (any box): the P ranks are played by this process
  on cuda:0 through rails_eval_finalize_peer_local -- the same kernel, ONE
  cooperative launch whose CTA (u, p) is rank p, so the ranks' flag waits run
  co-resident (spinning kernels in separate processes sharing one GPU are not
  guaranteed to run concurrently; see include/rails.h).
* test_peer_finalize_per_gpu (boxes with >= P GPUs): one process per GPU, CUDA-IPC
  mappings, NVLink stores, checked against the NCCL all-reduce + finalize.
"""
import numpy as np
import pytest
import torch

import gen
from mp_ranks import run_ranks

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
CFGS = [
    dict(M=8, N=8, C=1 << 20, U=3, V=64 << 20, P=4),
    dict(M=5, N=4, C=65536, U=2, V=8 << 20, P=3),     # uneven node shards
    dict(M=4, N=8, C=32768, U=2, V=16 << 20, P=2),
    dict(M=16, N=8, C=1 << 20, U=2, V=32 << 20, P=8),
]


def _inputs(cfg):
    M, N, U = cfg["M"], cfg["N"], cfg["U"]
    gcfg = dict(gen.CONFIGS["c2"], M=M, N=N, V=cfg["V"])
    return [gen.d1_units(gcfg, gen.config_seed(2), 0, U),
            gen.d1_units(gcfg, gen.config_seed(2) + 1, 0, U)]


def _check_oracle(cfg, msg_all, finals, errors):
    import oracle
    from helpers import oracle_eval_from_scheds
    M, N, C, U = cfg["M"], cfg["N"], cfg["C"], cfg["U"]
    for i in range(2):
        for u in range(U):
            scheds = [oracle.schedule_node(msg_all[i][u, d], C) for d in range(M)]
            ev = oracle_eval_from_scheds(M, N, msg_all[i][u], scheds)
            for kk in ("T", "T_star", "busbw", "T_e", "busbw_e", "T_u", "busbw_u"):
                g = float(finals[i][kk][u].item())
                w = float(ev[kk])
                if abs(g - w) > 1e-6 * max(abs(w), 1e-300):
                    errors.append(f"input{i} u{u} {kk} {g} vs {w}")
            for kk in ("maxload", "maxload_e", "maxload_u", "total", "rowmax", "colmax"):
                if int(finals[i][kk][u].item()) != int(ev[kk]):
                    errors.append(f"input{i} u{u} {kk}")


@pytest.mark.parametrize("cfg", CFGS)
def test_peer_finalize_local_ranks(cfg):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.dist import shard_nodes
    from paper_2510_19262_b200.pipeline import MatrixPipeline
    dev = torch.device("cuda", 0)
    M, N, C, U, P = cfg["M"], cfg["N"], cfg["C"], cfg["U"], cfg["P"]
    msg_all = _inputs(cfg)
    ref = MatrixPipeline(M, N, C, U, 0, M, dev)  # every node in one call
    want = []
    for i in range(2):
        ref.step(torch.from_numpy(msg_all[i]).to(dev))
        torch.cuda.synchronize()
        want.append(({k: v.clone() for k, v in ref.final.items()}, ref.ev.red_sum.clone(),
                     ref.ev.red_max.clone()))
    ranks = []
    for p in range(P):
        d0, nd = shard_nodes(M, p, P)
        pipe = MatrixPipeline(M, N, C, U, d0, nd, dev)
        ranks.append((pipe, [torch.from_numpy(m[:, d0:d0 + nd].copy()).to(dev) for m in msg_all]))
    nbuf = rails.peer_buffer_bytes(ranks[0][0].tp, U, P)
    bufs = [torch.zeros(nbuf, dtype=torch.uint8, device=dev) for _ in range(P)]
    ptrs = [b.data_ptr() for b in bufs]
    gen_ = [0]

    def step(i):
        for pipe, msgs in ranks:  # each rank's partial evaluation of its own nodes
            rails.schedule_eval(pipe.tp, pipe.sh, msgs[i], pipe.sched, pipe.ev, pipe.ws)
        gen_[0] += 1
        rails.eval_finalize_peer_local(ranks[0][0].tp, U, [r[0].ev.red_sum for r in ranks],
                                       [r[0].ev.red_max for r in ranks], gen_[0], ptrs,
                                       [r[0].final for r in ranks])

    errors = []
    for it in range(3):  # host-synchronised calls, gen 1..3
        i = it % 2
        step(i)
        torch.cuda.synchronize()
        rails.check()
        fin, rs, rm = want[i]
        for p, (pipe, _) in enumerate(ranks):
            if not torch.equal(rs, pipe.ev.red_sum):
                errors.append(f"it{it} rank{p} red_sum")
            if not torch.equal(rm, pipe.ev.red_max):
                errors.append(f"it{it} rank{p} red_max")
            for kk in fin:
                if not torch.equal(fin[kk], pipe.final[kk]):
                    errors.append(f"it{it} rank{p} {kk}")
    # back to back on alternating inputs, no host synchronisation: a call that read
    # the previous call's partials would give the other input's result
    got = []
    for it in range(20):
        step(it % 2)
        got.append([{k: v.clone() for k, v in pipe.final.items()} for pipe, _ in ranks])
    torch.cuda.synchronize()
    rails.check()
    for it, g in enumerate(got):
        fin = want[it % 2][0]
        for p in range(P):
            for kk in fin:
                if not torch.equal(fin[kk], g[p][kk]):
                    errors.append(f"back-to-back call {it} rank{p} {kk}")
    if torch.equal(want[0][0]["T"], want[1][0]["T"]):
        errors.append("the two inputs must give different T (test is vacuous)")
    _check_oracle(cfg, msg_all, [got[18][P - 1], got[19][0]], errors)
    assert not errors, errors


def _body(rank, world, dev, cfg):
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.dist import PeerFinalize, make_reduce, shard_nodes
    from paper_2510_19262_b200.pipeline import MatrixPipeline
    M, N, C, U = cfg["M"], cfg["N"], cfg["C"], cfg["U"]
    d0, nd = shard_nodes(M, rank, world)
    msg_all = _inputs(cfg)
    msgs = [torch.from_numpy(m[:, d0:d0 + nd].copy()).to(dev) for m in msg_all]
    ref = MatrixPipeline(M, N, C, U, d0, nd, dev)
    fused = MatrixPipeline(M, N, C, U, d0, nd, dev)
    peer = PeerFinalize(fused.tp, U, dev)
    assert peer.ok(), peer.error
    coll = make_reduce()
    errors, want = [], []
    for i in range(2):
        ref.step(msgs[i], coll)
        torch.cuda.synchronize()
        want.append({k: v.clone() for k, v in ref.final.items()})
    got = []
    for it in range(20):  # back to back, alternating inputs
        fused.step(msgs[it % 2], peer)
        got.append({k: v.clone() for k, v in fused.final.items()})
    torch.cuda.synchronize()
    rails.check()
    for it, g in enumerate(got):
        for kk in g:
            if not torch.equal(want[it % 2][kk], g[kk]):
                errors.append(f"call {it} {kk}")
    _check_oracle(cfg, msg_all, [got[18], got[19]], errors)
    peer.close()
    return errors


if NGPU >= 2:
    @pytest.mark.parametrize("cfg", [c for c in CFGS if c["P"] <= NGPU])
    def test_peer_finalize_per_gpu(cfg):
        run_ranks(_body, cfg["P"], "per_gpu", cfg)
