"""a6 fused with the finalize over peer memory (-m gpu, multi-rank).

P processes hold different source nodes of the same units (each
node schedules independently; the receive loads need every source node).
The fused rails_eval_finalize_peer (push partials to every rank, flag, wait,
reduce, finalize in one kernel) must give exactly what the collective all-reduce
followed by rails_eval_finalize gives -- reduced red_sum / red_max and every final
output -- over several calls (the call counter `gen` reuses the flags), also for
back-to-back calls on CHANGING inputs with no host synchronisation (the
double-buffered partials), and the finalize of every unit must match the oracle's
evaluation of the whole unit.

Runs on any box: all ranks on cuda:0 (gloo, CUDA-IPC on one device) always, and one
rank per GPU (NCCL, NVLink) when the box has enough GPUs (tests/mp_ranks.py).
"""
import numpy as np
import pytest
import torch

import gen
from mp_ranks import placements, run_ranks

pytestmark = pytest.mark.gpu


def _body(rank, world, dev, cfg):
    import oracle
    from helpers import oracle_eval_from_scheds
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.dist import PeerFinalize, make_reduce, shard_nodes
    from paper_2510_19262_b200.pipeline import MatrixPipeline
    M, N, C, U = cfg["M"], cfg["N"], cfg["C"], cfg["U"]
    d0, nd = shard_nodes(M, rank, world)
    gcfg = dict(gen.CONFIGS["c2"], M=M, N=N, V=cfg["V"])
    msg_all = [gen.d1_units(gcfg, gen.config_seed(2), 0, U),
               gen.d1_units(gcfg, gen.config_seed(2) + 1, 0, U)]
    msgs = [torch.from_numpy(m[:, d0:d0 + nd].copy()).to(dev) for m in msg_all]
    ref = MatrixPipeline(M, N, C, U, d0, nd, dev)
    fused = MatrixPipeline(M, N, C, U, d0, nd, dev)
    peer = PeerFinalize(fused.tp, U, dev)
    assert peer.ok(), peer.error
    coll = make_reduce()
    errors = []
    want = []
    for i in range(2):
        ref.step(msgs[i], coll)
        torch.cuda.synchronize()
        want.append(({k: v.clone() for k, v in ref.final.items()}, ref.ev.red_sum.clone(),
                     ref.ev.red_max.clone()))
    for it in range(3):  # gen 1, 2, 3, host-synchronised
        i = it % 2
        fused.step(msgs[i], peer)
        torch.cuda.synchronize()
        rails.check()
        fin, rs, rm = want[i]
        if not torch.equal(rs, fused.ev.red_sum):
            errors.append(f"it{it} red_sum")
        if not torch.equal(rm, fused.ev.red_max):
            errors.append(f"it{it} red_max")
        for kk in fin:
            if not torch.equal(fin[kk], fused.final[kk]):
                errors.append(f"it{it} {kk}")
    # back-to-back calls on alternating inputs, no host synchronisation: a call
    # that read the previous call's partials would give the other input's result
    got = []
    for it in range(20):
        fused.step(msgs[it % 2], peer)
        got.append({k: v.clone() for k, v in fused.final.items()})
    torch.cuda.synchronize()
    rails.check()
    for it, g in enumerate(got):
        fin = want[it % 2][0]
        for kk in fin:
            if not torch.equal(fin[kk], g[kk]):
                errors.append(f"back-to-back call {it} {kk}")
    if torch.equal(want[0][0]["T"], want[1][0]["T"]):
        errors.append("the two inputs must give different T (test is vacuous)")
    # the fused result against the oracle's evaluation of the whole unit
    for i in range(2):
        for u in range(U):
            scheds = [oracle.schedule_node(msg_all[i][u, d], C) for d in range(M)]
            ev = oracle_eval_from_scheds(M, N, msg_all[i][u], scheds)
            for kk in ("T", "T_star", "busbw", "T_e", "busbw_e"):
                g = float(got[18 + i][kk][u].item())
                w = float(ev[kk])
                if abs(g - w) > 1e-6 * max(abs(w), 1e-300):
                    errors.append(f"input{i} u{u} {kk} {g} vs {w}")
            for kk in ("maxload", "maxload_e", "total", "rowmax", "colmax"):
                if int(got[18 + i][kk][u].item()) != int(ev[kk]):
                    errors.append(f"input{i} u{u} {kk}")
    peer.close()
    return errors


@pytest.mark.parametrize("cfg", [
    dict(M=8, N=8, C=1 << 20, U=3, V=64 << 20, P=4),
    dict(M=5, N=4, C=65536, U=2, V=8 << 20, P=3),     # uneven node shards
    dict(M=4, N=8, C=32768, U=2, V=16 << 20, P=2),
])
def test_peer_finalize_matches_collective_and_oracle(cfg):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    for placement in placements(cfg["P"]):
        run_ranks(_body, cfg["P"], placement, cfg)
