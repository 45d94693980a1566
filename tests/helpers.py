"""Shared test helpers: run the oracle and the CUDA path on the same seeded inputs."""
from __future__ import annotations

import numpy as np
import torch

import gen
import oracle

R2 = 5.0e10
SEED = 0x9E3779B97F4A7C15


def oracle_schedule_unit_nodes(msg_unit_nodes: np.ndarray, C: int):
    """Per node (axis 0) oracle schedule dicts."""
    return [oracle.schedule_node(msg_unit_nodes[i], C) for i in range(msg_unit_nodes.shape[0])]


def compare_schedule(gpu_sched, u: int, dl: int, orc: dict, where: str = ""):
    fb = gpu_sched.full_base[u, dl].cpu().numpy()
    rr = gpu_sched.rem_rail[u, dl].cpu().numpy()
    ro = gpu_sched.rem_off[u, dl].cpu().numpy()
    sl = gpu_sched.send_load[u, dl].cpu().numpy()
    nf = int(gpu_sched.n_full[u, dl])
    nr = int(gpu_sched.n_rem[u, dl])
    assert nf == orc["n_full"], f"{where} n_full {nf} != {orc['n_full']}"
    assert nr == orc["n_rem"], f"{where} n_rem {nr} != {orc['n_rem']}"
    assert np.array_equal(fb, orc["full_base"]), f"{where} full_base"
    assert np.array_equal(rr, orc["rem_rail"]), f"{where} rem_rail"
    assert np.array_equal(ro, orc["rem_off"]), f"{where} rem_off"
    assert np.array_equal(sl, orc["send_load"]), f"{where} send_load"


def oracle_eval_from_scheds(M, N, msg_unit, scheds, R2=R2, seed=SEED):
    cd, chh, cs, cr = [], [], [], []
    for d, s in enumerate(scheds):
        F = len(s["chunks"]["size"])
        cd.append(np.full(F, d, np.int32)); chh.append(s["chunks"]["h"])
        cs.append(s["chunks"]["size"]); cr.append(s["rail"])
    ev = oracle.eval_unit(M, N, R2, seed, msg_unit, np.concatenate(cd), np.concatenate(chh),
                          np.concatenate(cs), np.concatenate(cr))
    ev.update(oracle.eval_uniform(M, N, R2, msg_unit))  # S_u, R_u, maxload_u, T_u, busbw_u
    return ev


def rel_err(a: float, b: float) -> float:
    if a == b:
        return 0.0
    return abs(a - b) / max(abs(a), abs(b))


def random_msg(rng, U, M, N, p=0.6, hi=200000, mult=1, nodes=None):
    G = M * N
    nodes = range(M) if nodes is None else nodes
    nodes = list(nodes)
    msg = (rng.integers(1, hi, size=(U, len(nodes), N, G)) * mult) * (
        rng.random((U, len(nodes), N, G)) < p)
    for i, d in enumerate(nodes):
        msg[:, i, :, d * N:(d + 1) * N] = 0
    return msg.astype(np.int64)


def routing_inputs(M, N, T, k, E, seed, u0, U, device="cpu"):
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u0 + u, device=device) for u in range(U)])
    lut = gen.inst_lut(M, N, E).to(device)
    return topk, lut
