#!/usr/bin/env python
"""NEXT f4 benchmark and report: batched fluid simulations on the GPU.

One all-to-all round per simulation, every (workload family, unit, policy) of the
batch in ONE rails_flowsim launch sequence (one CTA per simulation).  Reports the
batch time (CUDA events), simulations/s and completion events/s, the oracle's
single-core time on a bounded sample of the same simulations, and the paper-style
comparison: BusBw normalised to ECMP and CCT percentiles normalised to
RailS's mean, per workload family.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402

DEV = "cuda:0"
POLS = ["lpt", "uniform", "ecmp", "reps", "minrtt", "plb"]


def family_msg(fam, M, N, V, seed, u):
    if fam == "uniform":
        return gen.d1_uniform(M, N, V)
    if fam.startswith("sparse"):
        return gen.d1_sparse_topk(M, N, V, float(fam.split("-")[1]), 2, seed, u)
    if fam == "sender":
        return gen.d1_sender_skew(M, N, V, 1.2, seed, u)
    return gen.d1_receiver_skew(M, N, V, 1.2, seed, u)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--N", type=int, default=8)
    ap.add_argument("--S", type=int, default=None)
    ap.add_argument("--V", type=int, default=16 << 20, help="bytes per source GPU")
    ap.add_argument("--C", type=int, default=32768)
    ap.add_argument("--units", type=int, default=2)
    ap.add_argument("--families", default="uniform,sparse-0.6,sparse-0.4,sparse-0.2,sparse-0,"
                                          "sender,receiver")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--oracle", type=int, default=5, help="oracle sample: simulations timed")
    ap.add_argument("--rs", type=float, default=None, help="leaf-spine rate / R2 (default M/S)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    M, N, C = a.M, a.N, a.C
    S = N if a.S is None else a.S
    R2 = 5.0e10
    fams = a.families.split(",")
    seed = gen.config_seed(6)
    msgs, pols, keys = [], [], []
    for fam in fams:
        for u in range(a.units):
            m = family_msg(fam, M, N, a.V, seed, u)
            for p in POLS:
                msgs.append(m)
                pols.append(rails.FS_POLICIES[p])
                keys.append((fam, u, p))
    tp = rails.topo(M, N, C, R2=R2)
    fb = rails.fabric(M, N, R2, S=S, Rs=None if a.rs is None else a.rs * R2)
    msg_t = torch.from_numpy(np.stack(msgs)).to(DEV)
    pol_t = torch.tensor(pols, dtype=torch.int32, device=DEV)
    rails.flowsim(tp, fb, pol_t, msg_t)  # warm-up (also sizes the workspace)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cct, lb, st = rails.flowsim(tp, fb, pol_t, msg_t)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    rails.check()
    st = st.cpu().numpy()
    ms = min(ts)
    n_sim = len(keys)
    ev = float(st[:, 8].sum())
    res = {"M": M, "N": N, "S": S, "Rs_over_R2": fb.Rs / R2, "V": a.V, "C": C, "units": a.units,
           "families": fams,
           "n_sim": n_sim, "batch_ms": ms, "sims_per_s": n_sim / (ms / 1e3),
           "events": ev, "events_per_s": ev / (ms / 1e3),
           "flows": float(st[:, 9].sum()), "max_sim_events": float(st[:, 8].max())}
    # paper-style comparison, averaged over units
    rep = {}
    for fam in fams:
        row = {}
        for p in POLS:
            idx = [i for i, k in enumerate(keys) if k[0] == fam and k[2] == p]
            row[p] = {s: float(np.mean(st[idx, j])) for j, s in enumerate(rails.FS_STATS)}
        base_bw = row["ecmp"]["busbw"]
        base_cct = row["lpt"]["cct_mean"]
        for p in POLS:
            r = row[p]
            r["busbw_over_ecmp"] = r["busbw"] / base_bw if base_bw else None
            for q in ("cct_mean", "cct_p80", "cct_p95", "cct_p99"):
                r[q + "_over_rails_mean"] = r[q] / base_cct if base_cct else None
        rep[fam] = row
    res["report"] = rep
    # oracle on a bounded sample of the same simulations (single core)
    if a.oracle > 0:
        import oracle
        sample = list(range(0, n_sim, max(1, n_sim // a.oracle)))[:a.oracle]
        t0 = time.perf_counter()
        for i in sample:
            oracle.flowsim(M, N, S, fb.R1, R2, fb.Rs, C, pols[i], msgs[i])
        dt = time.perf_counter() - t0
        res["oracle_sample"] = [keys[i] for i in sample]
        res["oracle_s"] = dt
        res["oracle_sims_per_s"] = len(sample) / dt
        res["oracle_events"] = float(st[sample, 8].sum())
        res["oracle_events_per_s"] = res["oracle_events"] / dt
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
