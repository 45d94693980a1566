#!/usr/bin/env python
"""BASELINE config 5: chunk-granularity sweep 4 KiB - 4 MiB at 256 nodes x 8 rails.

For each chunk size C (11 points, 4 KiB << i): the receiver-skewed Zipf D^(1) of
C5 (one unit, every node) through schedule + eval on the GPU -- CUDA-event time of
the step, (unit, node) schedules per second, remainders per node -- and the
method's quality: T_LPT / T*, T_ECMP / T* and busbw LPT / ECMP.  Two nodes per
point are re-scheduled by the CPU oracle and compared exactly (a spot check; the
full parity suite is tests/test_gpu_parity.py)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402
from paper_2510_19262_b200.pipeline import MatrixPipeline  # noqa: E402

DEV = "cuda:0"


def timed(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--check-nodes", type=int, default=2)
    a = ap.parse_args()
    import oracle
    cfg = gen.CONFIGS["c5"]
    M, N = cfg["M"], cfg["N"]
    msg_np = gen.d1_units(cfg, gen.config_seed(5), 0, 1)
    msg = torch.from_numpy(msg_np).to(DEV)
    rows = []
    for C in cfg["C_sweep"]:
        pipe = MatrixPipeline(M, N, C, 1, 0, M, DEV)
        ms = timed(lambda: pipe.step(msg))
        rails.check()
        fin = {k: v.cpu() for k, v in pipe.final.items()}
        ok = True
        for d in np.linspace(0, M - 1, a.check_nodes).astype(int):
            o = oracle.schedule_node(msg_np[0, d], C)
            ok &= bool(np.array_equal(pipe.sched.send_load[0, d].cpu().numpy(), o["send_load"]))
            ok &= bool(np.array_equal(pipe.sched.rem_off[0, d].cpu().numpy(), o["rem_off"]))
        rows.append({"C": C, "step_ms": ms, "nodes_per_s": M / (ms / 1e3),
                     "remainders_per_node": float(pipe.sched.n_rem.float().mean()),
                     "full_chunks_per_node": float(pipe.sched.n_full.double().mean()),
                     "T_lpt_over_Tstar": float(fin["T"][0] / fin["T_star"][0]),
                     "T_ecmp_over_Tstar": float(fin["T_e"][0] / fin["T_star"][0]),
                     "busbw_lpt_over_ecmp": float(fin["busbw"][0] / fin["busbw_e"][0]),
                     "oracle_spot_check": ok})
        print(json.dumps(rows[-1]), flush=True)
    if a.out:
        json.dump({"config": "c5", "M": M, "N": N, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
