#!/usr/bin/env python
"""NEXT f3: LPT spraying vs ECMP hashing vs the Theorem-3 optimum on the paper's
workload families (Table 1), in the static rail-load model (R#7-R#10).

For each family the CUDA path schedules and evaluates U seeded units; reported per
family: T_LPT/T*, T_ECMP/T*, T_uniform/T* (T* = the Theorem-3 optimum, Thm 2 + 3;
"uniform" = the discrete P* = 1/N split the kernels evaluate, R#41), normalized
busbw LPT/ECMP and LPT/uniform, and the per-node normalized MSE of the sending loads
 for LPT, ECMP and uniform.  Clocks are sampled while the kernels run.  The topology follows the paper's testbed
scale: 128 domains x 8 GPUs; chunks 32 KiB.  Directional only: the
paper's numbers come from an emulated network (Mininet + Soft-RoCE).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2510_19262_b200.pipeline import MatrixPipeline  # noqa: E402

FAMILIES = [
    ("uniform", dict(skew="uniform")),
    ("sparse-0.6", dict(skew="sparse", sparsity=0.6, K=2)),
    ("sparse-0.4", dict(skew="sparse", sparsity=0.4, K=2)),
    ("sparse-0.2", dict(skew="sparse", sparsity=0.2, K=2)),
    ("sparse-0", dict(skew="sparse", sparsity=0.0, K=2)),
    ("sender-skewed", dict(skew="sender", zipf_s=1.2)),
    ("receiver-skewed", dict(skew="receiver", zipf_s=1.2)),
]


def nmse_rows(S: np.ndarray) -> np.ndarray:
    """nMSE of each node's rail loads (R#12), report-side arithmetic only."""
    S = S.astype(np.float64)
    tot = S.sum(axis=-1, keepdims=True)
    frac = np.divide(S, tot, out=np.zeros_like(S), where=tot > 0)
    return ((frac - 1.0 / S.shape[-1]) ** 2).mean(axis=-1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=128)
    ap.add_argument("--N", type=int, default=8)
    ap.add_argument("--C", type=int, default=32 << 10)
    ap.add_argument("--V", type=int, default=64 << 20)
    ap.add_argument("--units", type=int, default=4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = "cuda:0"
    rows = []
    with ClockSampler(0) as clk:
        for name, extra in FAMILIES:
            cfg = dict(M=a.M, N=a.N, V=a.V, zipf_s=1.2)
            cfg.update(extra)
            msg = gen.d1_units(cfg, gen.config_seed(9), 0, a.units)
            pipe = MatrixPipeline(a.M, a.N, a.C, a.units, 0, a.M, dev)
            m = torch.from_numpy(msg).to(dev)
            pipe.step(m)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe.step(m)
            e1.record()
            torch.cuda.synchronize()
            f = {k: v.cpu().numpy() for k, v in pipe.final.items()}
            S, Se, Su = (pipe.ev.S.cpu().numpy(), pipe.ev.S_e.cpu().numpy(),
                         pipe.ev.S_u.cpu().numpy())
            rows.append({
                "family": name,
                "T_lpt_over_Tstar": float(np.mean(f["T"] / f["T_star"])),
                "T_ecmp_over_Tstar": float(np.mean(f["T_e"] / f["T_star"])),
                "T_uniform_over_Tstar": float(np.mean(f["T_u"] / f["T_star"])),
                "busbw_lpt_over_ecmp": float(np.mean(f["busbw"] / f["busbw_e"])),
                "busbw_lpt_over_uniform": float(np.mean(f["busbw"] / f["busbw_u"])),
                "nmse_lpt_mean": float(nmse_rows(S).mean()),
                "nmse_ecmp_mean": float(nmse_rows(Se).mean()),
                "nmse_uniform_mean": float(nmse_rows(Su).mean()),
                "gpu_nmse_lpt_mean": float(pipe.ev.nmse.mean().item()),
                "schedule_eval_ms": e0.elapsed_time(e1),
            })
            print(json.dumps(rows[-1]), flush=True)
    res = {"topology": f"{a.M} domains x {a.N} rails", "chunk_bytes": a.C,
           "bytes_per_source_gpu": a.V, "units": a.units, "rows": rows,
           "clocks": clk.summary(), "gpu": torch.cuda.get_device_name(0)}
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
