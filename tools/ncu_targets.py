#!/usr/bin/env python
"""One launch of each kernel worth an ncu --set full capture, in one process:
the C3 path (histogram, chunk/sort, LPT, expand, eval, finalize, pack), a C4
iteration's batched histogram / schedule / eval, and one fluid-simulation batch.
Usage (profiling only; times printed under ncu are not measurements):
  ncu --set full -k regex:"k_" -o out python tools/ncu_targets.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402
from paper_2510_19262_b200.pipeline import MatrixPipeline, RoutingPipeline  # noqa: E402

DEV = "cuda:0"


def c3():
    cfg = gen.CONFIGS["c3"]
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    seed = gen.config_seed(3)
    topk = gen.routing(M, N, T, k, E, seed, 0, device=DEV)[None].contiguous()
    lut = gen.inst_lut(M, N, E).to(DEV)
    x = gen.payload(M, N, T, RB, seed, 0, 0, M, device=DEV)[None].contiguous()
    pipe = RoutingPipeline(M, N, T, k, RB, C, 1, 0, M, lut.numel(), DEV)
    pipe.step(topk, lut, x)
    torch.cuda.synchronize()


def c4():
    cfg = gen.CONFIGS["c4"]
    M, N, T, k, E, C, U = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"], cfg["U"]
    RB = cfg["H"] * 2
    seed = gen.config_seed(4)
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u, device=DEV) for u in range(U)])
    lut = gen.inst_lut(M, N, E).to(DEV)
    tp, sh = rails.topo(M, N, C), rails.shard(U, 0, M)
    _, msg, _ = rails.histogram(tp, sh, topk, lut, RB)
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(msg)
    torch.cuda.synchronize()


def flowsim():
    M, N, R2 = 8, 8, 5.0e10
    msg = gen.d1_receiver_skew(M, N, 4 << 20, 1.2, 7, 0)
    tp = rails.topo(M, N, 32768, R2=R2)
    fb = rails.fabric(M, N, R2)
    pol = torch.arange(6, dtype=torch.int32, device=DEV)
    rails.flowsim(tp, fb, pol, torch.from_numpy(np.stack([msg] * 6)).to(DEV))
    torch.cuda.synchronize()


if __name__ == "__main__":
    c3()
    c4()
    flowsim()
    rails.check()
    print("ok")
