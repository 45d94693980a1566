#!/usr/bin/env python
"""NEXT f1 benchmark: the combine round on one GPU (all nodes resident).

Dispatch (histogram, schedule, pack) then combine: traffic transpose, receive
offsets, combine LPT schedule, combine pack (expert outputs -> rail buffers) and
unpack with the top-k weighted fp32 combine.  Reports per-kernel CUDA-event times
and GB/s against their algorithmic bytes:
  combine pack: read the railed expert-output rows once + write them once;
  unpack:       read k rows (RB each) per token + write the fp32 output (2*RB).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402
from paper_2510_19262_b200.pipeline import RoutingPipeline  # noqa: E402

DEV = "cuda:0"


def timed(fn, iters=5, warm=2):
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
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=32)
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = gen.CONFIGS["c3"]
    M, N, T, k, E, C = a.M, cfg["N"], a.T, cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    seed = gen.config_seed(3)
    topk = gen.routing(M, N, T, k, E, seed, 0, device=DEV)[None].contiguous()
    lut = gen.inst_lut(M, N, E).to(DEV)
    x = gen.payload(M, N, T, RB, seed, 0, 0, M, device=DEV)[None].contiguous()
    disp = RoutingPipeline(M, N, T, k, RB, C, 1, 0, M, lut.numel(), DEV)
    disp.step(topk, lut, x)
    del x
    tp, sh = disp.tp, disp.sh
    msg_t = rails.transpose_traffic(tp, disp.msg)
    in_off, rows_in = rails.recv_offsets(tp, disp.counts)
    sched_c = rails.lpt_schedule(tp, sh, msg_t)
    rb_c, tot_c = rails.rail_offsets(tp, sh, sched_c.send_load)
    torch.cuda.synchronize()
    Rcap = int(rows_in.max().item())
    y = gen.expert_outputs((1, M, N, Rcap, RB // 2), 23, 0, device=DEV)
    comb = torch.empty(int(tot_c.item()) + 16, dtype=torch.uint8, device=DEV)
    w = gen.gate_weights((1, M, N, T, k), 29, 0, device=DEV)
    out = torch.empty((1, M, N, T, RB // 2), dtype=torch.float32, device=DEV)
    res = {"M": M, "N": N, "T": T, "k": k, "row_bytes": RB, "chunk_bytes": C}
    res["transpose_ms"] = timed(lambda: rails.transpose_traffic(tp, disp.msg, out=msg_t))
    res["recv_offsets_ms"] = timed(lambda: rails.recv_offsets(tp, disp.counts, in_off, rows_in))
    res["combine_schedule_ms"] = timed(lambda: rails.lpt_schedule(tp, sh, msg_t, out=sched_c))
    t = timed(lambda: rails.pack_combine(tp, sh, RB, y, in_off, rows_in, msg_t, sched_c, rb_c, comb))
    moved = 2 * int(tot_c.item())
    res["combine_pack_ms"] = t
    res["combine_pack_gbs"] = moved / (t / 1e3) / 1e9
    t = timed(lambda: rails.unpack_combine(tp, sh, T, k, topk, lut, disp.rank, w, y, in_off,
                                           msg_t, sched_c, rb_c, comb, RB, out=out))
    moved = M * N * T * (k * RB + 2 * RB)
    res["unpack_ms"] = t
    res["unpack_gbs"] = moved / (t / 1e3) / 1e9
    rails.check()
    print(json.dumps(res))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
