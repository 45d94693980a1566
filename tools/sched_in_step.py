#!/usr/bin/env python
"""Where the bench's schedule_only time goes on C3: the schedule part timed (CUDA
events on the launching stream) in three settings --
  after_pack   the bench's step order (previous step's pack, then the schedule part)
  after_flush  after a 256 MiB L2-dirtying fill (tools/sched_bench.py's setting)
  hot          back to back
-- each split into the histogram and the fused schedule+eval kernel (separate
calls) and the single bound call the bench makes.  Prints JSON.  Not a bench line."""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402
from paper_2510_19262_b200.pipeline import RoutingPipeline  # noqa: E402

DEV = "cuda:0"


def main():
    if len(sys.argv) > 1:  # another build (tools/ab_build.py)
        rails.LIB_PATH = os.path.abspath(sys.argv[1])
    cfg = gen.CONFIGS["c3"]
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    seed = gen.config_seed(3)
    topk = gen.routing(M, N, T, k, E, seed, 0, device=DEV)[None]
    lut = gen.inst_lut(M, N, E).to(DEV)
    x = torch.empty((1, M, N, T, RB // 8), dtype=torch.int64, device=DEV)
    gen.payload(M, N, T, RB, seed, 0, 0, M, device=DEV, out=x[0])
    pipe = RoutingPipeline(M, N, T, k, RB, C, 1, 0, M, lut.numel(), DEV)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def split_call():
        rails.histogram(pipe.tp, pipe.sh, topk, lut, pipe.RB,
                        out=(pipe.counts, pipe.msg, pipe.rank))

    def fused_call():
        rails.schedule_eval(pipe.tp, pipe.sh, pipe.msg, pipe.sched, pipe.ev, pipe.ws,
                            final=pipe.final, rail_base=pipe.rail_base, rail_total=pipe.total)

    # a second, independent pipeline: running its schedule part after the pack puts
    # the kernels' code back in L2 without touching the measured pipeline's data
    pipe2 = RoutingPipeline(M, N, T, k, RB, C, 1, 0, M, lut.numel(), DEV)
    topk2 = topk.clone()

    def before(mode):
        if mode == "after_pack":
            pipe.pack_part(topk, lut, x)
        elif mode == "after_pack_code_warm":
            pipe.pack_part(topk, lut, x)
            pipe2.schedule_part(topk2, lut)
        elif mode == "after_flush":
            flush.fill_(1)

    pipe.schedule_part(topk, lut)  # the pack below reads a valid schedule from here on
    pipe2.schedule_part(topk2, lut)
    torch.cuda.synchronize()
    rails.check()
    res = {}
    with ClockSampler(0) as clk:
        for mode in ("after_pack", "after_pack_code_warm", "after_flush", "hot"):
            for _ in range(3):
                before(mode)
                pipe.schedule_part(topk, lut)
            torch.cuda.synchronize()
            one, hist, node, pk = [], [], [], []
            for _ in range(40):
                p0, p1 = ev(), ev()
                p0.record()
                before(mode)
                p1.record()
                a, b = ev(), ev()
                a.record()
                pipe.schedule_part(topk, lut)
                b.record()
                before(mode)
                c, d, e = ev(), ev(), ev()
                c.record()
                split_call()
                d.record()
                fused_call()
                e.record()
                torch.cuda.synchronize()
                one.append(a.elapsed_time(b) * 1e3)
                pk.append(p0.elapsed_time(p1) * 1e3)
                hist.append(c.elapsed_time(d) * 1e3)
                node.append(d.elapsed_time(e) * 1e3)
            rails.check()
            med = lambda v: round(sorted(v)[len(v) // 2], 2)  # noqa: E731
            res[mode] = {"schedule_part_us": med(one), "histogram_us": med(hist),
                         "schedule_eval_us": med(node), "before_us": med(pk)}
    res["clocks"] = clk.summary()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
