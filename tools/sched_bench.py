#!/usr/bin/env python
"""Schedule-side timing (a1 histogram, a2-a5 fused schedule + eval) on the BASELINE
configs, CUDA events on the launching stream, L2 flushed before every timed
iteration, clocks sampled while timing.  Writes one JSON object to stdout.

  c3      64 nodes x 8 rails, one unit: histogram, fused kernel, both (eager)
  c2      1000 iterations x 16 nodes (receiver-skew Zipf bytes): fused kernel
  c4      one iteration = 32 layers x 128 nodes: histogram (HBM roofline), fused
  c5_<C>  256 nodes x 8 rails, one unit per chunk size: fused kernel
Not a bench line (bench.py is); used for DESIGN.md and profiles/.
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
from bench import ClockSampler  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402
from paper_2510_19262_b200.pipeline import MatrixPipeline, RoutingPipeline  # noqa: E402

DEV = "cuda:0"
_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    _flush.fill_(1)


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1000.0)
    rails.check()
    ts.sort()
    return {"median_us": round(ts[len(ts) // 2], 2), "best_us": round(ts[0], 2)}


def loop_us(fn, iters=50, warm=5):
    """Mean per call over `iters` back-to-back calls between one event pair (hot L2;
    resolves differences far below the single-call event granularity)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    rails.check()
    return round(a.elapsed_time(b) * 1000.0 / iters, 2)


def routing_pipe(name, U=1):
    cfg = gen.CONFIGS[name]
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    seed = gen.config_seed(int(name[1]))
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u, device=DEV) for u in range(U)])
    lut = gen.inst_lut(M, N, E).to(DEV)
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, 0, M, lut.numel(), DEV, out_cap=16)
    return pipe, topk, lut


def bench_routing(res, name, U):
    pipe, topk, lut = routing_pipe(name, U)
    hist = lambda: rails.histogram(pipe.tp, pipe.sh, topk, lut, pipe.RB,  # noqa: E731
                                   out=(pipe.counts, pipe.msg, pipe.rank))
    fused = lambda: rails.schedule_eval(pipe.tp, pipe.sh, pipe.msg, pipe.sched, pipe.ev,  # noqa
                                        pipe.ws, final=pipe.final, rail_base=pipe.rail_base,
                                        rail_total=pipe.total)
    th = timeit(hist)
    hb = rails.bind_histogram(pipe.tp, pipe.sh, topk, lut, pipe.RB,
                              (pipe.counts, pipe.msg, pipe.rank))
    th["loop_hot_us"] = loop_us(lambda: hb(None))
    tf = timeit(fused)
    fb = rails.bind_schedule_eval(pipe.tp, pipe.sh, pipe.msg, pipe.sched, pipe.ev, pipe.ws,
                                  final=pipe.final, rail_base=pipe.rail_base,
                                  rail_total=pipe.total)
    tf["loop_hot_us"] = loop_us(lambda: fb(None))
    split = lambda: (rails.lpt_schedule(pipe.tp, pipe.sh, pipe.msg, out=pipe.sched,  # noqa: E731
                                        workspace=pipe.ws),
                     rails.eval(pipe.tp, pipe.sh, pipe.msg, pipe.sched, out=pipe.ev))
    tsp = timeit(split)
    tsch = timeit(lambda: rails.lpt_schedule(pipe.tp, pipe.sh, pipe.msg, out=pipe.sched,
                                             workspace=pipe.ws))
    tb = timeit(lambda: pipe.schedule_part(topk, lut))
    tb["loop_hot_us"] = loop_us(lambda: pipe.schedule_part(topk, lut))
    ne = topk.numel()
    G = pipe.M * pipe.N
    nseg = U * pipe.M * pipe.N
    hbytes = ne * 4 * 2 + nseg * G * (4 + 8)  # ids in, ranks out, counts + bytes out
    out = {"units": U, "nodes": U * pipe.M, "histogram": th, "fused_sched_eval": tf,
           "schedule_then_eval": tsp, "schedule_only_kernel": tsch,
           "schedule_part": tb, "hist_algorithmic_bytes": hbytes,
           "hist_gbs": round(hbytes / (th["median_us"] * 1e-6) / 1e9, 1),
           "nodes_per_s_schedule_part": round(U * pipe.M / (tb["median_us"] * 1e-6))}
    res[name] = out


def bench_matrix(res, name, C=None, U=None):
    cfg = dict(gen.CONFIGS[name])
    if C is not None:
        cfg["C"] = C
    U = U if U is not None else cfg.get("U", 1)
    M, N = cfg["M"], cfg["N"]
    msg = torch.from_numpy(gen.d1_units(cfg, gen.config_seed(int(name[1])), 0, U)).to(DEV)
    pipe = MatrixPipeline(M, N, cfg["C"], U, 0, M, DEV)
    t = timeit(lambda: pipe.step(msg))
    t["loop_hot_us"] = loop_us(lambda: pipe.step(msg), iters=10, warm=2)
    tsp = timeit(lambda: (rails.lpt_schedule(pipe.tp, pipe.sh, msg, out=pipe.sched,
                                             workspace=pipe.ws),
                          rails.eval(pipe.tp, pipe.sh, msg, pipe.sched, out=pipe.ev)))
    key = name if C is None else f"{name}_C{C}"
    res[key] = {"units": U, "nodes": U * M, "fused_sched_eval": t, "schedule_then_eval": tsp,
                "nodes_per_s": round(U * M / (t["median_us"] * 1e-6))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c3,c2,c4,c5")
    ap.add_argument("--lib", default=None, help="time another build (tools/ab_build.py)")
    args = ap.parse_args()
    if args.lib:
        rails.LIB_PATH = os.path.abspath(args.lib)
    want = args.only.split(",")
    res = {"gpu": torch.cuda.get_device_name(0), "lib": rails.LIB_PATH}
    jobs = []
    if "c3" in want:
        jobs.append(("c3", lambda: bench_routing(res, "c3", 1)))
    if "c2" in want:
        jobs.append(("c2", lambda: bench_matrix(res, "c2")))
    if "c4" in want:
        jobs.append(("c4", lambda: bench_routing(res, "c4", 32)))
    if "c5" in want:
        for C in (4096, 32768, 1 << 20, 4 << 20):
            jobs.append((f"c5_C{C}", lambda C=C: bench_matrix(res, "c5", C=C, U=1)))
    with ClockSampler(0) as clk:
        for name, job in jobs:
            try:
                job()
            except Exception as e:  # noqa: BLE001 -- reported in the JSON
                res[name] = {"error": repr(e)}
            torch.cuda.empty_cache()
    res["clocks"] = clk.summary()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
