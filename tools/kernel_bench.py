#!/usr/bin/env python
"""Per-kernel timing on representative batched launches (CUDA events, warm-up,
inputs larger than L2 or L2 flushed between iterations).  Writes one JSON object.

  pack      C3 launch (64 nodes), impl 1 (LDG/STG registers) vs 2 (TMA bulk)
  histogram C4 iteration (32 layers x 128 nodes, 1 GiB routing) -- HBM roofline
  schedule  C2 (1000 iterations x 16 nodes = 16000 chains), C3, C5 sweep points
  eval      same launches as schedule
Not a bench line: bench.py is.  Used to fill DESIGN.md section 7 and profiles/.
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
from paper_2510_19262_b200.pipeline import MatrixPipeline, RoutingPipeline  # noqa: E402

DEV = "cuda:0"
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    _flush.random_(0, 255)


def timeit(fn, iters=10, warm=3, flush=True):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush:
            flush_l2()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return {"median_ms": ts[len(ts) // 2], "best_ms": ts[0]}


def bench_pack(res):
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
    total = int(pipe.total.item())
    algo = M * N * T * RB + total
    ref = None
    variants = os.environ.get("KB_PACK_VARIANTS", "1,2,1cs,1v8,1v4,3s436,3s328,3s644,3s426,3s218")
    for impl in variants.split(","):
        os.environ["RAILS_PACK_IMPL"] = impl[0]
        os.environ.pop("RAILS_PACK_ST", None)
        os.environ.pop("RAILS_PACK_VPL", None)
        os.environ.pop("RAILS_PACK_TMA", None)
        os.environ.pop("RAILS_PACK_CTAS", None)
        os.environ.pop("RAILS_PACK_RPW", None)
        if impl.startswith("1r"):  # 1rN: N rows per warp
            os.environ["RAILS_PACK_RPW"] = impl[2:]
        if impl.startswith("1g"):  # 1gN: N CTAs per SM
            os.environ["RAILS_PACK_CTAS"] = impl[2:]
        if impl.startswith("1cs"):  # 1cs: .cs stores; 1cs2: .cs loads; 1cs3: both
            os.environ["RAILS_PACK_ST"] = impl[3:] or "1"
        if impl.startswith("1v"):
            os.environ["RAILS_PACK_VPL"] = impl[2:]
        if impl.startswith("3s"):
            os.environ["RAILS_PACK_TMA"] = impl[2:]
        pipe.out.zero_()
        t = timeit(lambda: rails.pack(pipe.tp, pipe.sh, T, k, x, topk, lut, pipe.rank, pipe.msg, RB,
                                      pipe.sched, pipe.rail_base, pipe.out), flush=False)
        rails.check()
        h = torch.sum(pipe.out[:total].view(torch.int64) * 0 + 1).item()  # touch
        snap = pipe.out[:total:4099].clone()
        if ref is None:
            ref = snap
        same = bool(torch.equal(ref, snap))
        gbs = algo / (t["median_ms"] / 1e3) / 1e9
        res[f"pack_impl{impl}"] = dict(t, gbs=gbs, frac=gbs / PEAK, bytes=algo, same_as_impl1=same)
        del h
    os.environ.pop("RAILS_PACK_IMPL", None)
    os.environ.pop("RAILS_PACK_ST", None)
    os.environ.pop("RAILS_PACK_VPL", None)
    os.environ.pop("RAILS_PACK_TMA", None)
    # context only (NOT the roofline denominator): the same 1-read : 2-write byte
    # mix as the pack, done by a plain torch broadcast copy of every 8 KiB row into
    # two adjacent slots (second read of a row hits L2)
    xs = x.view(-1, RB // 8)
    nrow = min(xs.shape[0], pipe.out.numel() // (2 * RB))
    dst = pipe.out[:nrow * 2 * RB].view(torch.int64).view(nrow, 2, RB // 8)
    t = timeit(lambda: dst.copy_(xs[:nrow, None, :].expand(nrow, 2, RB // 8)), flush=False)
    b = nrow * RB * 3
    res["torch_dup_copy_1r2w"] = dict(t, gbs=b / (t["median_ms"] / 1e3) / 1e9, bytes=b)
    t = timeit(lambda: dst[:, 0, :].copy_(xs[:nrow]), flush=False)
    b = nrow * RB * 2
    res["torch_copy_1r1w_strided"] = dict(t, gbs=b / (t["median_ms"] / 1e3) / 1e9, bytes=b)
    # schedule-side kernels of the same C3 unit
    res["c3_schedule"] = timeit(lambda: rails.lpt_schedule(pipe.tp, pipe.sh, pipe.msg, out=pipe.sched,
                                                           workspace=pipe.ws))
    qp = torch.empty(pipe.sched.rem_rail.shape, dtype=torch.int32, device=DEV)
    res["c3_schedule_qp64"] = timeit(lambda: rails.lpt_schedule_qp(
        pipe.tp, pipe.sh, pipe.msg, 64, out=pipe.sched, rem_qp=qp, workspace=pipe.ws))
    res["c3_histogram"] = timeit(lambda: rails.histogram(pipe.tp, pipe.sh, topk, lut, RB,
                                                         out=(pipe.counts, pipe.msg, pipe.rank)))
    res["c3_eval"] = timeit(lambda: rails.eval(pipe.tp, pipe.sh, pipe.msg, pipe.sched, out=pipe.ev))
    del pipe, x
    torch.cuda.empty_cache()


def bench_hist_c3(res):
    """The C3 launch of a1 (64 nodes x 8 source GPUs = 512 segments of 8192 ids)."""
    cfg = gen.CONFIGS["c3"]
    M, N, T, k, E = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"]
    topk = gen.routing(M, N, T, k, E, gen.config_seed(3), 0, device=DEV)[None].contiguous()
    lut = gen.inst_lut(M, N, E).to(DEV)
    tp, sh = rails.topo(M, N, cfg["C"]), rails.shard(1, 0, M)
    G = M * N
    out = (torch.empty((1, M, N, G), dtype=torch.int32, device=DEV),
           torch.empty((1, M, N, G), dtype=torch.int64, device=DEV),
           torch.empty((1, M, N, T, k), dtype=torch.int32, device=DEV))
    t = timeit(lambda: rails.histogram(tp, sh, topk, lut, cfg["H"] * 2, out=out), iters=20)
    algo = M * N * (T * k * 4 * 2 + G * 12)
    gbs = algo / (t["median_ms"] / 1e3) / 1e9
    res["hist_c3"] = dict(t, gbs=gbs, frac=gbs / PEAK, bytes=algo)


def bench_hist_c4(res):
    cfg = gen.CONFIGS["c4"]
    M, N, T, k, E = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"]
    U = cfg["U"]
    seed = gen.config_seed(4)
    topk = torch.empty((U, M, N, T, k), dtype=torch.int32, device=DEV)
    for u in range(U):
        topk[u] = gen.routing(M, N, T, k, E, seed, u, device=DEV)
    lut = gen.inst_lut(M, N, E).to(DEV)
    tp, sh = rails.topo(M, N, cfg["C"]), rails.shard(U, 0, M)
    G = M * N
    out = (torch.empty((U, M, N, G), dtype=torch.int32, device=DEV),
           torch.empty((U, M, N, G), dtype=torch.int64, device=DEV),
           torch.empty((U, M, N, T, k), dtype=torch.int32, device=DEV))
    t = timeit(lambda: rails.histogram(tp, sh, topk, lut, cfg["H"] * 2, out=out))
    algo = U * M * N * (T * k * 4 * 2 + G * 12)
    gbs = algo / (t["median_ms"] / 1e3) / 1e9
    res["hist_c4_iteration"] = dict(t, gbs=gbs, frac=gbs / PEAK, bytes=algo)
    # schedule + eval over the whole C4 iteration (4096 chains of ~7K remainders)
    msg = out[1]
    pipe = MatrixPipeline(M, N, cfg["C"], U, 0, M, DEV)
    res["c4_schedule"] = timeit(lambda: rails.lpt_schedule(pipe.tp, pipe.sh, msg, out=pipe.sched,
                                                           workspace=pipe.ws))
    qp = torch.empty(pipe.sched.rem_rail.shape, dtype=torch.int32, device=DEV)
    res["c4_schedule_qp64"] = timeit(lambda: rails.lpt_schedule_qp(
        pipe.tp, pipe.sh, msg, 64, out=pipe.sched, rem_qp=qp, workspace=pipe.ws))
    res["c4_eval"] = timeit(lambda: rails.eval(pipe.tp, pipe.sh, msg, pipe.sched, out=pipe.ev))
    del topk, out, msg, pipe
    torch.cuda.empty_cache()


def bench_matrix(res, name, C=None, U=None):
    cfg = gen.CONFIGS[name]
    M, N = cfg["M"], cfg["N"]
    C = cfg["C"] if C is None else C
    U = cfg["U"] if U is None else U
    msg = torch.from_numpy(gen.d1_units(cfg, gen.config_seed(int(name[1])), 0, U)).to(DEV)
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    ts = timeit(lambda: rails.lpt_schedule(pipe.tp, pipe.sh, msg, out=pipe.sched, workspace=pipe.ws))
    te = timeit(lambda: rails.eval(pipe.tp, pipe.sh, msg, pipe.sched, out=pipe.ev))
    tf = timeit(lambda: pipe.step(msg))
    fin = {k: v.cpu() for k, v in pipe.final.items()}
    res[f"{name}_C{C}"] = {"schedule": ts, "eval": te, "step": tf,
                           "nodes_per_s": U * M / (tf["median_ms"] / 1e3),
                           "n_rem_mean": float(pipe.sched.n_rem.float().mean()),
                           "T_over_Tstar": float((fin["T"] / fin["T_star"]).max()),
                           "Te_over_Tstar": float((fin["T_e"] / fin["T_star"]).max())}


def bench_bw(res):
    """Context for the pack's roofline: torch's own streaming kernels on 8 GiB
    buffers -- write-only (fill), read-only (sum) and 1:1 copy -- so the 1 read :
    2 write mix of the pack can be set against pure read / write bandwidth."""
    n = 8 << 30
    a = torch.empty(n // 4, dtype=torch.float32, device=DEV)
    b = torch.empty(n // 4, dtype=torch.float32, device=DEV)
    a.fill_(1.0)
    t = timeit(lambda: a.fill_(2.0), iters=5)
    res["bw_write_fill"] = dict(t, gbs=n / (t["median_ms"] / 1e3) / 1e9)
    t = timeit(lambda: a.sum(), iters=5)
    res["bw_read_sum"] = dict(t, gbs=n / (t["median_ms"] / 1e3) / 1e9)
    t = timeit(lambda: b.copy_(a), iters=5)
    res["bw_copy"] = dict(t, gbs=2 * n / (t["median_ms"] / 1e3) / 1e9)
    del a, b
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="pack,hist,c2,c5")
    a = ap.parse_args()
    res = {"device": torch.cuda.get_device_name(0), "peak_gbs": PEAK}
    only = a.only.split(",")
    if "bw" in only:
        bench_bw(res)
    if "pack" in only:
        bench_pack(res)
    if "hist3" in only:
        bench_hist_c3(res)
    if "hist" in only:
        bench_hist_c4(res)
    if "c2" in only:
        bench_matrix(res, "c2")
    if "c5" in only:
        for C in (4 << 10, 64 << 10, 1 << 20, 4 << 20):
            bench_matrix(res, "c5", C=C)
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
