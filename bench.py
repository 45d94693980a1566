#!/usr/bin/env python
"""Benchmark of the RailS hot path on B200 (one JSON line on rank 0).

Workload (default, --workload c3): BASELINE.json config 3, Mixtral 8x7B expert-
parallel routing shape -- 64 nodes x 8 rails, T = 4096 tokens per GPU, top-2 of 8
experts, H = 4096 bf16 rows (RB = 8 KiB), 32 KiB chunks.  It is the configuration
that exercises every row of SURVEY section 8(a) (routing -> histogram -> chunk ->
sort -> LPT -> eval -> reduction -> pack) and fits one GPU; configs[1] (C2) is a
byte matrix with no routing or payload, so it cannot run a1/a7 (available as
--workload c2, schedule+eval only).

A step = one pass of the whole path over one batch: every rank holds M/P source
nodes of each of U = P units (weak scaling: 64 (unit, node) schedules + packs per
GPU per step); a6 all-reduces the partial receive loads (NCCL SUM) and maxima (MAX).
value = (unit, node) pairs completed by all ranks / max-over-ranks device time.

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cuda.synchronize, CUDA events on the launching stream; the payload (16 GiB) and rail
buffers (31.5 GiB) per rank exceed L2 (126 MB), so every step streams from HBM.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402

METRIC = ("LPT-scheduled nodes/sec and pack GB/s (vs HBM peak) at 1/2/4/8 B200; "
          "makespan/OPT")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c2", "c1", "c4"])
    ap.add_argument("--reduce", default="peer", choices=["peer", "nccl"],
                    help="a6 at N > 1: fused finalize over NVLink peer memory, or NCCL")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-ring", action="store_true",
                    help="force the pinned-ring staging of the payload (testing)")
    ap.add_argument("--nd", type=int, default=None,
                    help="nodes per rank override (profiling runs only; not a bench line)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        time.sleep(0.2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- oracle (CPU) arm
_INPUT_CACHE = {}


def _oracle_inputs(cfg_name: str, i: int):
    """Inputs of the i-th sampled node of unit 0 (generation is not timed; the first
    16 are kept for the all-cores run, which must not generate after fork)."""
    key = (cfg_name, i)
    if key in _INPUT_CACHE:
        return _INPUT_CACHE[key]
    cfg = gen.CONFIGS[cfg_name]
    M, N = cfg["M"], cfg["N"]
    seed = gen.config_seed(int(cfg_name[1]))
    if cfg["kind"] == "routing":
        T, k, E, RB = cfg["T"], cfg["k"], cfg["E"], cfg["H"] * 2
        d = (i * 37) % M
        inp = {"d": d, "lut": gen.inst_lut(M, N, E).numpy(),
               "topk": gen.routing(M, N, T, k, E, seed, 0, d, 1)[0].numpy(),
               "x": gen.payload(M, N, T, RB, seed, 0, d, 1)[0].numpy().view(np.uint8)}
    else:
        inp = {"d": i % M, "msg": _d1_unit0(cfg_name)}
    if i < 16:
        _INPUT_CACHE[key] = inp
    return inp


_D1_CACHE = {}


def _d1_unit0(cfg_name: str):
    if cfg_name not in _D1_CACHE:
        cfg = gen.CONFIGS[cfg_name]
        _D1_CACHE[cfg_name] = gen.d1_units(cfg, gen.config_seed(int(cfg_name[1])), 0, 1)[0]
    return _D1_CACHE[cfg_name]


def _oracle_node(cfg_name: str, inp) -> None:
    """One (unit, node) through the CPU oracle as it stands: routing configs run the
    full path (histogram, chunk, sort, LPT, eval, pack), matrix configs schedule + eval."""
    import oracle

    cfg = gen.CONFIGS[cfg_name]
    M, N, C = cfg["M"], cfg["N"], cfg["C"]
    d = inp["d"]
    if cfg["kind"] == "routing":
        T, k, RB = cfg["T"], cfg["k"], cfg["H"] * 2
        topk, lut = inp["topk"], inp["lut"]
        c, m, r = oracle.histogram_node(M, N, d, T, k, topk, lut, RB)
        s = oracle.schedule_node(m, C)
        ch = s["chunks"]
        oracle.eval_unit(M, N, 5.0e10, gen.ECMP_SEED, np.pad(m[None], ((d, M - d - 1), (0, 0), (0, 0))),
                         np.full(len(ch["size"]), d, np.int32), ch["h"], ch["size"], s["rail"])
        L = s["send_load"]
        base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
        oracle.pack_node(M, N, d, T, k, RB, C, inp["x"], topk, lut, m, s, base, int(L.sum()))
    else:
        msg = inp["msg"]
        s = oracle.schedule_node(msg[d], C)
        ch = s["chunks"]
        oracle.eval_unit(M, N, 5.0e10, gen.ECMP_SEED, msg,
                         np.full(len(ch["size"]), d, np.int32), ch["h"], ch["size"], s["rail"])


def oracle_sample(cfg_name: str, budget_s: float = 12.0, max_nodes: int = 24):
    """Time the CPU oracle, as it stands, on a bounded sample of the same workload
    (sampled nodes of unit 0), single-threaded: SURVEY 8(d) d.5 (i)."""
    cfg = gen.CONFIGS[cfg_name]
    routing = cfg["kind"] == "routing"
    cap = max_nodes if routing else max_nodes * 1000
    done, t_used = 0, 0.0
    while done < cap and t_used < budget_s:
        inp = _oracle_inputs(cfg_name, done)
        t0 = time.perf_counter()
        _oracle_node(cfg_name, inp)
        t_used += time.perf_counter() - t0
        done += 1
    what = "full path incl. pack" if routing else "schedule + eval"
    sample = f"{done} sampled nodes of unit 0 ({what}), single-threaded C oracle"
    return {"value": done / t_used, "unit": "nodes/s", "cores": 1, "kind": "oracle",
            "sample": sample, "seconds": round(t_used, 3)}


def _oracle_worker(cfg_name, inps, barrier, q):
    try:
        barrier.wait(timeout=300)
        t0 = time.perf_counter()  # CLOCK_MONOTONIC: comparable across processes
        for inp in inps:
            _oracle_node(cfg_name, inp)
        q.put((t0, time.perf_counter()))
    except BaseException as e:  # noqa: BLE001 -- reported by the parent
        try:
            barrier.abort()
        except Exception:
            pass
        q.put(repr(e))


def oracle_sample_all_cores(cfg_name: str, max_procs: int = 16):
    """the same single-threaded oracle on every host core at once
    (one process per core, up to max_procs, each owning its own sampled nodes; the
    oracle's comparator context is process-global, so processes, not threads).  Wall
    time = first start to last end after a common barrier; input generation excluded."""
    import multiprocessing as mp

    cfg = gen.CONFIGS[cfg_name]
    import psutil

    routing = cfg["kind"] == "routing"
    # a routing node holds ~0.8 GiB (payload + packed rail buffers) while it runs
    fit = int(psutil.virtual_memory().available // (3 << 29)) if routing else max_procs
    P = max(1, min(os.cpu_count() or 1, max_procs, fit))
    per = 3 if routing else 2000
    # every input is generated here, before the fork: the generator uses torch CPU ops,
    # which deadlock in a forked child; the children run numpy + the C oracle only
    inps = [[_oracle_inputs(cfg_name, (i * per + j) % 16) for j in range(per)] for i in range(P)]
    ctx = mp.get_context("fork")
    barrier, q = ctx.Barrier(P), ctx.Queue()
    ps = [ctx.Process(target=_oracle_worker, args=(cfg_name, inps[i], barrier, q))
          for i in range(P)]
    for p in ps:
        p.start()
    import queue

    res = []
    try:
        for _ in ps:
            res.append(q.get(timeout=300))
    except queue.Empty:
        res.append("timeout: an oracle process did not report within 300 s")
    for p in ps:
        p.join(timeout=5)
        if p.is_alive():
            p.kill()
    bad = [r for r in res if not isinstance(r, tuple)]
    if bad:
        return {"error": bad[0]}
    wall = max(r[1] for r in res) - min(r[0] for r in res)
    what = "full path incl. pack" if cfg["kind"] == "routing" else "schedule + eval"
    return {"value": P * per / wall, "unit": "nodes/s", "cores": P, "kind": "oracle",
            "host_cpus": os.cpu_count(),
            "sample": f"{P * per} sampled nodes of unit 0 ({what}), {per} per process, "
                      f"{P} oracle processes in parallel", "seconds": round(wall, 3)}


def arm_config(args, P, nd=None):
    """The workload description both arms print (weak scaling: U = P units, M/P
    nodes of each per rank)."""
    cfg = gen.CONFIGS[args.workload]
    M, N = cfg["M"], cfg["N"]
    U = P * (cfg.get("U", 1) if cfg["kind"] == "matrix" else 1)
    nd = M // P if nd is None else nd
    if cfg["kind"] == "routing":
        return {"workload": "c3: Mixtral 8x7B EP routing shape, 64 nodes x 8 rails, "
                "T=4096 tokens/GPU, top-2 of 8 experts, H=4096 bf16 rows (8 KiB), "
                "32 KiB chunks" if args.workload == "c3" else args.workload,
                "units": U, "nodes_per_rank": nd * U, "M": M, "N": N, "T": cfg["T"],
                "k": cfg["k"], "row_bytes": cfg["H"] * 2, "chunk_bytes": cfg["C"],
                "parallelism": f"nodes{P}", "a6": (args.reduce if P > 1 else "none"),
                "l2": "inputs larger than L2: 16 GiB payload + 31.5 GiB rail buffers "
                      "streamed per step per GPU"}
    return {"workload": args.workload, "units": U, "nodes_per_rank": nd * U, "M": M, "N": N,
            "chunk_bytes": cfg["C"], "parallelism": f"nodes{P}",
            "a6": (args.reduce if P > 1 else "none")}


def run_reference(args, rank, world):
    if rank != 0:
        return
    vals = []
    for _ in range(args.warmup):
        oracle_sample(args.workload, budget_s=2.0, max_nodes=1)
    t0 = time.perf_counter()
    info = None
    for _ in range(args.steps):
        info = oracle_sample(args.workload, budget_s=8.0, max_nodes=4)
        vals.append(info["value"])
    wall = time.perf_counter() - t0
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "nodes/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * wall / max(1, args.steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": arm_config(args, max(1, world)), "gpu_launches": 0,
            "cpu_baseline": dict(info, value=v),
            "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------- GPU arm
_JSON_OUT = None


def emit(obj):
    """The one JSON line on the original stdout (everything else goes to stderr)."""
    _JSON_OUT.write(json.dumps(obj) + "\n")
    _JSON_OUT.flush()


def main():
    global _JSON_OUT
    # NCCL and CUDA libraries may print banners on fd 1: keep stdout for the JSON line
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import MatrixPipeline, RoutingPipeline

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    cfg = gen.CONFIGS[args.workload]
    M, N = cfg["M"], cfg["N"]
    P = world
    assert M % P == 0, "M must divide over ranks"
    nd = M // P
    d0 = rank * nd
    if args.nd is not None:
        nd = min(nd, args.nd)
    # weak scaling: per GPU, M/P nodes of each of P units = M node schedules; byte-
    # matrix configs batch their iterations (C2: 1000) as units of one step
    U = P * (cfg.get("U", 1) if cfg["kind"] == "matrix" else 1)
    seed = gen.config_seed(int(args.workload[1]))
    C = cfg["C"]

    def reduce(red_sum, red_max):
        if dist is not None:
            dist.all_reduce(red_sum, op=dist.ReduceOp.SUM)
            dist.all_reduce(red_max, op=dist.ReduceOp.MAX)

    stream = torch.cuda.current_stream()
    if cfg["kind"] == "routing":
        T, k, E, RB = cfg["T"], cfg["k"], cfg["E"], cfg["H"] * 2
        topk = torch.empty((U, nd, N, T, k), dtype=torch.int32, device=dev)
        for u in range(U):
            topk[u] = gen.routing(M, N, T, k, E, seed, u, d0, nd, device=dev)
        lut = gen.inst_lut(M, N, E).to(dev)
        x = torch.empty((U, nd, N, T, RB // 8), dtype=torch.int64, device=dev)
        for u in range(U):
            gen.payload(M, N, T, RB, seed, u, d0, nd, device=dev, out=x[u])
        pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), dev)

        def step(ev_p0, ev_p1, ev_s0=None):
            if ev_s0 is not None:
                ev_s0.record(stream)
            pipe.schedule_part(topk, lut)
            pipe.finalize_part(reduce if dist is not None else None)
            rails.rail_offsets(pipe.tp, pipe.sh, pipe.sched.send_load, pipe.rail_base, pipe.total)
            ev_p0.record(stream)
            rails.pack(pipe.tp, pipe.sh, T, k, x, topk, lut, pipe.rank, pipe.msg, RB, pipe.sched,
                       pipe.rail_base, pipe.out)
            ev_p1.record(stream)
    else:
        msg = torch.from_numpy(gen.d1_units(cfg, seed, 0, U)[:, d0:d0 + nd].copy()).to(dev)
        pipe = MatrixPipeline(M, N, C, U, d0, nd, dev)

        def step(ev_p0, ev_p1, ev_s0=None):
            if ev_s0 is not None:
                ev_s0.record(stream)
            ev_p0.record(stream)
            pipe.step(msg, reduce if dist is not None else None)
            ev_p1.record(stream)

    peer = None
    if dist is not None and args.reduce == "peer":
        # a6 + finalize in one kernel over NVLink peer memory;
        # GPUs without peer access keep the NCCL all-reduce (noted in config.a6)
        from paper_2510_19262_b200.dist import PeerFinalize
        peer = PeerFinalize(pipe.tp, U, dev)
        if peer.ok():
            reduce = peer  # noqa: F811 -- the pipelines call reduce.finalize
        else:
            print(f"peer a6 unavailable ({peer.error}); using NCCL", file=sys.stderr)
            peer.close()
            peer = None
            args.reduce = "nccl"

    def evpair():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    for _ in range(max(args.warmup, 1)):
        step(*evpair())
    rails.check()

    # timed region
    # per-step events around the dominant kernel (k_pack), on its launch stream
    kev = [evpair() for _ in range(args.steps)]
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    rails.launch_count(reset=True)
    with ClockSampler(local) as clk:
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        t_all0.record(stream)
        for i in range(args.steps):
            step(*kev[i], sev[i])
        t_all1.record(stream)
        torch.cuda.synchronize()
    launches = rails.launch_count(reset=True)
    if dist is not None:
        dist.barrier()
    total_ms = t_all0.elapsed_time(t_all1)
    kern_avg_ms = sum(a.elapsed_time(b) for a, b in kev) / len(kev)
    pack_avg_ms = kern_avg_ms
    # schedule part of the step (K1-K5 + the a6 NCCL reduction + rail offsets; the
    # SURVEY d.1 "LPT-scheduled nodes/s", pack excluded)
    if cfg["kind"] == "routing":
        sched_avg_ms = sum(sev[i].elapsed_time(kev[i][0]) for i in range(args.steps)) / args.steps
    else:
        sched_avg_ms = kern_avg_ms
    rails.check()

    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    nodes = U * nd * P  # all ranks together: U units x (nd per rank) nodes
    value = nodes * args.steps / (total_ms / 1000.0)
    peak, peak_kind = measured_peaks()

    out = {"metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
           "data": "synthetic"}
    ts = torch.tensor([sched_avg_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
    out["schedule_only"] = {"value": nodes / (float(ts.item()) / 1000.0), "unit": "nodes/s",
                            "ms_per_step": float(ts.item()),
                            "what": "histogram + chunk/sort + LPT + eval + a6 reduction + "
                                    "rail offsets per step, pack excluded (SURVEY 8(d) d.1)"}
    fin = {kk: vv.cpu() for kk, vv in pipe.final.items()}
    quality = {"T_lpt_over_Tstar": float((fin["T"] / fin["T_star"]).max()),
               "T_ecmp_over_Tstar": float((fin["T_e"] / fin["T_star"]).max()),
               "busbw_lpt_over_ecmp": float((fin["busbw"] / fin["busbw_e"]).min())}
    # per-node send makespan over the mean rail load (an upper bound on makespan/OPT,
    # since OPT >= ceil(sum/N)); report-side arithmetic on the kernels' S
    S = pipe.ev.S.double()
    tot = S.sum(-1)
    mk = torch.where(tot > 0, S.amax(-1) / torch.ceil(tot / N).clamp(min=1), torch.ones_like(tot))
    quality["node_makespan_over_mean_max"] = float(mk.max())
    if cfg["kind"] == "routing":
        tokens = U * nd * N * T
        pack_bytes = tokens * RB + int(pipe.total.item())  # read each row once + write copies
        t2 = torch.tensor([pack_bytes], dtype=torch.float64, device=dev)
        pk_t = torch.tensor([pack_avg_ms], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(t2)
            dist.all_reduce(pk_t, op=dist.ReduceOp.MAX)
        pack_gbs = float(t2.item()) / (float(pk_t.item()) / 1000.0) / 1e9
        per_gpu_pack = pack_bytes / (pack_avg_ms / 1000.0) / 1e9
        out["pack_gbs"] = pack_gbs
        out["config"] = arm_config(args, P, nd)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "pack_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(args.workload)
            except Exception:
                traffic = None
        out["roofline"] = {"kernel": "k_pack", "bound": "hbm", "achieved": per_gpu_pack,
                           "peak": peak, "unit": "GB/s", "frac": per_gpu_pack / peak,
                           "peak_kind": peak_kind, "traffic": traffic,
                           "peak_note": "peak = a 1:1 HBM copy; the pack moves 1 read : 2 "
                                        "writes (writes stream faster), so frac can pass 1.0; "
                                        "plain-kernel ceiling of this mix: tools/bw_mix.py",
                           "algorithmic_bytes_per_launch": pack_bytes,
                           "avg_launch_ms": pack_avg_ms,
                           "share_of_step": pack_avg_ms / (total_ms / args.steps)}
    else:
        out["config"] = arm_config(args, P, nd)
    out["quality"] = quality
    out["clocks"] = clk.summary()
    out["gpu_launches"] = int(launches)

    # ---- the same step replayed from a CUDA graph (N = 1: the a6 peer exchange's
    # call counter lives on the host, so multi-rank steps are not captured)
    if world == 1 and cfg["kind"] == "routing" and not args.no_graph:
        from paper_2510_19262_b200.pipeline import GraphStep
        g = GraphStep(lambda: pipe.step(topk, lut, x))
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            g()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / args.steps
        out["graph"] = {"value": nodes / (gms / 1000.0), "unit": "nodes/s", "ms_per_step": gms,
                        "what": "the same step captured once into a CUDA graph and replayed"}
        del g

        def sched():
            pipe.schedule_part(topk, lut)
            pipe.finalize_part(None)
            rails.rail_offsets(pipe.tp, pipe.sh, pipe.sched.send_load, pipe.rail_base, pipe.total)
        g = GraphStep(sched)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        evs = [evpair() for _ in range(args.steps)]
        torch.cuda.synchronize()
        for e0, e1 in evs:
            flush.fill_(1)  # L2 flushed between replays (outside the events)
            e0.record(stream)
            g()
            e1.record(stream)
        torch.cuda.synchronize()
        sms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / args.steps
        out["schedule_only"]["graph"] = {
            "value": nodes / (sms / 1000.0), "ms_per_step": sms,
            "what": "the schedule part alone captured into a CUDA graph and replayed, L2 "
                    "flushed before each replay (host launch gaps removed)"}
        del g, flush
    # ---- e2e: host buffers, H2D of the step's inputs + D2H of its results, timed
    if not args.no_e2e:
        out["e2e"] = e2e(args, cfg, pipe, rails, stream, dist, world, locals())
    # ---- cpu baseline (rank 0, N = 1 only)
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = oracle_sample(args.workload)
        out["cpu_baseline"]["all_cores"] = oracle_sample_all_cores(args.workload)
    if rank == 0:
        emit(out)
    if peer is not None:
        peer.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def e2e(args, cfg, pipe, rails, stream, dist, world, env):
    """Same metric through the public API with pinned HOST inputs/outputs."""
    import psutil
    dev = env["dev"]
    steps = max(1, args.e2e_steps)
    if cfg["kind"] == "routing":
        topk, x, lut = env["topk"], env["x"], env["lut"]
        need = topk.numel() * 4 + x.numel() * 8
        local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        full_copy = (psutil.virtual_memory().available > 2.0 * need * local_ranks
                     and not args.e2e_ring)
        h_topk = torch.empty(topk.shape, dtype=topk.dtype, pin_memory=True)
        h_topk.copy_(topk)
        xs = x.view(-1, x.shape[-2], x.shape[-1])  # [U*nd*N][T][W]: one GPU's rows per slice
        if full_copy:
            h_x = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h_x.copy_(x)
        else:
            # host RAM cannot pin every rank's payload: stage the same number of bytes
            # per step from a pinned ring of 4 per-GPU slices (contents repeat)
            h_x = torch.empty((4,) + tuple(xs.shape[1:]), dtype=x.dtype, pin_memory=True)
            h_x.copy_(xs[:4])
        h_res = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in pipe.final.items()}

        def one():
            topk.copy_(h_topk, non_blocking=True)
            if full_copy:
                x.copy_(h_x, non_blocking=True)
            else:
                for i in range(xs.shape[0]):
                    xs[i].copy_(h_x[i % 4], non_blocking=True)
            pipe.step(topk, lut, x, env["reduce"] if dist is not None else None)
            for kk, vv in pipe.final.items():
                h_res[kk].copy_(vv, non_blocking=True)
        h2d = h_topk.numel() * 4 + x.numel() * 8
    else:
        msg = env["msg"]
        h_msg = torch.empty(msg.shape, dtype=msg.dtype, pin_memory=True)
        h_msg.copy_(msg)
        h_res = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in pipe.final.items()}

        def one():
            msg.copy_(h_msg, non_blocking=True)
            pipe.step(msg, env["reduce"] if dist is not None else None)
            for kk, vv in pipe.final.items():
                h_res[kk].copy_(vv, non_blocking=True)
        h2d = h_msg.numel() * 8
    d2h = sum(v.numel() * v.element_size() for v in pipe.final.values())
    # ranks may be seconds apart after pinning multi-GiB host buffers; the first call
    # ends in the peer-memory a6, whose waits must not time out
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    one()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    e1.synchronize()
    rails.check()  # device-side errors (range, capacity, peer timeout) of the e2e steps
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    nodes = env["U"] * env["nd"] * env["P"]
    out = {"value": nodes * steps / (float(ms.item()) / 1000.0), "unit": "nodes/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps}
    if cfg["kind"] == "routing" and not full_copy:
        out["note"] = "payload staged from a pinned ring of 4 per-GPU slices (host RAM limit)"
    return out


if __name__ == "__main__":
    main()
