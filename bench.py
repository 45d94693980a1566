#!/usr/bin/env python
"""Benchmark of the RailS hot path on B200 (one JSON line on rank 0).

Workloads (BASELINE.json configs; gen.CONFIGS):
  c3 (default)  Mixtral 8x7B expert-parallel routing shape -- 64 nodes x 8 rails,
                T = 4096 tokens per GPU, top-2 of 8 experts, H = 4096 bf16 rows
                (RB = 8 KiB), 32 KiB chunks: every row of SURVEY section 8(a).
                --scaling weak (default): every rank holds M/P nodes of each of
                U = P units (64 (unit, node) schedules + packs per GPU per step);
                --scaling strong: one unit, M/P nodes per rank.  The default line
                also carries the strong-scaling measurement ("strong") and the
                batched-histogram roofline on a C4 iteration ("roofline_hist").
  c4            Mixtral 8x22B: 128 nodes x 8 rails, 12 KiB rows, one ITERATION of
                32 layers sharded over the ranks (32/P layers each, every node of a
                layer on one rank: strong scaling, a MAX-only exchange); the pack is
                timed on 16 seeded (node, layer) units per GPU per step (4.5 TiB
                per iteration is too much to pack fully).
  c2            16 nodes x 8 rails, receiver-skew Zipf byte matrices, 1000
                iterations per rank and step (schedule + eval; no routing/payload).
  c1            4 nodes x 4 rails, the small parity case.
A step = one pass of the path over one batch.  value = (unit, node) schedules
completed by all ranks per second of max-over-ranks device time (CUDA events on the
launching stream, barrier + synchronize on both sides, >= 3 warm-up steps).
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
L2_BYTES = 126 * 1000 * 1000
HBM_SPEC_GBS = 8000.0  # BASELINE.json's 8 TB/s denominator (the measured copy peak is the roofline)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c2", "c1", "c4"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="c3/c1/c2: weak (U = P units, M/P nodes each per rank) or strong "
                         "(one unit's nodes split over the ranks); c4 is always an iteration")
    ap.add_argument("--reduce", default="peer", choices=["peer", "nccl"],
                    help="a6 at N > 1: fused finalize over NVLink peer memory, or NCCL")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the strong-scaling and histogram-roofline sub-measurements")
    ap.add_argument("--nvtx", action="store_true", help="NVTX ranges around every phase")
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


def profile_traffic(name: str, key: str):
    """ncu dram__bytes (read + write) per launch recorded in profiles/<name>."""
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        try:
            return json.load(open(p)).get(key)
        except Exception:  # noqa: BLE001
            return None
    return None


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
    """The workload description both arms print."""
    cfg = gen.CONFIGS[args.workload]
    M, N = cfg["M"], cfg["N"]
    if args.workload == "c4":
        L = cfg["U"] // P
        return {"workload": "c4: Mixtral 8x22B routing shape, 128 nodes x 8 rails, one iteration "
                            "of 32 layers sharded over the ranks, T=4096 tokens/GPU, top-2 of 8 "
                            "experts, H=6144 bf16 rows (12 KiB), 32 KiB chunks; pack timed on 16 "
                            "(node, layer) units per GPU",
                "units": cfg["U"], "layers_per_rank": L, "nodes_per_unit": M, "M": M, "N": N,
                "T": cfg["T"], "k": cfg["k"], "row_bytes": cfg["H"] * 2, "chunk_bytes": cfg["C"],
                "pack_sample_units_per_rank": 16, "parallelism": f"layers{P}",
                "a6": "max-only" if P > 1 else "none",
                "l2": l2_note(args.workload, P)}
    strong = args.scaling == "strong"
    U = (1 if strong else P) * (cfg.get("U", 1) if cfg["kind"] == "matrix" else 1)
    nd = M // P if nd is None else nd
    if cfg["kind"] == "routing":
        desc = {"c3": "c3: Mixtral 8x7B EP routing shape, 64 nodes x 8 rails, T=4096 tokens/GPU, "
                      "top-2 of 8 experts, H=4096 bf16 rows (8 KiB), 32 KiB chunks",
                "c1": "c1: 4 nodes x 4 rails, T=4096 tokens/GPU, top-2 of 8 experts, H=4096 "
                      "bf16 rows, 64 KiB chunks"}[args.workload]
        return {"workload": desc, "units": U, "nodes_per_rank": nd * U, "M": M, "N": N,
                "T": cfg["T"], "k": cfg["k"], "row_bytes": cfg["H"] * 2, "chunk_bytes": cfg["C"],
                "parallelism": f"nodes{P}", "scaling": args.scaling,
                "a6": (args.reduce if P > 1 else "none"), "l2": l2_note(args.workload, P, U, nd)}
    return {"workload": "c2: 16 nodes x 8 rails, receiver-skew Zipf s=1.2 byte matrices, 256 MiB "
                        "per source GPU, 1 MiB chunks, 1000 iterations per rank and step",
            "units": U, "nodes_per_rank": nd * U, "M": M, "N": N, "chunk_bytes": cfg["C"],
            "parallelism": f"nodes{P}", "scaling": args.scaling,
            "a6": (args.reduce if P > 1 else "none"), "l2": l2_note(args.workload, P, U, nd)}


def l2_note(name, P, U=1, nd=None):
    """Bytes one step streams per GPU against the 126 MB L2 (why no flush is needed,
    or that one is done)."""
    cfg = gen.CONFIGS[name]
    M, N = cfg["M"], cfg["N"]
    if cfg["kind"] == "routing":
        T, k, RB = cfg["T"], cfg["k"], cfg["H"] * 2
        if name == "c4":
            L = cfg["U"] // P
            ids = L * M * N * T * k * 4 * 2
            pk = 16 * N * T * RB * 3
            b = ids + pk
            what = (f"{ids / 2**30:.1f} GiB routing ids + ranks and ~{pk / 2**30:.1f} GiB of "
                    "sampled pack traffic per step per GPU")
        else:
            nd = M // P if nd is None else nd
            x = U * nd * N * T * RB
            b = x * 3
            what = (f"{x / 2**30:.1f} GiB payload read + ~{2 * x / 2**30:.1f} GiB rail "
                    "buffers written per step per GPU")
    else:
        nd = M // P if nd is None else nd
        b = U * nd * N * M * N * 8 * 6
        what = f"~{b / 2**20:.0f} MiB of byte matrices and schedules per step per GPU"
    return ("inputs larger than L2 (no flush needed): " if b > 4 * L2_BYTES
            else "L2 flushed before every step: ") + what


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
            "scaling": "strong" if args.workload == "c4" else args.scaling,
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
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


def evpair():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def max_over_ranks(v: float, dist, dev, op="max") -> float:
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def timed(step, steps, stream, dist, local, flush=None):
    """W warm-up steps done by the caller; here K timed steps bracketed by barrier +
    synchronize, CUDA events on the launching stream, clocks sampled meanwhile.
    step(i) gets the step index.  Returns (total_ms, launches, clocks)."""
    from paper_2510_19262_b200 import rails
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    rails.launch_count(reset=True)
    with ClockSampler(local) as clk:
        t0, t1 = evpair()
        if flush is None:
            t0.record(stream)
            for i in range(steps):
                step(i)
            t1.record(stream)
            torch.cuda.synchronize()
            total = t0.elapsed_time(t1)
        else:  # L2 flushed between steps, outside the events
            total = 0.0
            for i in range(steps):
                flush()
                t0.record(stream)
                step(i)
                t1.record(stream)
                t1.synchronize()
                total += t0.elapsed_time(t1)
    launches = rails.launch_count(reset=True)
    if dist is not None:
        dist.barrier()
    return total, launches, clk.summary()


# How the line maps onto BASELINE.json's metric ("LPT-scheduled nodes/sec and pack GB/s
# (vs HBM peak) at 1/2/4/8 B200; makespan/OPT").
METRIC_PARTS = {
    "value": "(unit, node) schedules + packs completed per second: the whole step, pack "
             "included (stricter than SURVEY d.1's pack-free nodes/s)",
    "schedule_only": "BASELINE's 'LPT-scheduled nodes/sec' (pack excluded)",
    "pack_gbs / roofline": "BASELINE's 'pack GB/s (vs HBM peak)'",
    "quality": "BASELINE's 'makespan/OPT' (T/T*, makespan/LB with LB <= OPT)",
}


def sched_times(sev, kev, steps):
    """Per-step schedule-part times (ms) between the step's first event and the pack's
    start event.  Reported as the median: step 0 follows the synchronize that opens
    the timed region, so its kernels wait on host launches (its time is in the list)."""
    per = [sev[i].elapsed_time(kev[i][0]) for i in range(steps)]
    return sorted(per)[len(per) // 2], per


def quality_routing(pipe, C, N, dist, dev):
    """makespan/OPT and balance figures (report-side arithmetic on the kernels' outputs):
    T/T* for LPT, ECMP-hash (R#13), uniform (R#41) and the ecmp_nic reading (R#42);
    per-node send makespan over LB = max(ceil(sum/N), w_max, w_(N) + w_(N+1)) <= OPT."""
    f = {k: v.double() for k, v in pipe.final.items()}
    q = {"T_lpt_over_Tstar": float((f["T"] / f["T_star"]).max()),
         "T_ecmp_over_Tstar": float((f["T_e"] / f["T_star"]).max()),
         "T_uniform_over_Tstar": float((f["T_u"] / f["T_star"]).max()),
         "busbw_lpt_over_ecmp": float((f["busbw"] / f["busbw_e"]).min())}
    msg = pipe.msg  # [U][nd][N][G]
    U, nd, _, G = msg.shape
    row = msg.sum(-1).amax().double()             # bytes out of one source GPU's NIC
    col = msg.sum(dim=(1, 2)).double()            # [U][G] bytes into one GPU's NIC (partial)
    if dist is not None:
        dist.all_reduce(row, op=dist.ReduceOp.MAX)
        dist.all_reduce(col, op=dist.ReduceOp.SUM)
    T_nic = torch.maximum(row, col.amax(-1))       # / R2 cancels in the ratio
    q["T_ecmp_nic_over_Tstar"] = float((T_nic / (f["T_star"] * pipe.tp.R2)).max())
    # per-node send makespan / LB
    S = pipe.ev.S.double()                         # [U][nd][N]
    tot = S.sum(-1)
    rem = (msg % C).view(U, nd, -1)
    top = torch.topk(rem, min(N + 1, rem.shape[-1]), dim=-1).values.double()
    nf = pipe.sched.n_full.double().unsqueeze(-1)  # [U][nd][1]
    idx = torch.arange(top.shape[-1], device=dev, dtype=torch.float64)
    # the N+1 largest chunk sizes: min(n_full, N+1) full chunks, then the largest remainders
    shifted = torch.cat([top, torch.zeros_like(top)], dim=-1)
    pos = (idx - nf).clamp(min=0).long()
    w = torch.where(idx < nf, torch.full_like(top, float(C)), torch.gather(shifted, -1, pos))
    wmax = w[..., 0]
    pair = w[..., N - 1] + w[..., N] if w.shape[-1] > N else torch.zeros_like(wmax)
    lb = torch.maximum(torch.ceil(tot / N), torch.maximum(wmax, pair)).clamp(min=1)
    mk = torch.where(tot > 0, S.amax(-1) / lb, torch.ones_like(tot))
    mk_mean = torch.where(tot > 0, S.amax(-1) / torch.ceil(tot / N).clamp(min=1), torch.ones_like(tot))
    q["node_makespan_over_LB_max"] = max_over_ranks(float(mk.max()), dist, dev)
    q["node_makespan_over_mean_max"] = max_over_ranks(float(mk_mean.max()), dist, dev)
    q["LB"] = "max(ceil(sum w / N), w_max, w_(N) + w_(N+1)) per node (<= OPT, SURVEY 8(d) d.1)"
    return q


def hist_roofline(dev, local, steps):
    """Batched histogram roofline on one C4 iteration (32 layers x 128 nodes, 1 GiB of
    routing ids): CUDA events around each launch inside the clock sampler, inputs 20x
    the L2 (no flush).  Algorithmic bytes per launch: ids read + ranks written (4 B
    each per (t, s)) + counts (4 B) and msg_bytes (8 B) per (segment, GPU)."""
    from paper_2510_19262_b200 import rails
    cfg = gen.CONFIGS["c4"]
    M, N, T, k, E, U = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["U"]
    G = M * N
    seed = gen.config_seed(4)
    topk = torch.empty((U, M, N, T, k), dtype=torch.int32, device=dev)
    for u in range(U):
        topk[u] = gen.routing(M, N, T, k, E, seed, u, device=dev)
    lut = gen.inst_lut(M, N, E).to(dev)
    tp, sh = rails.topo(M, N, cfg["C"]), rails.shard(U, 0, M)
    out = (torch.empty((U, M, N, G), dtype=torch.int32, device=dev),
           torch.empty((U, M, N, G), dtype=torch.int64, device=dev),
           torch.empty((U, M, N, T, k), dtype=torch.int32, device=dev))
    run = lambda: rails.histogram(tp, sh, topk, lut, cfg["H"] * 2, out=out)  # noqa: E731
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    evs = [evpair() for _ in range(max(steps, 5))]
    with ClockSampler(local) as clk:
        for a, b in evs:
            a.record(stream)
            run()
            b.record(stream)
        torch.cuda.synchronize()
    rails.check()
    ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    alg = topk.numel() * 4 * 2 + U * M * N * G * (4 + 8)
    peak, kind = measured_peaks()
    ach = alg / (ms / 1000.0) / 1e9
    return {"kernel": "k_hist_w1a", "bound": "hbm", "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak, "peak_kind": kind,
            "frac_of_8TBs_spec": ach / HBM_SPEC_GBS,
            "traffic": profile_traffic("hist_traffic.json", "c4_iteration"),
            "algorithmic_bytes_per_launch": alg, "avg_launch_ms": ms, "launches": len(evs),
            "workload": "one C4 iteration: 32 layers x 128 nodes x 8 GPUs x 4096 tokens x top-2",
            "clocks": clk.summary()}


def main():
    global _JSON_OUT
    # NCCL and CUDA libraries may print banners on fd 1: keep stdout for the JSON line
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    cfg = gen.CONFIGS[args.workload]
    if args.workload == "c4":
        out = run_c4(args, cfg, rank, world, local, dev, dist)
    elif cfg["kind"] == "routing":
        out = run_routing(args, cfg, rank, world, local, dev, dist)
    else:
        out = run_matrix(args, cfg, rank, world, local, dev, dist)
    if rank == 0:
        emit(out)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _peer_or_nccl(args, tp, U, dev, dist):
    """The a6 hook at P > 1: the fused peer-memory finalize, or the NCCL all-reduce."""
    from paper_2510_19262_b200.dist import PeerFinalize, make_reduce
    if dist is None:
        return None, None
    if args.reduce == "peer":
        peer = PeerFinalize(tp, U, dev)
        if peer.ok():
            return peer, peer
        print(f"peer a6 unavailable ({peer.error}); using NCCL", file=sys.stderr)
        peer.close()
        args.reduce = "nccl"
    return make_reduce(), None


def routing_inputs(M, N, T, k, E, RB, seed, U, d0, nd, dev, u0=0):
    topk = torch.empty((U, nd, N, T, k), dtype=torch.int32, device=dev)
    for u in range(U):
        topk[u] = gen.routing(M, N, T, k, E, seed, u0 + u, d0, nd, device=dev)
    x = torch.empty((U, nd, N, T, RB // 8), dtype=torch.int64, device=dev)
    for u in range(U):
        gen.payload(M, N, T, RB, seed, u0 + u, d0, nd, device=dev, out=x[u])
    return topk, x


def run_routing(args, cfg, rank, world, local, dev, dist):
    """c3 / c1: histogram -> fused schedule + eval -> [a6] -> pack per step."""
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import RoutingPipeline
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    P = world
    assert M % P == 0, "M must divide over ranks"
    nd = M // P
    d0 = rank * nd
    if args.nd is not None:
        nd = min(nd, args.nd)
    U = 1 if args.scaling == "strong" else P
    seed = gen.config_seed(int(args.workload[1]))
    topk, x = routing_inputs(M, N, T, k, E, RB, seed, U, d0, nd, dev)
    lut = gen.inst_lut(M, N, E).to(dev)
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, d0, nd, lut.numel(), dev, nvtx=args.nvtx)
    reduce, peer = _peer_or_nccl(args, pipe.tp, U, dev, dist)
    stream = torch.cuda.current_stream()
    kev = [evpair() for _ in range(args.steps)]
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    def step(i=None):
        if i is not None:
            sev[i].record(stream)
        pipe.schedule_part(topk, lut)
        pipe.finalize_part(reduce)
        if i is not None:
            kev[i][0].record(stream)
        pipe.pack_part(topk, lut, x)
        if i is not None:
            kev[i][1].record(stream)

    for _ in range(max(args.warmup, 1)):
        step()
    rails.check()
    total_ms, launches, clocks = timed(step, args.steps, stream, dist, local)
    rails.check()
    total_ms = max_over_ranks(total_ms, dist, dev)
    pack_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    sched_ms, sched_per = sched_times(sev, kev, args.steps)
    nodes = U * nd * P
    value = nodes * args.steps / (total_ms / 1000.0)
    peak, peak_kind = measured_peaks()
    out = {"metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
           "dtype": "int64", "data": "synthetic", "config": arm_config(args, P, nd),
           "metric_parts": METRIC_PARTS}
    sched_ms = max_over_ranks(sched_ms, dist, dev)
    out["schedule_only"] = {
        "value": nodes / (sched_ms / 1000.0), "unit": "nodes/s", "ms_per_step": sched_ms,
        "stat": "median over the timed steps (max over ranks)",
        "per_step_ms": [round(v, 5) for v in sched_per],
        "what": "a1 histogram + a2-a5 fused schedule/eval (+ rail offsets, + finalize at P = 1) "
                "+ a6 exchange per step, pack excluded: SURVEY 8(d) d.1 'LPT-scheduled nodes/s', "
                "eager launches"}
    tokens = U * nd * N * T
    pack_bytes = tokens * RB + int(pipe.total.item())  # each row read once + each copy written
    per_gpu_pack = pack_bytes / (pack_ms / 1000.0) / 1e9
    out["pack_gbs"] = max_over_ranks(pack_bytes, dist, dev, "sum") / (
        max_over_ranks(pack_ms, dist, dev) / 1000.0) / 1e9
    out["roofline"] = {"kernel": "k_pack", "bound": "hbm", "achieved": per_gpu_pack,
                       "peak": peak, "unit": "GB/s", "frac": per_gpu_pack / peak,
                       "peak_kind": peak_kind, "frac_of_8TBs_spec": per_gpu_pack / HBM_SPEC_GBS,
                       "traffic": profile_traffic("pack_traffic.json", args.workload),
                       "peak_note": "peak = a 1:1 HBM copy; the pack moves 1 read : 2 writes "
                                    "(writes stream faster), so frac can pass 1.0",
                       "algorithmic_bytes_per_launch": pack_bytes, "avg_launch_ms": pack_ms,
                       "share_of_step": pack_ms / (total_ms / args.steps)}
    out["quality"] = quality_routing(pipe, C, N, dist, dev)
    out["clocks"] = clocks
    out["gpu_launches"] = int(launches)
    if world == 1 and not args.no_graph:
        out["graph"], out["schedule_only"]["graph"] = graph_replay(pipe, topk, lut, x, args,
                                                                    stream, nodes, dev)
    if not args.no_e2e:
        out["e2e"] = e2e_routing(args, pipe, topk, lut, x, reduce, stream, dist, world, dev, nodes)
    if peer is not None:
        peer.close()
    del pipe, x, topk
    torch.cuda.empty_cache()
    if not args.no_extra and args.workload == "c3" and args.scaling == "weak":
        out["strong"] = strong_c3(args, cfg, rank, world, local, dev, dist, out)
        out["roofline_hist"] = hist_roofline(dev, local, args.steps)
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = oracle_sample(args.workload)
        out["cpu_baseline"]["all_cores"] = oracle_sample_all_cores(args.workload)
    return out


def strong_c3(args, cfg, rank, world, local, dev, dist, weak):
    """SURVEY 8(d) d.2 strong scaling of C3: ONE unit, M/P nodes per rank, the a6
    exchange every step.  At P = 1 it is the main line's configuration."""
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import RoutingPipeline
    if world == 1:
        return {"value": weak["value"], "unit": "nodes/s", "ms_per_step": weak["ms_per_step"],
                "nodes_per_rank": cfg["M"], "note": "P = 1: the main line's configuration"}
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    nd = M // world
    d0 = rank * nd
    seed = gen.config_seed(3)
    topk, x = routing_inputs(M, N, T, k, E, RB, seed, 1, d0, nd, dev)
    lut = gen.inst_lut(M, N, E).to(dev)
    pipe = RoutingPipeline(M, N, T, k, RB, C, 1, d0, nd, lut.numel(), dev)
    reduce, peer = _peer_or_nccl(args, pipe.tp, 1, dev, dist)
    stream = torch.cuda.current_stream()
    step = lambda i=None: pipe.step(topk, lut, x, reduce)  # noqa: E731
    for _ in range(max(args.warmup, 1)):
        step()
    rails.check()
    total_ms, _, clocks = timed(step, args.steps, stream, dist, local)
    rails.check()
    total_ms = max_over_ranks(total_ms, dist, dev)
    if peer is not None:
        peer.close()
    return {"value": M * args.steps / (total_ms / 1000.0), "unit": "nodes/s",
            "ms_per_step": total_ms / args.steps, "nodes_per_rank": nd, "units": 1,
            "a6": args.reduce, "clocks": clocks,
            "what": "one C3 unit (64 nodes) split over the ranks; every step ends in the a6 "
                    "exchange (strong scaling, SURVEY 8(d) d.2)"}


def graph_replay(pipe, topk, lut, x, args, stream, nodes, dev):
    """The same step captured once into a CUDA graph and replayed; and the schedule
    part alone, L2 flushed before each replay."""
    from paper_2510_19262_b200.pipeline import GraphStep
    g = GraphStep(lambda: pipe.step(topk, lut, x))
    torch.cuda.synchronize()
    g0, g1 = evpair()
    g0.record(stream)
    for _ in range(args.steps):
        g()
    g1.record(stream)
    torch.cuda.synchronize()
    gms = g0.elapsed_time(g1) / args.steps
    full = {"value": nodes / (gms / 1000.0), "unit": "nodes/s", "ms_per_step": gms,
            "what": "the same step captured once into a CUDA graph and replayed"}
    del g
    g = GraphStep(lambda: pipe.schedule_part(topk, lut))
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
    sched = {"value": nodes / (sms / 1000.0), "ms_per_step": sms,
             "what": "the schedule part alone captured into a CUDA graph and replayed, L2 "
                     "flushed before each replay"}
    return full, sched


def e2e_routing(args, pipe, topk, lut, x, reduce, stream, dist, world, dev, nodes):
    """Same metric through the public API with HOST buffers: every step copies the
    routing and the payload in from pinned memory and copies the results out -- the
    per-unit finals AND the compact schedule + rail offsets a host-side RDMA transport
    consumes (the packed rail buffers stay in HBM for GPUDirect RDMA)."""
    import psutil

    from paper_2510_19262_b200 import rails
    steps = max(1, args.e2e_steps)
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
        # host RAM cannot pin every rank's payload: stage the same number of bytes per
        # step from a pinned ring of 4 per-GPU slices (contents repeat)
        h_x = torch.empty((4,) + tuple(xs.shape[1:]), dtype=x.dtype, pin_memory=True)
        h_x.copy_(xs[:4])
    s = pipe.sched
    outs = dict(pipe.final)
    outs.update(full_base=s.full_base, rem_rail=s.rem_rail, rem_off=s.rem_off,
                send_load=s.send_load, n_full=s.n_full, n_rem=s.n_rem, rail_base=pipe.rail_base)
    h_res = {kk: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for kk, v in outs.items()}

    def one():
        topk.copy_(h_topk, non_blocking=True)
        if full_copy:
            x.copy_(h_x, non_blocking=True)
        else:
            for i in range(xs.shape[0]):
                xs[i].copy_(h_x[i % 4], non_blocking=True)
        pipe.step(topk, lut, x, reduce)
        for kk, vv in outs.items():
            h_res[kk].copy_(vv, non_blocking=True)

    h2d = h_topk.numel() * 4 + x.numel() * 8
    d2h = sum(v.numel() * v.element_size() for v in outs.values())
    # ranks may be seconds apart after pinning multi-GiB host buffers; the first call
    # ends in the peer-memory a6, whose waits must not time out
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    one()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = evpair()
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    e1.synchronize()
    rails.check()  # device-side errors (range, capacity, peer timeout) of the e2e steps
    ms = max_over_ranks(e0.elapsed_time(e1), dist, dev)
    res = {"value": nodes * steps / (ms / 1000.0), "unit": "nodes/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
           "d2h": "per-unit finals + compact schedule (full_base, rem_rail, rem_off, send_load, "
                  "n_full, n_rem) + rail offsets; rail buffers stay device-resident for "
                  "GPUDirect RDMA"}
    if not full_copy:
        res["note"] = "payload staged from a pinned ring of 4 per-GPU slices (host RAM limit)"
    return res


def run_c4(args, cfg, rank, world, local, dev, dist):
    """One C4 iteration per step: 32 layers sharded 32/P per rank (every node of a
    layer on its rank, so each unit is finalized in the rank's own kernels), then a
    MAX-only exchange of the iteration's completion time; the pack runs on 16 seeded
    (node, layer) units per GPU per step."""
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import RoutingPipeline
    M, N, T, k, E, C, UT = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"], cfg["U"]
    RB = cfg["H"] * 2
    P = world
    assert UT % P == 0, "32 layers must divide over ranks"
    L = UT // P
    seed = gen.config_seed(4)
    topk = torch.empty((L, M, N, T, k), dtype=torch.int32, device=dev)
    for u in range(L):
        topk[u] = gen.routing(M, N, T, k, E, seed, rank * L + u, device=dev)
    lut = gen.inst_lut(M, N, E).to(dev)
    pipe = RoutingPipeline(M, N, T, k, RB, C, L, 0, M, lut.numel(), dev, out_cap=16,
                           nvtx=args.nvtx)
    # pack sample: 16 consecutive nodes of the rank's first layer
    SN = 16
    sd0 = (rank * SN) % M
    sx = torch.empty((1, SN, N, T, RB // 8), dtype=torch.int64, device=dev)
    gen.payload(M, N, T, RB, seed, rank * L, sd0, SN, device=dev, out=sx[0])
    ssh = rails.shard(1, sd0, SN)
    sl = slice(sd0, sd0 + SN)
    ssched = rails.Schedule(*(t[0:1, sl] for t in (pipe.sched.full_base, pipe.sched.rem_rail,
                                                    pipe.sched.rem_off, pipe.sched.send_load,
                                                    pipe.sched.n_full, pipe.sched.n_rem)))
    srb = torch.empty((1, SN, N), dtype=torch.int64, device=dev)
    stot = torch.empty(1, dtype=torch.int64, device=dev)
    sout = torch.empty(SN * N * T * k * RB, dtype=torch.uint8, device=dev)
    stopk, srank, smsg = topk[0:1, sl], pipe.rank[0:1, sl], pipe.msg[0:1, sl]
    tmax = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    kev = [evpair() for _ in range(args.steps)]
    sev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    def step(i=None):
        if i is not None:
            sev[i].record(stream)
        pipe.schedule_part(topk, lut)           # every layer x node of the rank
        if dist is not None:                    # the iteration's completion time: MAX only
            torch.amax(pipe.final["T"], dim=0, keepdim=True, out=tmax)
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        rails.rail_offsets(pipe.tp, ssh, ssched.send_load, srb, stot)
        if i is not None:
            kev[i][0].record(stream)
        rails.pack(pipe.tp, ssh, T, k, sx, stopk, lut, srank, smsg, RB, ssched, srb, sout)
        if i is not None:
            kev[i][1].record(stream)

    for _ in range(max(args.warmup, 1)):
        step()
    rails.check()
    total_ms, launches, clocks = timed(step, args.steps, stream, dist, local)
    rails.check()
    total_ms = max_over_ranks(total_ms, dist, dev)
    pack_ms = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    sched_ms, sched_per = sched_times(sev, kev, args.steps)
    sched_ms = max_over_ranks(sched_ms, dist, dev)
    nodes = UT * M  # (node, layer) schedules of the whole iteration, all ranks together
    peak, peak_kind = measured_peaks()
    pack_bytes = SN * N * T * RB + int(stot.item())
    per_gpu_pack = pack_bytes / (pack_ms / 1000.0) / 1e9
    out = {"metric": METRIC, "value": nodes * args.steps / (total_ms / 1000.0), "unit": "nodes/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "int64", "data": "synthetic",
           "config": arm_config(args, P), "metric_parts": METRIC_PARTS,
           "schedule_only": {"value": nodes / (sched_ms / 1000.0), "unit": "nodes/s",
                             "ms_per_step": sched_ms,
                             "stat": "median over the timed steps (max over ranks)",
                             "per_step_ms": [round(v, 5) for v in sched_per],
                             "what": "histogram + schedule + eval + finalize of the rank's "
                                     "layers + the MAX exchange, sampled pack excluded"},
           "pack_gbs": max_over_ranks(pack_bytes, dist, dev, "sum") / (
               max_over_ranks(pack_ms, dist, dev) / 1000.0) / 1e9,
           "roofline": {"kernel": "k_pack", "bound": "hbm", "achieved": per_gpu_pack,
                        "peak": peak, "unit": "GB/s", "frac": per_gpu_pack / peak,
                        "peak_kind": peak_kind, "frac_of_8TBs_spec": per_gpu_pack / HBM_SPEC_GBS,
                        "traffic": profile_traffic("pack_traffic.json", "c4"),
                        "algorithmic_bytes_per_launch": pack_bytes, "avg_launch_ms": pack_ms,
                        "share_of_step": pack_ms / (total_ms / args.steps)},
           "quality": quality_routing(pipe, C, N, None, dev),
           "clocks": clocks, "gpu_launches": int(launches)}
    if not args.no_e2e:
        out["e2e"] = e2e_c4(args, pipe, topk, lut, step, stream, dist, dev, nodes)
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = oracle_sample(args.workload, budget_s=15.0, max_nodes=8)
    return out


def e2e_c4(args, pipe, topk, lut, step, stream, dist, dev, nodes):
    """C4 through the public API with host buffers: the iteration's routing ids in
    from pinned memory, the per-layer finals and compact schedules out, per step."""
    from paper_2510_19262_b200 import rails
    steps = max(1, args.e2e_steps)
    h_topk = torch.empty(topk.shape, dtype=topk.dtype, pin_memory=True)
    h_topk.copy_(topk)
    s = pipe.sched
    outs = dict(pipe.final)
    outs.update(full_base=s.full_base, rem_rail=s.rem_rail, rem_off=s.rem_off,
                send_load=s.send_load, n_full=s.n_full, n_rem=s.n_rem)
    h_res = {kk: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for kk, v in outs.items()}

    def one():
        topk.copy_(h_topk, non_blocking=True)
        step()
        for kk, vv in outs.items():
            h_res[kk].copy_(vv, non_blocking=True)

    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    one()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = evpair()
    e0.record(stream)
    for _ in range(steps):
        one()
    e1.record(stream)
    e1.synchronize()
    rails.check()
    ms = max_over_ranks(e0.elapsed_time(e1), dist, dev)
    return {"value": nodes * steps / (ms / 1000.0), "unit": "nodes/s",
            "h2d_bytes_per_step": int(h_topk.numel() * 4),
            "d2h_bytes_per_step": int(sum(v.numel() * v.element_size() for v in outs.values())),
            "steps": steps,
            "note": "the 16 sampled units' payload is device-resident (see config)"}


def run_matrix(args, cfg, rank, world, local, dev, dist):
    """c2: byte matrices, schedule + eval per step."""
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import MatrixPipeline
    M, N, C = cfg["M"], cfg["N"], cfg["C"]
    P = world
    assert M % P == 0, "M must divide over ranks"
    nd = M // P
    d0 = rank * nd
    U = (1 if args.scaling == "strong" else P) * cfg.get("U", 1)
    seed = gen.config_seed(int(args.workload[1]))
    msg = torch.from_numpy(gen.d1_units(cfg, seed, 0, U)[:, d0:d0 + nd].copy()).to(dev)
    pipe = MatrixPipeline(M, N, C, U, d0, nd, dev)
    reduce, peer = _peer_or_nccl(args, pipe.tp, U, dev, dist)
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    step = lambda i=None: pipe.step(msg, reduce)  # noqa: E731
    for _ in range(max(args.warmup, 1)):
        step()
    rails.check()
    total_ms, launches, clocks = timed(step, args.steps, stream, dist, local,
                                       flush=lambda: flush_buf.fill_(1))
    rails.check()
    total_ms = max_over_ranks(total_ms, dist, dev)
    nodes = U * nd * P
    f = {kk: v.double() for kk, v in pipe.final.items()}
    out = {"metric": METRIC, "value": nodes * args.steps / (total_ms / 1000.0), "unit": "nodes/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": total_ms / args.steps, "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic",
           "config": arm_config(args, P, nd),
           "quality": {"T_lpt_over_Tstar": float((f["T"] / f["T_star"]).max()),
                       "T_ecmp_over_Tstar": float((f["T_e"] / f["T_star"]).max()),
                       "T_uniform_over_Tstar": float((f["T_u"] / f["T_star"]).max())},
           "clocks": clocks, "gpu_launches": int(launches)}
    if not args.no_e2e:
        h_msg = torch.empty(msg.shape, dtype=msg.dtype, pin_memory=True)
        h_msg.copy_(msg)
        s = pipe.sched
        outs = dict(pipe.final)
        outs.update(full_base=s.full_base, rem_rail=s.rem_rail, rem_off=s.rem_off,
                    send_load=s.send_load)
        h_res = {kk: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for kk, v in outs.items()}

        def one():
            msg.copy_(h_msg, non_blocking=True)
            pipe.step(msg, reduce)
            for kk, vv in outs.items():
                h_res[kk].copy_(vv, non_blocking=True)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        one()
        torch.cuda.synchronize()
        e0, e1 = evpair()
        e0.record(stream)
        for _ in range(max(1, args.e2e_steps)):
            one()
        e1.record(stream)
        e1.synchronize()
        rails.check()
        ms = max_over_ranks(e0.elapsed_time(e1), dist, dev)
        out["e2e"] = {"value": nodes * max(1, args.e2e_steps) / (ms / 1000.0), "unit": "nodes/s",
                      "h2d_bytes_per_step": int(h_msg.numel() * 8),
                      "d2h_bytes_per_step": int(sum(v.numel() * v.element_size()
                                                    for v in outs.values()))}
    if peer is not None:
        peer.close()
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"] = oracle_sample(args.workload)
        out["cpu_baseline"]["all_cores"] = oracle_sample_all_cores(args.workload)
    return out


if __name__ == "__main__":
    main()
