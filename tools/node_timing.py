#!/usr/bin/env python
"""Phase timeline of the fused per-node kernel on C3 (debug build with
-DRAILS_NODE_TIMING: globaltimer stamps of CTA 0 at each phase boundary, plus the
unit's last CTA's finalize end and the grid's last CTA's rail-offset end).  Builds
the debug library under gpurun_out/ and runs it; prints JSON.  Not part of the
product (the product library has no timing code)."""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build_debug(out_dir, extra=()):
    from paper_2510_19262_b200 import build as b
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in b.SOURCES:
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        subprocess.check_call([b.NVCC, *b.FLAGS, "-DRAILS_NODE_TIMING", *extra, "-c",
                               os.path.join(b.CSRC, src), "-o", obj],
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        objs.append(obj)
    lib = os.path.join(out_dir, "librails_timing.so")
    subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-o", lib, *objs])
    return lib


def main():
    extra = [a for a in sys.argv[1:] if a.startswith("-D")]
    lib = build_debug(os.path.join(ROOT, "gpurun_out", "timing_build"), extra)
    from paper_2510_19262_b200 import rails
    rails.LIB_PATH = lib
    import torch
    from tools.sched_bench import routing_pipe
    L = rails.lib()
    L.rails_debug_node_times.argtypes = [ctypes.c_void_p]
    L.rails_debug_node_cta.argtypes = [ctypes.c_void_p]
    L.rails_debug_node_reset()
    pipe, topk, lut = routing_pipe("c3", 1)
    rails.histogram(pipe.tp, pipe.sh, topk, lut, pipe.RB, out=(pipe.counts, pipe.msg, pipe.rank))
    names = {1: "start A", 2: "B sort", 3: "C chain", 4: "chain start (warp 0)", 5: "D expand",
             6: "E eval", 7: "F publish", 8: "CTA0 end", 9: "chain end (warp 0)",
             10: "unit-last finalize end", 11: "grid-last rail offsets end",
             13: "workers' message pass end", 0: "kernel entry (before PDL wait)",
             14: "A: first tile loads consumed", 15: "A: first tile scanned",
             16: "A: tiles done", 17: "A: key or/and reduced",
             12: "F: unit-last CTA elected", 18: "F: its fence done",
             19: "F: record copied (thread 0)", 24: "chain second pass start (CHAIN_TWICE)",
             30: "F: record copied (all threads)"}
    alone = lambda: rails.schedule_eval(  # noqa: E731
        pipe.tp, pipe.sh, pipe.msg, pipe.sched, pipe.ev, pipe.ws, final=pipe.final,
        rail_base=pipe.rail_base, rail_total=pipe.total)
    part = lambda: pipe.schedule_part(topk, lut)  # noqa: E731 -- histogram + PDL launch
    runs = {}
    for mode, fn in (("schedule_eval alone", alone), ("schedule part (histogram, PDL)", part)):
        out = []
        for it in range(6):
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            fn()
            s1.record()
            torch.cuda.synchronize()
            t = (ctypes.c_ulonglong * 32)()
            L.rails_debug_node_times(t)
            t0 = t[1]
            ct = (ctypes.c_ulonglong * 2048)()
            L.rails_debug_node_cta(ct)
            nseg = pipe.sched.n_rem.numel()
            cta = [[ct[k * 512 + b] for b in range(nseg)] for k in range(4)]
            a0 = min(cta[0])
            per = {"A start": [round((x - a0) / 1000.0, 2) for x in cta[0]],
                   "A+B": [round((c - x) / 1000.0, 2) for x, c in zip(cta[0], cta[1])],
                   "C": [round((c - x) / 1000.0, 2) for x, c in zip(cta[1], cta[2])],
                   "D+E": [round((c - x) / 1000.0, 2) for x, c in zip(cta[2], cta[3])],
                   "F arrival": [round((x - a0) / 1000.0, 2) for x in cta[3]]}
            nrem = pipe.sched.n_rem.reshape(-1).tolist()
            slow = sorted(range(nseg), key=lambda b: -per["F arrival"][b])[:4]
            summ = {k: {"min": min(v), "median": sorted(v)[len(v) // 2], "max": max(v)}
                    for k, v in per.items()}
            summ["slowest CTAs"] = [{"cta": b, "n_rem": nrem[b], **{k: per[k][b] for k in per}}
                                   for b in slow]
            summ["fastest CTA"] = min(range(nseg), key=lambda b: per["F arrival"][b])
            out.append({"per_cta": summ,"event_us": round(s0.elapsed_time(s1) * 1000, 2),
                        **{names[i]: round((t[i] - t0) / 1000.0, 2) for i in sorted(names)
                           if t[i] > 0},
                        "chain_counts(runs,steps,windows,groups8)": [t[20], t[21], t[22], t[23]],
                        "chain_cycles(run_end,lead,run_record,whole)": [t[25], t[26], t[27],
                                                                        t[28]],
                        "n_rem_node0": int(pipe.sched.n_rem[0, 0])})
            L.rails_debug_node_reset()
        runs[mode] = out[-2:]
    print(json.dumps(runs, indent=1))


if __name__ == "__main__":
    main()
