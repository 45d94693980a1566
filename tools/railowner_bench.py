#!/usr/bin/env python
"""NEXT f2 benchmark: rail-owner pack fused with the NVLink hop (run under torchrun,
one process per GPU; P GPUs of a box form one RailS node of N = 8 rails).

Per step: histogram of the local rows, NCCL all-gather of the node's message
rows, node-wide LPT schedule, rail offsets, and the fused pack that stores every
chunk piece into the rail owner's HBM through peer pointers.  Reports max-over-
ranks device time, pack-kernel time, bytes written to peers (NVLink) and local,
and the fraction of the NVLink store roofline (770 GB/s per direction per GPU,
the measured peer-copy figure of the B200 profiling guide; 900 nominal).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gen  # noqa: E402
from paper_2510_19262_b200 import rails  # noqa: E402
from paper_2510_19262_b200.railowner import RailOwnerNode  # noqa: E402

NVLINK_GBS = 770.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=8)
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = gen.CONFIGS["c3"]
    M, N, T, k, E, C = cfg["M"], cfg["N"], cfg["T"], cfg["k"], cfg["E"], cfg["C"]
    RB = cfg["H"] * 2
    U, d = a.units, 0
    seed = gen.config_seed(3)
    node = RailOwnerNode(M, N, T, k, RB, C, U, d, M * E, exchange=a.exchange)
    g0, ng = node.g0, node.ng
    topk = torch.stack([gen.routing(M, N, T, k, E, seed, u, d, 1, device=dev)
                        for u in range(U)])[:, :, g0:g0 + ng].contiguous()
    x = torch.stack([gen.payload(M, N, T, RB, seed, u, d, 1, device=dev)
                     for u in range(U)])[:, :, g0:g0 + ng].contiguous()
    lut = gen.inst_lut(M, N, E).to(dev)
    for _ in range(a.warmup):
        node.step(topk, lut, x)
    torch.cuda.synchronize()
    rails.check()
    # bytes this rank writes: its rows' remote copies; to peers: rails owned elsewhere
    r = node.rank_loc.cpu()
    topk_c = topk.cpu()
    lut_c = lut.cpu()
    h = lut_c[topk_c.long()]  # [U][1][ng][T][k]
    remote = (h // N) != d
    wr_bytes = int(remote.sum()) * RB
    rd_bytes = U * ng * T * RB
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(a.steps):
        node.schedule_part(topk, lut)
        ev[i][0].record()
        node.pack_part(topk, lut, x)
        ev[i][1].record()
        node.fence()
    t1.record()
    torch.cuda.synchronize()
    rails.check()
    step_ms = t0.elapsed_time(t1) / a.steps
    pack_ms = sum(s.elapsed_time(e) for s, e in ev) / a.steps
    tt = torch.tensor([step_ms, pack_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    step_ms, pack_ms = float(tt[0]), float(tt[1])
    # chunk pieces land on rail j with probability ~1/N; owner = j // ng
    peer_frac = 1.0 - ng / N
    nv_bytes = wr_bytes * peer_frac
    out = {"mode": "railowner", "exchange": a.exchange, "n_gpus": world, "units_per_step": U,
           "N_rails": N,
           "rails_per_gpu": ng, "step_ms": step_ms, "pack_ms": pack_ms,
           "pack_read_bytes_per_gpu": rd_bytes, "pack_write_bytes_per_gpu": wr_bytes,
           "nvlink_bytes_per_gpu_est": nv_bytes,
           "pack_gbs_per_gpu": (rd_bytes + wr_bytes) / (pack_ms / 1e3) / 1e9,
           "nvlink_store_gbs_per_gpu": nv_bytes / (pack_ms / 1e3) / 1e9,
           "nvlink_roofline_frac": nv_bytes / (pack_ms / 1e3) / 1e9 / NVLINK_GBS,
           "nodes_per_s": U / (step_ms / 1e3)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    node.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
