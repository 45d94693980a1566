"""NEXT f2 -- rail-owner pack fused with the intra-node hop (-m gpu, multi-rank).

P processes form one RailS node (NIC j hangs off GPU j; the intra-domain hop
P:303): each packs its own source GPUs' rows into the rail buffers owned
by the other ranks through CUDA-IPC peer pointers.  Every owned rail buffer must
equal, byte for byte, the oracle's rail buffer of the node (oracle.pack_node on all
N source GPUs, by definition), after two steps (flags reused: gen 2).

Runs on any box: all ranks on cuda:0 (gloo) always, one rank per GPU (NCCL, NVLink
stores) when the box has enough GPUs (tests/mp_ranks.py).
"""
import numpy as np
import pytest
import torch

import gen
from mp_ranks import placements, run_ranks

pytestmark = pytest.mark.gpu


def _body(rank, world, dev, cfg):
    import torch.distributed as dist

    import oracle
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.railowner import RailOwnerNode
    M, N, T, k, E, RB, C, U, d = (cfg[x] for x in "M N T k E RB C U d".split())
    seed = 31
    topk_all = torch.stack([gen.routing(M, N, T, k, E, seed, u, d, 1) for u in range(U)])
    x_all = torch.stack([gen.payload(M, N, T, RB, seed, u, d, 1) for u in range(U)])
    lut = gen.inst_lut(M, N, E)
    node = RailOwnerNode(M, N, T, k, RB, C, U, d, lut.numel(), exchange=cfg.get("ex", "peer"))
    g0, ng = node.g0, node.ng
    topk = topk_all[:, :, g0:g0 + ng].contiguous().to(dev)
    x = x_all[:, :, g0:g0 + ng].contiguous().to(dev)
    lut_d = lut.to(dev)
    node.buf.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    node.step(topk, lut_d, x)
    torch.cuda.synchronize()
    dist.barrier()
    node.buf.zero_()  # a second step re-gathers and re-packs (flags reused, gen 2)
    torch.cuda.synchronize()
    dist.barrier()
    node.step(topk, lut_d, x)
    torch.cuda.synchronize()
    rails.check()
    errors = []
    for u in range(U):
        c, m, r = oracle.histogram_node(M, N, d, T, k, topk_all[u, 0].numpy(), lut.numpy(), RB)
        s = oracle.schedule_node(m, C)
        L = s["send_load"]
        base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
        want = oracle.pack_node(M, N, d, T, k, RB, C, x_all[u, 0].numpy().view(np.uint8),
                                topk_all[u, 0].numpy(), lut.numpy(), m, s, base, int(L.sum()))
        if not np.array_equal(node.sched.send_load[u, 0].cpu().numpy(), L):
            errors.append(f"u{u} send_load")
        rb = node.rail_base[u, 0].cpu().numpy()
        for j in range(g0, g0 + ng):
            got = node.own_rail(j)[int(rb[j]):int(rb[j]) + int(L[j])].cpu().numpy()
            if not np.array_equal(got, want[base[j]:base[j] + L[j]]):
                errors.append(f"u{u} rail{j}")
    dist.barrier()
    node.close()
    return errors


@pytest.mark.parametrize("cfg", [
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1, P=2),   # 2-piece path
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1, P=4),   # one rail per rank
    dict(M=3, N=4, T=128, k=2, E=6, RB=2048, C=1024, U=1, d=2, P=2),   # C < RB multi-piece
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1, P=2, ex="nccl"),  # collective
    dict(M=3, N=4, T=100, k=2, E=8, RB=12288, C=32768, U=1, d=0, P=2),  # 12 KiB rows: windows
])
def test_railowner_pack_matches_oracle(cfg):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    for placement in placements(cfg["P"]):
        run_ranks(_body, cfg["P"], placement, cfg)
