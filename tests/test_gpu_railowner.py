"""NEXT f2 -- rail-owner pack fused with the intra-node hop (-m gpu, multi-rank).

P ranks form one RailS node (NIC j hangs off GPU j; the intra-domain hop
P:303): each histograms its own source GPUs' rows, the node's message
rows are gathered into every rank (peer stores + flags), every rank runs the same
node-wide schedule, and each packs its rows straight into the rail buffers owned
by the other ranks.  Every owned rail buffer must equal, byte for byte, the
oracle's rail buffer of the node (oracle.pack_node on all N source GPUs, by
definition), after two steps (flags reused: gen 2).

* test_railowner_local_ranks (any box): this process plays the P ranks on cuda:0;
  the two exchanges that wait on other ranks (row gather, barrier) are the *_local
  cooperative launches (one kernel, CTA (u, p) = rank p); histogram, schedule and
  the owner pack run per rank exactly as a rank process would run them.
* test_railowner_per_gpu (boxes with >= P GPUs): railowner.RailOwnerNode, one
  process per GPU, CUDA-IPC peer pointers, NVLink stores.
"""
import numpy as np
import pytest
import torch

import gen
from mp_ranks import run_ranks

pytestmark = pytest.mark.gpu

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
CFGS = [
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1, P=2),   # 2-piece path
    dict(M=4, N=4, T=300, k=2, E=8, RB=1024, C=4096, U=2, d=1, P=4),   # one rail per rank
    dict(M=3, N=4, T=128, k=2, E=6, RB=2048, C=1024, U=1, d=2, P=2),   # C < RB multi-piece
    dict(M=3, N=4, T=100, k=2, E=8, RB=12288, C=32768, U=1, d=0, P=2),  # 12 KiB rows: windows
    dict(M=4, N=8, T=256, k=2, E=8, RB=2048, C=8192, U=2, d=3, P=8),   # a full 8-GPU node
]


def _inputs(cfg):
    M, N, T, k, E, RB, U, d = (cfg[x] for x in "M N T k E RB U d".split())
    seed = 31
    topk_all = torch.stack([gen.routing(M, N, T, k, E, seed, u, d, 1) for u in range(U)])
    x_all = torch.stack([gen.payload(M, N, T, RB, seed, u, d, 1) for u in range(U)])
    return topk_all, x_all, gen.inst_lut(M, N, E)


def _oracle_rails(cfg, topk_all, x_all, lut):
    """Per unit: (send_load, rail bases, node rail buffer) by the oracle's definition."""
    import oracle
    M, N, T, k, RB, C, U, d = (cfg[x] for x in "M N T k RB C U d".split())
    out = []
    for u in range(U):
        c, m, r = oracle.histogram_node(M, N, d, T, k, topk_all[u, 0].numpy(), lut.numpy(), RB)
        s = oracle.schedule_node(m, C)
        L = s["send_load"]
        base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
        want = oracle.pack_node(M, N, d, T, k, RB, C, x_all[u, 0].numpy().view(np.uint8),
                                topk_all[u, 0].numpy(), lut.numpy(), m, s, base, int(L.sum()))
        out.append((L, base, want))
    return out


@pytest.mark.parametrize("cfg", CFGS)
def test_railowner_local_ranks(cfg):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2510_19262_b200 import rails
    dev = torch.device("cuda", 0)
    M, N, T, k, RB, C, U, d, P = (cfg[x] for x in "M N T k RB C U d P".split())
    G = M * N
    ng = N // P
    topk_all, x_all, lut = _inputs(cfg)
    lut_d = lut.to(dev)
    tp, sh = rails.topo(M, N, C), rails.shard(U, d, 1)
    xb, moff = rails.owner_exchange_layout(tp, U, P)
    xbufs = [torch.zeros(xb, dtype=torch.uint8, device=dev) for _ in range(P)]
    xptrs = [b.data_ptr() for b in xbufs]
    cap = (U * (T * k * RB + C) + 255) // 256 * 256  # the RailOwnerNode bound
    own = [torch.zeros(ng * cap, dtype=torch.uint8, device=dev) for _ in range(P)]
    rail_ptrs = [own[j // ng].data_ptr() + (j % ng) * cap for j in range(N)]
    R = []
    for p in range(P):
        g0 = p * ng
        R.append(dict(
            g0=g0, topk=topk_all[:, :, g0:g0 + ng].contiguous().to(dev),
            x=x_all[:, :, g0:g0 + ng].contiguous().to(dev),
            out=(torch.empty((U, 1, ng, G), dtype=torch.int32, device=dev),
                 torch.empty((U, 1, ng, G), dtype=torch.int64, device=dev),
                 torch.empty((U, 1, ng, T, k), dtype=torch.int32, device=dev)),
            msg_node=xbufs[p][moff:moff + U * N * G * 8].view(torch.int64).view(U, 1, N, G),
            sched=rails.Schedule.empty(tp, sh, dev), ws=rails.new_workspace(tp, sh, dev),
            rail_base=torch.empty((U, 1, N), dtype=torch.int64, device=dev),
            rail_total=torch.empty(N, dtype=torch.int64, device=dev)))
    gen_ = [0]

    def step():
        for r in R:  # 1. local histogram of each rank's own source GPUs
            rails.histogram_gpus(tp, sh, r["g0"], r["topk"], lut_d, RB, out=r["out"])
        gen_[0] += 1  # 2. node rows into every rank (one cooperative launch)
        rails.gather_rows_peer_local(tp, U, ng, [r["out"][1] for r in R], gen_[0], xptrs)
        for r in R:  # 3.-4. identical node-wide schedule, owner pack into every rank's rails
            rails.lpt_schedule(tp, sh, r["msg_node"], out=r["sched"], workspace=r["ws"])
            rails.rail_offsets_owner(tp, sh, r["sched"].send_load, r["rail_base"], r["rail_total"])
            rails.pack_owner(tp, sh, r["g0"], T, k, r["x"], r["topk"], lut_d, r["out"][2],
                             r["msg_node"], RB, r["sched"], r["rail_base"], rail_ptrs,
                             [cap] * N)
        gen_[0] += 1  # 5. barrier: every rank's pack precedes every consumer
        rails.peer_barrier_local(P, gen_[0], xptrs)

    step()
    for b in own:
        b.zero_()
    step()  # flags reused
    torch.cuda.synchronize()
    rails.check()
    errors = []
    for u, (L, base, want) in enumerate(_oracle_rails(cfg, topk_all, x_all, lut)):
        for p, r in enumerate(R):
            if not np.array_equal(r["sched"].send_load[u, 0].cpu().numpy(), L):
                errors.append(f"u{u} rank{p} send_load")
        for j in range(N):
            q = j // ng
            rb = int(R[q]["rail_base"][u, 0, j].item())
            got = own[q][(j % ng) * cap + rb:(j % ng) * cap + rb + int(L[j])].cpu().numpy()
            if not np.array_equal(got, want[base[j]:base[j] + L[j]]):
                errors.append(f"u{u} rail{j}")
    assert not errors, errors


def _body(rank, world, dev, cfg):
    import torch.distributed as dist

    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.railowner import RailOwnerNode
    M, N, T, k, RB, C, U, d = (cfg[x] for x in "M N T k RB C U d".split())
    topk_all, x_all, lut = _inputs(cfg)
    node = RailOwnerNode(M, N, T, k, RB, C, U, d, lut.numel(), exchange=cfg.get("ex", "peer"))
    g0, ng = node.g0, node.ng
    topk = topk_all[:, :, g0:g0 + ng].contiguous().to(dev)
    x = x_all[:, :, g0:g0 + ng].contiguous().to(dev)
    lut_d = lut.to(dev)
    for _ in range(2):  # second step reuses the flags (gen 2)
        node.buf.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        node.step(topk, lut_d, x)
        torch.cuda.synchronize()
        dist.barrier()
    rails.check()
    errors = []
    for u, (L, base, want) in enumerate(_oracle_rails(cfg, topk_all, x_all, lut)):
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


if NGPU >= 2:
    @pytest.mark.parametrize("cfg", [c for c in CFGS + [dict(CFGS[0], ex="nccl")]
                                     if c["P"] <= NGPU])
    def test_railowner_per_gpu(cfg):
        run_ranks(_body, cfg["P"], "per_gpu", cfg)
