"""NEXT f1 -- the combine all-to-all and unpack (-m gpu), element by element vs the
oracle: transposed traffic and receive offsets (exact), the combine round's LPT
schedule (exact), combine rail buffers (byte-exact), and the top-k weighted
combine (fp32, bit-exact: the same products and sums in the same order, no FMA)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import compare_schedule, routing_inputs

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2510_19262_b200 import rails
    from paper_2510_19262_b200.pipeline import RoutingPipeline

DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    rails.check()


@pytest.mark.parametrize("M,N,T,k,E,RB,C,U", [
    (4, 4, 200, 2, 8, 256, 1024, 2),     # C >= RB
    (3, 2, 150, 3, 6, 512, 192, 1),      # C < RB, C not a power of two
    (5, 4, 64, 2, 8, 4096, 32768, 1),    # 4 KiB rows, 32 KiB chunks
    (3, 2, 150, 2, 6, 512, 192, 1),      # k = 2 (two-slot kernel) with C < RB
    (4, 4, 100, 1, 8, 1024, 4096, 2),    # k = 1 (one-slot kernel)
])
def test_combine_round_and_unpack(M, N, T, k, E, RB, C, U):
    G = M * N
    topk, lut = routing_inputs(M, N, T, k, E, 17, 0, U)
    x = torch.stack([gen.payload(M, N, T, RB, 17, u, 0, M) for u in range(U)])
    disp = RoutingPipeline(M, N, T, k, RB, C, U, 0, M, lut.numel(), DEV)
    disp.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
    tp, sh = disp.tp, disp.sh
    # combine traffic and expert-output layout
    msg_t = rails.transpose_traffic(tp, disp.msg)
    in_off, rows_in = rails.recv_offsets(tp, disp.counts)
    sched_c = rails.lpt_schedule(tp, sh, msg_t)
    rb_c, tot_c = rails.rail_offsets(tp, sh, sched_c.send_load)
    torch.cuda.synchronize()
    Rcap = int(rows_in.max().item())
    y = torch.stack([gen.expert_outputs((M, N, Rcap, RB // 2), 23, u) for u in range(U)])
    comb = torch.zeros(int(tot_c.item()) + 16, dtype=torch.uint8, device=DEV)
    rails.pack_combine(tp, sh, RB, y.to(DEV), in_off, rows_in, msg_t, sched_c, rb_c, comb)
    w = torch.stack([gen.gate_weights((M, N, T, k), 29, u) for u in range(U)])
    out = rails.unpack_combine(tp, sh, T, k, topk.to(DEV), lut.to(DEV), disp.rank, w.to(DEV),
                               y.to(DEV), in_off, msg_t, sched_c, rb_c, comb, RB)
    torch.cuda.synchronize()
    rails.check()
    msg_c, counts_c = disp.msg.cpu().numpy(), disp.counts.cpu().numpy()
    rank_c = disp.rank.cpu().numpy()
    comb_c = comb.cpu().numpy()
    y_b = y.numpy().view(np.uint8)  # [U][M][N][Rcap][RB]
    for u in range(U):
        mt = oracle.transpose(M, N, msg_c[u])
        assert np.array_equal(msg_t[u].cpu().numpy(), mt)
        cnt_flat = counts_c[u].reshape(G, G).astype(np.int64)
        io = np.stack([oracle.recv_offsets(cnt_flat[:, b]) for b in range(G)])
        assert np.array_equal(in_off[u].cpu().numpy(), io)
        assert np.array_equal(rows_in[u].cpu().numpy(), cnt_flat.sum(axis=0))
        scheds = [oracle.schedule_node(mt[f], C) for f in range(M)]
        rbase_all = rb_c[u].cpu().numpy()
        rails_bytes, rail_bases, firsts = [], [], []
        for f in range(M):
            compare_schedule(sched_c, u, f, scheds[f], f"combine u{u} f{f}")
            L = scheds[f]["send_load"]
            base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
            start = int(rbase_all[f, 0])
            assert np.array_equal(rbase_all[f] - start, base)
            want = oracle.pack_combine_node(M, N, f, RB, C, [y_b[u, f, m] for m in range(N)],
                                            io[f * N:(f + 1) * N], mt[f], scheds[f], base,
                                            int(L.sum()))
            got = comb_c[start:start + int(L.sum())]
            assert np.array_equal(got, want), f"combine pack u{u} f{f}"
            rails_bytes.append(want)
            rail_bases.append(base)
            firsts.append(oracle.first_chunk_table(N, G, scheds[f]))
        out_u = out[u].cpu().numpy()
        for d in range(M):
            for g in range(N):
                ref = oracle.unpack_combine(M, N, d, g, T, k, RB, C, topk[u, d, g].numpy(),
                                            lut.numpy(), rank_c[u, d, g], w[u, d, g].numpy(),
                                            [y_b[u, d, m] for m in range(N)],
                                            io[d * N:(d + 1) * N], rails_bytes, rail_bases,
                                            firsts, scheds)
                assert np.array_equal(out_u[d, g].view(np.uint32), ref.view(np.uint32)), (u, d, g)
