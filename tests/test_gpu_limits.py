"""Limits of the boundary (-m gpu): N = 32 rails (every warp lane), k = 32 slots,
T*k beyond the warp-per-segment histogram (65535 entries), many units -- each run
through the whole path and compared with the oracle element by element."""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import compare_schedule, oracle_eval_from_scheds, routing_inputs

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
    (2, 32, 96, 2, 32, 256, 4096, 1),      # N = 32: warp chain, eval tile of 8 nodes
    (3, 4, 40, 32, 32, 64, 192, 1),        # k = 32 slots per token
    (2, 2, 40000, 2, 4, 16, 4096, 1),      # T*k = 80000 > 65535: two-pass histogram
    (3, 8, 64, 2, 8, 128, 1024, 40),       # 40 units x 3 nodes in one launch
])
def test_limits_full_path(M, N, T, k, E, RB, C, U):
    topk, lut = routing_inputs(M, N, T, k, E, 41, 0, U)
    x = torch.stack([gen.payload(M, N, T, RB, 41, u, 0, M) for u in range(U)])
    pipe = RoutingPipeline(M, N, T, k, RB, C, U, 0, M, lut.numel(), DEV)
    pipe.step(topk.to(DEV), lut.to(DEV), x.to(DEV))
    torch.cuda.synchronize()
    for u in range(U):
        res = oracle.run_unit_routing(M, N, T, k, RB, C, 5.0e10, oracle.DEFAULT_ECMP_SEED,
                                      topk[u].numpy(), lut.numpy())
        assert np.array_equal(pipe.counts[u].cpu().numpy(), res["counts"])
        assert np.array_equal(pipe.rank[u].cpu().numpy(), res["rank"])
        for d in range(M):
            compare_schedule(pipe.sched, u, d, res["scheds"][d], f"u{u} d{d}")
        ev = res["eval"]
        assert np.array_equal(pipe.ev.R(M, N)[u].cpu().numpy(), ev["R"])
        assert pipe.final["maxload"][u].item() == ev["maxload"]
        if u == 0:
            for d in range(M):
                s = res["scheds"][d]
                L = s["send_load"]
                base = np.concatenate([[0], np.cumsum(L)[:-1]]).astype(np.int64)
                start = int(pipe.rail_base[u, d, 0].item())
                want = oracle.pack_node(M, N, d, T, k, RB, C, x[u, d].numpy().view(np.uint8),
                                        topk[u, d].numpy(), lut.numpy(), res["msg"][d], s, base,
                                        int(L.sum()))
                got = pipe.out[start:start + int(L.sum())].cpu().numpy()
                assert np.array_equal(got, want), f"pack d{d}"
