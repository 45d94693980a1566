"""NEXT f2 QP map (Alg. 2 step 4, R#34): rails_lpt_schedule_qp vs the
oracle's per-rail round-robin over the plain Alg. 2 assignment order (-m gpu)."""
import numpy as np
import pytest
import torch

import oracle
from helpers import compare_schedule, random_msg

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2510_19262_b200 import rails

DEV = "cuda:0"


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    rails.check()


@pytest.mark.parametrize("M,N,C,U,Q,kind", [
    (4, 4, 65536, 2, 2, "rand"),
    (5, 3, 1000, 1, 3, "rand"),         # N = 3: warp argmin chain
    (16, 8, 1 << 20, 1, 64, "rand"),    # 64 QPs (the abstract's configuration)
    (6, 8, 16, 1, 256, "rand"),         # tiny chunks: many full chunks per rail
    (3, 2, 1, 1, 7, "rand"),            # C = 1: no remainders
    (64, 8, 32768, 1, 4, "rows"),       # C3-like runs (warp-parallel run path)
    (40, 8, 32768, 32, 3, "rows"),      # 1280 chains: thread-per-chain kernel
    (5, 16, 65536, 1, 5, "rand"),       # N = 16
    (2, 1, 4096, 2, 2, "rand"),         # N = 1
    (4, 4, 4096, 1, 1, "rand"),         # one QP per rail: all 0
])
def test_qp_map_parity(M, N, C, U, Q, kind):
    rng = np.random.default_rng(M * 31 + N * 7 + Q)
    if kind == "rand":
        msg = random_msg(rng, U, M, N, p=0.8, hi=6 * C + 7)
    else:
        G = M * N
        msg = rng.integers(0, 40, size=(U, M, N, G)).astype(np.int64) * 12288
        for d in range(M):
            msg[:, d, :, d * N:(d + 1) * N] = 0
    tp = rails.topo(M, N, C)
    sh = rails.shard(U, 0, M)
    s, qp = rails.lpt_schedule_qp(tp, sh, torch.from_numpy(msg).to(DEV), Q)
    qp = qp.cpu().numpy()
    for u in range(U):
        for d in range(M):
            o = oracle.schedule_node(msg[u, d], C)
            compare_schedule(s, u, d, o, f"u{u} d{d}")
            want, _ = oracle.rem_qp_node(msg[u, d], C, Q, sched=o)
            assert np.array_equal(qp[u, d], want), f"u{u} d{d}"


def test_qp_map_rejects_bad_args():
    tp = rails.topo(2, 2, 64)
    sh = rails.shard(1, 0, 2)
    msg = torch.zeros((1, 2, 2, 4), dtype=torch.int64, device=DEV)
    with pytest.raises(rails.RailsError) as ei:
        rails.lpt_schedule_qp(tp, sh, msg, 0)
    assert ei.value.code == rails.RAILS_EINVAL
