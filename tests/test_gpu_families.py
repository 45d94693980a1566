"""NEXT f3 -- the paper's workload families through schedule + eval (-m gpu), against
the oracle element by element: Table 1 uniform, sparse Top-K with
K = 2 and sparsity s in {0, 0.2, 0.6} (R#33), sender-skewed and
receiver-skewed Zipf (s = 1.2, R#23), with the LPT schedule, the ECMP-hash baseline
(R#13) and Theorem 3's uniform split P* = 1/N (R#41) as first-class
outputs.  Two launch regimes: few segments (the fused per-node kernel) and many
(per-phase kernels + the evaluation kernel)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from helpers import compare_schedule, oracle_eval_from_scheds, rel_err

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2510_19262_b200.pipeline import MatrixPipeline

DEV = "cuda:0"
FAMILIES = {
    "uniform": dict(skew="uniform"),
    "sparse-0": dict(skew="sparse", sparsity=0.0, K=2),
    "sparse-0.2": dict(skew="sparse", sparsity=0.2, K=2),
    "sparse-0.6": dict(skew="sparse", sparsity=0.6, K=2),
    "sender-skewed": dict(skew="sender", zipf_s=1.2),
    "receiver-skewed": dict(skew="receiver", zipf_s=1.2),
}


@pytest.mark.parametrize("family", list(FAMILIES))
@pytest.mark.parametrize("M,N,C,V,U", [
    (16, 8, 32 << 10, 16 << 20, 2),     # 32 segments: fused per-node kernel
    (8, 8, 1 << 20, 64 << 20, 40),      # 320 segments: per-phase kernels + eval kernel
    (10, 4, 100_000, 8 << 20, 2),       # N = 4, C not a power of two
])
def test_family_schedule_eval_parity(family, M, N, C, V, U):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = dict(M=M, N=N, V=V, zipf_s=1.2)
    cfg.update(FAMILIES[family])
    msg = gen.d1_units(cfg, gen.config_seed(6), 0, U)
    pipe = MatrixPipeline(M, N, C, U, 0, M, DEV)
    pipe.step(torch.from_numpy(msg).to(DEV))
    torch.cuda.synchronize()
    units = range(U) if U <= 2 else [0, U // 2, U - 1]
    for u in units:
        scheds = [oracle.schedule_node(msg[u, d], C) for d in range(M)]
        for d in range(M):
            compare_schedule(pipe.sched, u, d, scheds[d], f"{family} u{u} d{d}")
        ev = oracle_eval_from_scheds(M, N, msg[u], scheds)
        e = pipe.ev
        assert np.array_equal(e.S[u].cpu().numpy(), ev["S"])
        assert np.array_equal(e.S_e[u].cpu().numpy(), ev["S_e"])
        assert np.array_equal(e.S_u[u].cpu().numpy(), ev["S_u"])
        assert np.array_equal(e.R(M, N)[u].cpu().numpy(), ev["R"])
        assert np.array_equal(e.R_e(M, N)[u].cpu().numpy(), ev["R_e"])
        assert np.array_equal(e.R_u(M, N)[u].cpu().numpy(), ev["R_u"])
        f = {k: v[u].item() for k, v in pipe.final.items()}
        for k in ("maxload", "maxload_e", "maxload_u", "total", "rowmax", "colmax"):
            assert f[k] == ev[k], (family, k)
        for k in ("T", "T_e", "T_u", "T_star", "busbw", "busbw_e", "busbw_u"):
            assert rel_err(f[k], ev[k]) <= 1e-6, (family, k)
        for dl in range(M):
            assert rel_err(e.nmse[u, dl].item(), ev["nmse"][dl]) <= 1e-6
        # Theorem 2 on every policy; Theorem 3: uniform attains T* when N divides
        # every message (the uniform and sparse families split V evenly)
        assert f["T"] >= f["T_star"] * (1 - 1e-12) and f["T_e"] >= f["T_star"] * (1 - 1e-12)
        assert f["T_u"] >= f["T_star"] * (1 - 1e-12)
        if (msg[u] % N == 0).all():
            assert rel_err(f["T_u"], f["T_star"]) <= 1e-12
