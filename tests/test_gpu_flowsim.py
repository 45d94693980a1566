"""NEXT f4 fluid simulator: rails_flowsim (one CTA per simulation) vs the CPU
oracle oracle/flowsim.c on the same seeded rounds (-m gpu).

Message completion times, link bytes and the statistics are floating point over
long event sequences whose order of summation differs (warp trees vs sequential
loops): compared within 1e-6 relative (BASELINE.json's float tolerance); flow
counts are exact.  Every policy runs in the same batched launch."""
import numpy as np
import pytest
import torch

import gen
import oracle

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2510_19262_b200 import rails

DEV = "cuda:0"
R2 = 100e9 / 8
TOL = 1e-6
POLS = ["lpt", "uniform", "ecmp", "reps", "minrtt", "plb"]


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    rails.check()


def _rand(rng, M, N, hi, p=0.7):
    G = M * N
    msg = rng.integers(1, hi, size=(M, N, G)) * (rng.random((M, N, G)) < p)
    for d in range(M):
        msg[d, :, d * N:(d + 1) * N] = 0
    return msg.astype(np.int64)


def _workload(kind, M, N, seed):
    rng = np.random.default_rng(seed)
    if kind == "rand":
        return _rand(rng, M, N, 3_000_000)
    if kind == "uniform":
        return gen.d1_uniform(M, N, 8 << 20)
    if kind == "recv":
        return gen.d1_receiver_skew(M, N, 8 << 20, 1.2, seed, 0)
    if kind == "sender":
        return gen.d1_sender_skew(M, N, 4 << 20, 1.2, seed, 0)
    return gen.d1_sparse_topk(M, N, 8 << 20, 0.5, 2, seed, 0)


def _close(a, b, what):
    a = np.atleast_1d(np.asarray(a, np.float64))
    b = np.atleast_1d(np.asarray(b, np.float64))
    err = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
    err[(a == 0) & (b == 0)] = 0
    assert err.max(initial=0) <= TOL, f"{what}: max rel err {err.max():g}"


@pytest.mark.parametrize("M,N,S,C,kind,rs", [
    (3, 2, 2, 65536, "rand", None),
    (4, 4, 4, 65536, "rand", None),
    (4, 4, 4, 65536, "rand", 0.25),      # oversubscribed spines: PLB repaths
    (4, 4, 4, 1 << 20, "uniform", None),
    (4, 4, 2, 262144, "recv", None),     # fewer spines than rails
    (5, 3, 3, 131072, "sender", 0.5),    # N not a power of two
    (6, 4, 4, 1 << 20, "sparse", None),
])
def test_flowsim_parity(M, N, S, C, kind, rs):
    msg = _workload(kind, M, N, M * 10 + N)
    tp = rails.topo(M, N, C, R2=R2)
    fb = rails.fabric(M, N, R2, S=S, Rs=None if rs is None else rs * R2)
    pol = torch.tensor([rails.FS_POLICIES[p] for p in POLS], dtype=torch.int32, device=DEV)
    msgs = torch.from_numpy(np.stack([msg] * len(POLS))).to(DEV)
    cct, lb, st = rails.flowsim(tp, fb, pol, msgs)
    cct, lb, st = cct.cpu().numpy(), lb.cpu().numpy(), st.cpu().numpy()
    for i, p in enumerate(POLS):
        o = oracle.flowsim(M, N, S, fb.R1, R2, fb.Rs, C, p, msg)
        _close(cct[i], o["msg_cct"], f"{p} msg_cct")
        scale = max(float(o["link_bytes"].max()), 1.0)
        assert np.abs(lb[i] - o["link_bytes"]).max() <= TOL * scale, f"{p} link_bytes"
        for j, k in enumerate(rails.FS_STATS):
            if k == "flows":
                assert st[i, j] == o[k], p
            elif k == "events":
                assert abs(st[i, j] - o[k]) <= max(2, 0.01 * o[k]), f"{p} events"
            else:
                _close(st[i, j], o[k], f"{p} {k}")


def test_flowsim_spec_single_flow():
    # 64 MB on one rail at 100 Gb/s -> 5.12 ms, every policy
    M, N = 2, 1
    msg = np.zeros((M, N, M * N), np.int64)
    msg[0, 0, 1] = 64_000_000
    tp = rails.topo(M, N, 1 << 30, R2=R2)
    fb = rails.fabric(M, N, R2)
    pol = torch.arange(6, dtype=torch.int32, device=DEV)
    cct, lb, st = rails.flowsim(tp, fb, pol, torch.from_numpy(np.stack([msg] * 6)).to(DEV))
    assert np.allclose(st[:, 0].cpu().numpy(), 5.12e-3, rtol=1e-12)


def test_flowsim_batch_independent():
    # a simulation's result does not depend on its batch neighbours
    M, N, S, C = 4, 4, 4, 65536
    a = _workload("rand", M, N, 1)
    b = _workload("recv", M, N, 2)
    tp = rails.topo(M, N, C, R2=R2)
    fb = rails.fabric(M, N, R2, S=S)
    pol = torch.tensor([0, 3, 4], dtype=torch.int32, device=DEV)
    one = rails.flowsim(tp, fb, pol, torch.from_numpy(np.stack([a, a, a])).to(DEV))[2]
    mix = rails.flowsim(tp, fb, pol.repeat(2), torch.from_numpy(
        np.stack([b, b, b, a, a, a])).to(DEV))[2]
    assert torch.equal(one, mix[3:])  # deterministic, bit for bit


def test_flowsim_bad_policy_flagged():
    M, N = 2, 1
    msg = np.zeros((1, M, N, M * N), np.int64)
    msg[0, 0, 0, 1] = 1000
    tp = rails.topo(M, N, 4096, R2=R2)
    fb = rails.fabric(M, N, R2)
    pol = torch.tensor([9], dtype=torch.int32, device=DEV)
    rails.flowsim(tp, fb, pol, torch.from_numpy(msg).to(DEV))
    with pytest.raises(rails.RailsError) as ei:
        rails.check()
    assert ei.value.code == rails.RAILS_ERANGE


def test_flowsim_global_link_state_path(monkeypatch):
    # fabrics too large for shared memory keep the link state in global memory
    # (k_fs_sim<true>); forced here on a small case, same results as the oracle
    monkeypatch.setenv("RAILS_FS_GLOBAL", "1")
    M, N, S, C = 4, 4, 4, 65536
    msg = _workload("recv", M, N, 5)
    tp = rails.topo(M, N, C, R2=R2)
    fb = rails.fabric(M, N, R2, S=S, Rs=0.5 * R2)
    pol = torch.tensor([rails.FS_POLICIES[p] for p in POLS], dtype=torch.int32, device=DEV)
    cct, lb, st = rails.flowsim(tp, fb, pol, torch.from_numpy(np.stack([msg] * len(POLS))).to(DEV))
    cct = cct.cpu().numpy()
    for i, p in enumerate(POLS):
        o = oracle.flowsim(M, N, S, fb.R1, R2, fb.Rs, C, p, msg)
        _close(cct[i], o["msg_cct"], f"{p} msg_cct (global link state)")


@pytest.mark.parametrize("seed", range(12))
def test_flowsim_fuzz(seed):
    # random fabrics (spines, oversubscription), chunk sizes and traffic; every
    # policy in one batch against the oracle
    rng = np.random.default_rng(3000 + seed)
    M = int(rng.integers(2, 6))
    N = int(rng.choice([1, 2, 3, 4]))
    S = int(rng.integers(1, 5))
    C = int(rng.choice([4096, 65536, 300000, 1 << 20]))
    rs = float(rng.choice([0.25, 0.5, 1.0, 4.0]))
    msg = _rand(rng, M, N, int(rng.choice([20000, 2_000_000])), p=float(rng.uniform(0.2, 1.0)))
    tp = rails.topo(M, N, C, R2=R2)
    fb = rails.fabric(M, N, R2, S=S, Rs=rs * R2)
    pol = torch.tensor([rails.FS_POLICIES[p] for p in POLS], dtype=torch.int32, device=DEV)
    cct, lb, st = rails.flowsim(tp, fb, pol, torch.from_numpy(np.stack([msg] * len(POLS))).to(DEV))
    cct, st = cct.cpu().numpy(), st.cpu().numpy()
    for i, p in enumerate(POLS):
        o = oracle.flowsim(M, N, S, fb.R1, R2, fb.Rs, C, p, msg)
        _close(cct[i], o["msg_cct"], f"seed{seed} {p} msg_cct")
        _close(st[i, 0], o["T"], f"seed{seed} {p} T")
