"""Pins for the NEXT f4 fluid-simulator oracle (oracle/flowsim.c), -m "not gpu".

Checked against things other than the simulator itself: SPEC's worked examples
(S:496-498), textbook max-min allocations, the paper's Theorems 1-2 as
invariants, exact conservation and scale laws of the fluid model
(S:526-530), and the scheduler's own LoadState.
"""
import numpy as np
import pytest

import gen
import oracle

R2 = 100e9 / 8  # 100 Gb/s in bytes/s


def _fab(M, N, S=None):
    S = N if S is None else S
    return dict(S=S, R1=8 * R2, R2=R2, Rs=M * R2 / S)  # S:100-101 defaults


def _sim(M, N, msg, policy, C=1 << 30, S=None):
    f = _fab(M, N, S)
    return oracle.flowsim(M, N, f["S"], f["R1"], f["R2"], f["Rs"], C, policy, msg)


def _link_ids(M, N, S):
    """Directed link layout of DESIGN.md R#35 (region starts)."""
    a = M * N * N
    return dict(gpu_up=0, nic_up=a, leaf_spine=a + M * N, spine_leaf=a + M * N + N * S,
                nic_down=a + M * N + 2 * N * S, gpu_down=a + 2 * M * N + 2 * N * S,
                end=2 * a + 2 * M * N + 2 * N * S)


def _rand_msg(rng, M, N, hi, p=0.7):
    G = M * N
    msg = rng.integers(1, hi, size=(M, N, G)) * (rng.random((M, N, G)) < p)
    for d in range(M):
        msg[d, :, d * N:(d + 1) * N] = 0
    return msg.astype(np.int64)


# ------------------------------------------------------------------ SPEC examples
def test_single_flow_one_rail_5_12_ms():
    # one 64 MB (decimal) flow on one rail, R2 = 100 Gb/s -> 5.12 ms
    msg = np.zeros((2, 1, 2), np.int64)
    msg[0, 0, 1] = 64_000_000
    for pol in oracle.FS_POLICIES:
        r = _sim(2, 1, msg, pol)
        assert r["T"] == pytest.approx(5.12e-3, rel=1e-12)
        assert r["msg_cct"][0, 0, 1] == pytest.approx(5.12e-3, rel=1e-12)


def test_two_flows_share_nic_uplink():
    # two equal flows sharing one NIC uplink run at R2/2 each and both
    # finish at twice the single-flow time
    B = 10_000_000
    msg = np.zeros((3, 1, 3), np.int64)
    msg[0, 0, 1] = msg[0, 0, 2] = B
    r = _sim(3, 1, msg, "lpt")
    assert r["msg_cct"][0, 0, 1] == pytest.approx(2 * B / R2, rel=1e-12)
    assert r["msg_cct"][0, 0, 2] == pytest.approx(2 * B / R2, rel=1e-12)
    assert r["events"] == 1


def test_max_min_spec_and_textbook():
    # S:512-515 and the textbook progressive-filling example
    assert np.allclose(oracle.max_min([[0], [0], [0]], [1, 1, 1], [3.0]), [1, 1, 1])
    assert np.allclose(oracle.max_min([[0, 1], [1]], [1, 1], [1.0, 1.0]), [0.5, 0.5])
    assert np.allclose(oracle.max_min([[0], [1]], [1, 1], [2.0, 5.0]), [2.0, 5.0])
    # links a (cap 1), b (cap 2): f1 on a, f2 on a+b, f3 and f4 on b:
    # a saturates first at 1/2; b's residual 1.5 is shared by f3, f4
    assert np.allclose(oracle.max_min([[0], [0, 1], [1], [1]], [1] * 4, [1.0, 2.0]),
                       [0.5, 0.5, 0.75, 0.75])
    # weighted sub-flows: weights 1/2 + 1/2 of one REPS flow against a weight-1 flow
    assert np.allclose(oracle.max_min([[0], [1], [1]], [0.5, 0.5, 1.0], [1.0, 3.0]),
                       [1.0, 1.0, 2.0])


def test_rail_path_links():
    # g != n and m != n -> 4 links (both intra hops); LPT on empty loads
    # puts the single chunk on rail 0
    M, N = 2, 4
    msg = np.zeros((M, N, M * N), np.int64)
    msg[0, 1, N + 2] = 1_000_000  # (0, g=1) -> (1, m=2)
    r = _sim(M, N, msg, "lpt")
    ids = _link_ids(M, N, N)
    lb = r["link_bytes"]
    want = {ids["gpu_up"] + (0 * N + 1) * N + 0, ids["nic_up"] + 0 * N + 0,
            ids["nic_down"] + 1 * N + 0, ids["gpu_down"] + (1 * N + 0) * N + 2}
    assert set(np.nonzero(lb)[0].tolist()) == want
    assert np.allclose(lb[sorted(want)], 1_000_000, rtol=1e-12)
    # ECMP from NIC 1 to NIC 2 crosses exactly one spine
    r = _sim(M, N, msg, "ecmp")
    nz = np.nonzero(r["link_bytes"])[0]
    assert len(nz) == 4
    assert sum(ids["leaf_spine"] <= i < ids["spine_leaf"] for i in nz) == 1
    assert sum(ids["spine_leaf"] <= i < ids["nic_down"] for i in nz) == 1


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("policy", list(oracle.FS_POLICIES))
def test_conservation_ceiling_and_lower_bound(policy):
    # each flow crosses exactly one NIC_UP and one NIC_DOWN (work conservation,
    # S:527); Theorem 1: the aggregate rate between two domains never
    # exceeds N*R2; Theorem 2: T >= T* for every policy
    rng = np.random.default_rng(7)
    for M, N in [(3, 2), (4, 4), (3, 3)]:
        msg = _rand_msg(rng, M, N, 3_000_000)
        r = _sim(M, N, msg, policy, C=65536)
        ids = _link_ids(M, N, N)
        lb = r["link_bytes"]
        tot = float(msg.sum())
        assert lb[ids["nic_up"]:ids["leaf_spine"]].sum() == pytest.approx(tot, rel=1e-9)
        assert lb[ids["nic_down"]:ids["gpu_down"]].sum() == pytest.approx(tot, rel=1e-9)
        assert r["max_pair_frac"] <= 1 + 1e-9
        row = msg.sum(axis=(1, 2)).max()
        col = msg.reshape(M, N, M, N).sum(axis=(0, 1, 3)).max()
        assert r["T"] >= max(row, col) / (N * R2) * (1 - 1e-9)
        # per-link bytes never exceed capacity * T
        caps = np.empty(ids["end"])
        caps[:] = 8 * R2
        caps[ids["nic_up"]:ids["leaf_spine"]] = R2
        caps[ids["leaf_spine"]:ids["nic_down"]] = M * R2 / N
        caps[ids["nic_down"]:ids["gpu_down"]] = R2
        assert np.all(lb <= caps * r["T"] * (1 + 1e-9))


@pytest.mark.parametrize("policy", list(oracle.FS_POLICIES))
def test_scale_invariance(policy):
    # doubling every flow's bytes doubles every completion time (chunk size
    # doubled too, so the chunking is the same)
    rng = np.random.default_rng(11)
    M, N = 3, 4
    msg = _rand_msg(rng, M, N, 2_000_000)
    a = _sim(M, N, msg, policy, C=65536)
    b = _sim(M, N, 2 * msg, policy, C=2 * 65536)
    assert b["T"] == pytest.approx(2 * a["T"], rel=1e-9)
    assert np.allclose(b["msg_cct"], 2 * a["msg_cct"], rtol=1e-9, atol=0)


def test_lpt_nic_send_volume_equals_loadstate():
    # under rails_lpt the per-NIC send volume is the scheduler's LoadState
    rng = np.random.default_rng(5)
    M, N, C = 4, 4, 65536
    msg = _rand_msg(rng, M, N, 3_000_000)
    r = _sim(M, N, msg, "lpt", C=C)
    ids = _link_ids(M, N, N)
    sent = r["link_bytes"][ids["nic_up"]:ids["leaf_spine"]].reshape(M, N)
    for d in range(M):
        s = oracle.schedule_node(msg[d], C)
        assert np.allclose(sent[d], s["send_load"], rtol=1e-12)


def test_uniform_policy_reaches_lower_bound_on_uniform_load():
    # uniform workload, M = N = 4, continuous P* = 1/N -> within 2% of the
    # LP bound (Theorem 3); here it is exact
    M, N = 4, 4
    msg = gen.d1_uniform(M, N, 16 << 20)
    r = _sim(M, N, msg, "uniform")
    Tstar = msg.sum(axis=(1, 2)).max() / (N * R2)
    assert r["T"] == pytest.approx(Tstar, rel=0.02)


def test_cct_percentiles_nearest_rank():
    # R#39: CCT statistics over messages; nearest rank = ceil(p*n)-th smallest
    rng = np.random.default_rng(3)
    M, N = 3, 2
    msg = _rand_msg(rng, M, N, 5_000_000, p=0.9)
    r = _sim(M, N, msg, "ecmp")
    c = np.sort(r["msg_cct"][msg > 0])
    n = len(c)
    assert r["cct_mean"] == pytest.approx(c.mean(), rel=1e-12)
    for key, p in [("cct_p80", 0.8), ("cct_p95", 0.95), ("cct_p99", 0.99)]:
        assert r[key] == c[int(np.ceil(p * n)) - 1]
    assert r["T"] == c[-1]


def test_receiver_skew_rails_beats_fixed_nic_policies():
    # P:874 direction (receiver-side bottleneck of NIC-bound schemes):
    # RailS spreads receive load over the destination's N NICs through intra-
    # domain forwarding; ECMP/REPS/MinRTT keep the destination GPU's own NIC
    M, N = 4, 4
    msg = gen.d1_receiver_skew(M, N, 8 << 20, 1.2, 99, 0)
    lpt = _sim(M, N, msg, "lpt", C=65536)
    for pol in ("ecmp", "reps", "minrtt"):
        assert _sim(M, N, msg, pol, C=65536)["T"] > 1.5 * lpt["T"]


def test_plb_equals_ecmp_without_spine_congestion():
    # R#36: PLB only repaths flows whose rate a spine link set; with spines far
    # faster than the NICs that never happens and PLB is ECMP, event for event
    rng = np.random.default_rng(21)
    M, N = 4, 4
    msg = _rand_msg(rng, M, N, 3_000_000)
    kw = dict(S=N, R1=8 * R2, R2=R2, Rs=100 * R2)
    e = oracle.flowsim(M, N, kw["S"], kw["R1"], R2, kw["Rs"], 65536, "ecmp", msg)
    p = oracle.flowsim(M, N, kw["S"], kw["R1"], R2, kw["Rs"], 65536, "plb", msg)
    assert np.array_equal(e["msg_cct"], p["msg_cct"])
    assert e["events"] == p["events"]


def test_plb_repaths_under_spine_congestion():
    # oversubscribed spines (Rs = R2/4): ECMP's hashed spine links are the
    # bottlenecks, PLB moves flows off them at completion events -- its spine
    # link loads differ from ECMP's, the bytes conserved and T still >= T*
    rng = np.random.default_rng(22)
    M, N = 4, 4
    msg = _rand_msg(rng, M, N, 3_000_000)
    Rs = R2 / 4
    e = oracle.flowsim(M, N, N, 8 * R2, R2, Rs, 65536, "ecmp", msg)
    p = oracle.flowsim(M, N, N, 8 * R2, R2, Rs, 65536, "plb", msg)
    ids = _link_ids(M, N, N)
    sp = slice(ids["leaf_spine"], ids["nic_down"])
    assert not np.allclose(e["link_bytes"][sp], p["link_bytes"][sp])
    tot = float(msg.sum())
    assert p["link_bytes"][ids["nic_up"]:ids["leaf_spine"]].sum() == pytest.approx(tot, rel=1e-9)
    assert p["T"] >= msg.sum(axis=(1, 2)).max() / (N * R2) * (1 - 1e-9)
