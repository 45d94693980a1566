"""Pins for the CPU oracle (-m "not gpu").

The oracle is checked against things other than itself: worked examples printed
in SPEC.md / derived by hand from the paper's definitions (tests/golden), closed
forms, the paper's theorems as invariants (Thm 2-4), brute force on
tiny inputs, and special cases that reduce to textbook routines.  Each test names
the passage it pins.
"""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle.brute import brute_force_opt, lower_bound

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
R2 = 5.0e10
SEED = oracle.DEFAULT_ECMP_SEED


# ------------------------------------------------------------------ chunking
@pytest.mark.parametrize("ex", GOLD["split_message"])
def test_split_worked_examples(ex):
    ch = oracle.split(np.array([[0, ex["message"]]], np.int64), ex["chunk"])
    assert ch["size"].tolist() == ex["sizes"]
    assert ch["c"].tolist() == list(range(len(ex["sizes"])))


def test_split_conservation_and_count():
    # S:277 / S:329: sum of chunk bytes = B, ceil(B/C) chunks, all but last = C
    rng = np.random.default_rng(1)
    for _ in range(200):
        N, G = rng.integers(1, 5), rng.integers(2, 9)
        C = int(rng.integers(1, 5000))
        msg = rng.integers(0, 20000, size=(N, G)) * (rng.random((N, G)) < 0.7)
        ch = oracle.split(msg, C)
        for g in range(N):
            for h in range(G):
                sel = (ch["g"] == g) & (ch["h"] == h)
                sizes = ch["size"][sel]
                B = int(msg[g, h])
                assert sizes.sum() == B
                assert len(sizes) == -(-B // C)
                if len(sizes):
                    assert (sizes[:-1] == C).all() and 0 < sizes[-1] <= C
        # emission order is (g, h, c) ascending
        key = list(zip(ch["g"].tolist(), ch["h"].tolist(), ch["c"].tolist()))
        assert key == sorted(key)


# ------------------------------------------------------------------ LPT
@pytest.mark.parametrize("ex", GOLD["lpt"])
def test_lpt_worked_examples(ex):
    order, rail, off, load = oracle.lpt(ex["w"], ex["N"])
    if "loads" in ex:
        assert load.tolist() == ex["loads"]
    if "makespan" in ex:
        assert int(load.max()) == ex["makespan"]
    if "opt" in ex:
        assert brute_force_opt(ex["w"], ex["N"])[0] == ex["opt"]
    if "mse" in ex:
        assert oracle.mse(load) == ex["mse"]
    if "makespan" in ex and "opt" in ex:
        # Graham-tight: LPT/OPT = 4/3 - 1/(3N) exactly (P:527 read against OPT, R#15)
        N = ex["N"]
        assert Fraction(ex["makespan"], ex["opt"]) == Fraction(4, 3) - Fraction(1, 3 * N)


def test_lpt_graham_bound_vs_brute_force():
    # P:527 (R#15): 3N * LPT <= (4N - 1) * OPT, exhaustive OPT on tiny inputs
    rng = random.Random(7)
    checked = 0
    for seed in range(200):
        N = rng.choice([2, 3])
        F = rng.randint(1, 12 if N == 2 else 9)
        w = [rng.randint(1, 50) for _ in range(F)]
        _, _, _, load = oracle.lpt(w, N)
        opt, _ = brute_force_opt(w, N)
        mk = int(load.max())
        assert opt <= mk
        assert 3 * N * mk <= (4 * N - 1) * opt
        assert lower_bound(w, N) <= opt
        checked += 1
    assert checked == 200


def test_lpt_theorem4_properties():
    # Thm 4: MSE <= w_max^2; stronger max-min <= w_max (R#16);
    # additive bound L_max <= mean + w_max
    rng = np.random.default_rng(3)
    for _ in range(1000):
        N = int(rng.choice([2, 4, 8, 16]))
        F = int(rng.integers(1, 501))
        w = rng.integers(1, 10 ** 6 + 1, size=F)
        order, rail, off, load = oracle.lpt(w, N)
        wmax = int(w.max())
        assert int(load.max() - load.min()) <= wmax
        assert oracle.mse(load) <= wmax * wmax
        assert N * int(load.max()) <= int(load.sum()) + N * wmax
        assert int(load.sum()) == int(w.sum())
        # LoadState equals per-rail sums of the assignment
        assert np.array_equal(np.bincount(rail, weights=w, minlength=N).astype(np.int64), load)


def test_lpt_sorted_order_and_offsets():
    # Alg. 2 step 2: order = (w desc, index asc); offsets = LoadState
    # before the update (R#19): rail buffers are gap-free and non-overlapping.
    rng = np.random.default_rng(4)
    for _ in range(100):
        N = int(rng.integers(1, 9))
        w = rng.integers(1, 6, size=int(rng.integers(1, 60)))
        order, rail, off, load = oracle.lpt(w, N)
        keys = [(-int(w[i]), int(i)) for i in order]
        assert keys == sorted(keys)
        for j in range(N):
            ids = [i for i in order if rail[i] == j]
            pos = 0
            for i in ids:
                assert off[i] == pos
                pos += int(w[i])
            assert pos == load[j]


def test_lpt_equal_weights_closed_form():
    # c*N equal weights -> every load c*w; flow i -> rail i mod N at i//N * w
    for N in (1, 2, 3, 4, 8):
        for c in range(1, 6):
            w = [7] * (c * N)
            order, rail, off, load = oracle.lpt(w, N)
            assert (load == c * 7).all()
            for i in range(c * N):
                assert rail[i] == i % N and off[i] == (i // N) * 7


def test_lpt_permutation_invariance_distinct_weights():
    # the schedule is a function of the flow set (total tie order)
    rng = np.random.default_rng(5)
    for _ in range(50):
        N = int(rng.integers(2, 9))
        w = rng.choice(10 ** 6, size=40, replace=False) + 1
        _, r1, o1, l1 = oracle.lpt(w, N)
        p = rng.permutation(40)
        _, r2, o2, l2 = oracle.lpt(w[p], N)
        assert np.array_equal(r1[p], r2) and np.array_equal(o1[p], o2)
        assert np.array_equal(l1, l2)


def test_lpt_single_rail():
    w = [5, 9, 1, 9]
    order, rail, off, load = oracle.lpt(w, 1)
    assert (rail == 0).all() and load.tolist() == [24]
    assert sorted(off.tolist()) == [0, 9, 18, 23]


def test_lpt_empty():
    order, rail, off, load = oracle.lpt([], 4)  # empty -> zero loads
    assert load.tolist() == [0, 0, 0, 0] and len(rail) == 0


# ------------------------------------------------------------------ MSE
@pytest.mark.parametrize("ex", GOLD["mse"])
def test_mse_worked(ex):
    assert oracle.mse(ex["loads"]) == ex["mse"]


@pytest.mark.parametrize("ex", GOLD["nmse"])
def test_nmse_worked(ex):
    assert oracle.nmse(ex["loads"]) == ex["nmse"]


def test_mse_matches_eq6_float():
    # Eq. 6 with T_opt = mean (Alg. 2 step 6 P:658-659), evaluated
    # naively in fp64, agrees with the exact-integer oracle form (R#11).
    rng = np.random.default_rng(6)
    for _ in range(300):
        N = int(rng.integers(1, 33))
        L = rng.integers(0, 10 ** 9, size=N)
        mu = L.sum() / N
        naive = float(((L - mu) ** 2).sum() / N)
        got = oracle.mse(L)
        assert got == pytest.approx(naive, rel=1e-9, abs=1e-6)
        # translation covariance
        assert oracle.mse(L + 12345) == got
    assert oracle.nmse([0, 0, 0]) == 0.0


# ------------------------------------------------------------------ eval
def _msg_from_entries(M, N, entries):
    G = M * N
    msg = np.zeros((M, N, G), np.int64)
    for d, g, h, b in entries:
        msg[d, g, h] += b
    return msg


def test_hand_example_M2N2C4():
    ex = GOLD["hand_eval_M2N2C4"]
    M, N, C = ex["M"], ex["N"], ex["C"]
    msg = _msg_from_entries(M, N, ex["messages"])
    scheds, ev = oracle.run_unit_matrix(M, N, C, R2, SEED, msg)
    s0 = scheds[0]
    ch = s0["chunks"]
    got = [[int(ch["g"][i]), int(ch["h"][i]), int(ch["c"][i]), int(ch["size"][i]),
            int(s0["rail"][i]), int(s0["off"][i])] for i in range(len(ch["size"]))]
    assert got == ex["chunks_node0"]
    assert ev["S"].tolist() == ex["S"] and ev["R"].tolist() == ex["R"]
    assert ev["maxload"] == ex["maxload"] and ev["total"] == ex["total"]
    assert ev["rowmax"] == ex["rowmax"] and ev["colmax"] == ex["colmax"]
    assert ev["T"] / ev["T_star"] == pytest.approx(ex["T_over_Tstar_num"] / ex["T_over_Tstar_den"], rel=1e-15)
    assert ev["busbw"] / R2 == pytest.approx(ex["busbw_over_R2"], rel=1e-15)
    assert ev["mse"][0] == ex["mse0"]
    # compact form (R#19): full chunks 0,1,2 -> rails 0,1,0 (closed form)
    assert s0["full_base"][0, 2] == 0 and s0["full_base"][1, 3] == 2 and s0["n_full"] == 3
    assert s0["rem_rail"][0, 2] == 1 and s0["rem_off"][0, 2] == 4
    assert s0["rem_rail"][1, 3] == 1 and s0["rem_off"][1, 3] == 6 and s0["n_rem"] == 2


@pytest.mark.parametrize("ex", GOLD["lp_lower_bound"])
def test_lp_lower_bound_worked(ex):
    # S:396-397; T* = max(max row sum, max col sum of D2) / (N R2) (Thm 2 + 3)
    d2 = ex["d2"]
    M = len(d2)
    N = ex["N"]
    entries = [(k, 0, f * N, d2[k][f]) for k in range(M) for f in range(M) if d2[k][f]]
    msg = _msg_from_entries(M, N, entries)
    _, ev = oracle.run_unit_matrix(M, N, 4, ex["R2"], SEED, msg)
    assert ev["T_star"] == ex["T_star"]


@pytest.mark.parametrize("ex", GOLD["aggregate"])
def test_aggregate_worked(ex):
    # Eq. 1: D2[d,f] = sum_n sum_m D1 -> row/col sums feed T*
    msg = _msg_from_entries(ex["M"], ex["N"], [(0, g, h, b) for (_, g, h, b) in ex["entries"]])
    _, ev = oracle.run_unit_matrix(ex["M"], ex["N"], 1 << 20, 1.0, SEED, msg)
    assert ev["rowmax"] == ex["d2_01"] and ev["colmax"] == ex["d2_01"]


def _random_msg(rng, M, N, p=0.6, hi=200000, mult=1):
    G = M * N
    msg = (rng.integers(1, hi, size=(M, N, G)) * mult) * (rng.random((M, N, G)) < p)
    for d in range(M):
        msg[d, :, d * N:(d + 1) * N] = 0  # intra-node traffic is not inter-domain (R#2)
    return msg.astype(np.int64)


def test_theorem3_uniform_split_symmetry():
    # Thm 3: with P* = 1/N, N*S[k][n] = row sum k and N*R[f][n] = col
    # sum f exactly; the oracle's eval accepts any per-chunk assignment.
    rng = np.random.default_rng(8)
    for _ in range(100):
        M, N = int(rng.integers(2, 17)), int(rng.integers(1, 17))
        G = M * N
        msg = _random_msg(rng, M, N, p=0.3, hi=1000, mult=N)
        cd, ch, cs, cr = [], [], [], []
        for d in range(M):
            for g in range(N):
                for h in range(G):
                    if msg[d, g, h]:
                        for n in range(N):
                            cd.append(d); ch.append(h); cs.append(msg[d, g, h] // N); cr.append(n)
        ev = oracle.eval_unit(M, N, R2, SEED, msg, cd, ch, cs, cr)
        D2 = msg.reshape(M, N, M, N).sum(axis=(1, 3))
        rows, cols = D2.sum(axis=1), D2.sum(axis=0)
        assert (ev["S"] * N == rows[:, None]).all()
        assert (ev["R"] * N == cols[:, None]).all()
        assert ev["T"] == pytest.approx(ev["T_star"], rel=1e-15)


def test_T_ge_Tstar_every_assignment():
    # Thm 2: T >= T* for every allocation (LPT, ECMP, random)
    rng = np.random.default_rng(9)
    for _ in range(60):
        M, N = int(rng.integers(2, 7)), int(rng.integers(1, 9))
        C = int(rng.integers(1, 50000))
        msg = _random_msg(rng, M, N)
        scheds, ev = oracle.run_unit_matrix(M, N, C, R2, SEED, msg)
        assert ev["T"] >= ev["T_star"] * (1 - 1e-15)
        assert ev["T_e"] >= ev["T_star"] * (1 - 1e-15)
        cd, ch, cs = [], [], []
        for d, s in enumerate(scheds):
            cd += [d] * len(s["chunks"]["size"]); ch += s["chunks"]["h"].tolist()
            cs += s["chunks"]["size"].tolist()
        cr = rng.integers(0, N, size=len(cs))
        ev_r = oracle.eval_unit(M, N, R2, SEED, msg, cd, ch, cs, cr)
        assert ev_r["T"] >= ev_r["T_star"] * (1 - 1e-15)


def test_lpt_multiple_of_NC_reaches_Tstar():
    # [derived, R#17] every message a multiple of N*C -> LPT loads uniform, T = T*
    rng = np.random.default_rng(10)
    for _ in range(30):
        M, N = int(rng.integers(2, 6)), int(rng.integers(1, 9))
        C = int(rng.integers(1, 64)) * 16
        msg = _random_msg(rng, M, N, hi=5, mult=N * C)
        _, ev = oracle.run_unit_matrix(M, N, C, R2, SEED, msg)
        assert (ev["S"] == ev["S"][:, :1]).all() and (ev["R"] == ev["R"][:, :1]).all()
        assert ev["T"] == pytest.approx(ev["T_star"], rel=1e-15)
    # N = 1: T = T* always
    msg = _random_msg(rng, 3, 1)
    _, ev = oracle.run_unit_matrix(3, 1, 1000, R2, SEED, msg)
    assert ev["T"] == pytest.approx(ev["T_star"], rel=1e-15) and ev["T_e"] == ev["T"]


def test_eval_conservation():
    # sum S = sum R = total inter-node bytes; row sums; send_load = S
    rng = np.random.default_rng(11)
    for _ in range(40):
        M, N = int(rng.integers(2, 7)), int(rng.integers(1, 9))
        msg = _random_msg(rng, M, N)
        scheds, ev = oracle.run_unit_matrix(M, N, int(rng.integers(1, 70000)), R2, SEED, msg)
        tot = int(msg.sum())
        assert ev["S"].sum() == tot == ev["R"].sum() == ev["total"]
        assert ev["S_e"].sum() == tot == ev["R_e"].sum() == ev["total_e"]
        assert (ev["S"].sum(axis=1) == msg.sum(axis=(1, 2))).all()
        for d in range(M):
            assert np.array_equal(scheds[d]["send_load"], ev["S"][d])
        if tot:
            assert ev["busbw"] == pytest.approx(tot / ev["T"], rel=1e-15)
            # policy against itself: normalized busbw exactly 1
            assert ev["busbw"] / ev["busbw"] == 1.0


def test_mse_bound_per_node_in_unit():
    # Thm 4 per node of a unit: MSE <= w_max^2 with w_max = the largest chunk
    rng = np.random.default_rng(12)
    for _ in range(30):
        M, N = 4, int(rng.integers(2, 9))
        C = int(rng.integers(100, 50000))
        msg = _random_msg(rng, M, N)
        scheds, ev = oracle.run_unit_matrix(M, N, C, R2, SEED, msg)
        for d in range(M):
            sz = scheds[d]["chunks"]["size"]
            if len(sz):
                assert ev["mse"][d] <= float(sz.max()) ** 2


# ------------------------------------------------------------------ ECMP hash
@pytest.mark.parametrize("ex", GOLD["splitmix64"])
def test_splitmix64_textbook(ex):
    assert oracle.mix64(ex["z"]) == int(ex["out"], 16)


def test_ecmp_rail_pins():
    # R#14 is this build's choice ("parity unpinned" beyond these hand-computed values)
    pins = {(0, 8): 4, (0, 9): 7, (1, 8): 5, (7, 1023): 6, (1000, 5): 7, (2047, 0): 1}
    for (s, d), r in pins.items():
        assert oracle.ecmp_rail(SEED, s, d, 8) == r
    # cross-check the formula with an independent pure-Python splitmix64
    def mix(z):
        m = (1 << 64) - 1
        z = (z + 0x9E3779B97F4A7C15) & m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)
    rng = random.Random(13)
    for _ in range(200):
        s, d, N = rng.randrange(4096), rng.randrange(4096), rng.randint(1, 32)
        assert oracle.ecmp_rail(SEED, s, d, N) == (mix(((s << 32) | d) ^ SEED) >> 32) % N


# ------------------------------------------------------------------ histogram
def test_histogram_brute_force_rank():
    # P:193 (D^(1)) and R#18: rank = position among earlier (t,s) with same dest
    rng = np.random.default_rng(14)
    for _ in range(20):
        M, N, T, k, E = int(rng.integers(2, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 40)), \
            int(rng.integers(1, 4)), int(rng.integers(1, 6))
        lut = rng.integers(0, M * N, size=M * E).astype(np.int32)
        topk = rng.integers(0, M * E, size=(N, T, k)).astype(np.int32)
        d = int(rng.integers(0, M))
        RB = 48
        counts, msg, rank = oracle.histogram_node(M, N, d, T, k, topk, lut, RB)
        seen = {}
        for g in range(N):
            for t in range(T):
                for s in range(k):
                    h = int(lut[topk[g, t, s]])
                    assert rank[g, t, s] == seen.get((g, h), 0)
                    seen[(g, h)] = seen.get((g, h), 0) + 1
        for g in range(N):
            assert counts[g].sum() == T * k
            for h in range(M * N):
                assert counts[g, h] == seen.get((g, h), 0)
                assert msg[g, h] == (0 if h // N == d else counts[g, h] * RB)


def test_histogram_range_error():
    lut = np.array([0, 1, 99], np.int32)
    topk = np.zeros((1, 2, 1), np.int32)
    topk[0, 1, 0] = 2
    with pytest.raises(ValueError):
        oracle.histogram_node(2, 1, 0, 2, 1, topk, lut, 16)


# ------------------------------------------------------------------ pack
def _streams_from_x(M, N, d, T, k, RB, x, topk, lut):
    """Independent restatement of R#18: message (g,h) = rows of remote (t,s) in order."""
    G = M * N
    st = {}
    for g in range(N):
        for t in range(T):
            for s in range(k):
                h = int(lut[topk[g, t, s]])
                if h // N == d:
                    continue
                st.setdefault((g, h), []).append(x[g, t].tobytes())
    return {key: b"".join(v) for key, v in st.items()}


def test_pack_unpack_roundtrip():
    # a7 by definition: unpack(pack(x)) rebuilds every (g,h) message stream byte
    # for byte; rail j length = S[d][j]; every remote (t,s) copy appears once.
    rng = np.random.default_rng(15)
    for trial in range(6):
        M, N, T, k, E = 3, int(rng.integers(1, 5)), int(rng.integers(5, 60)), 2, 4
        RB = 32 * int(rng.integers(1, 4))
        C = 16 * int(rng.integers(1, 9))
        lut = (np.arange(M * E) // E * N + (np.arange(M * E) % E) % N).astype(np.int32)
        d = trial % M
        topk = rng.integers(0, M * E, size=(N, T, k)).astype(np.int32)
        x = rng.integers(0, 256, size=(N, T, RB)).astype(np.uint8)
        counts, msg, rank = oracle.histogram_node(M, N, d, T, k, topk, lut, RB)
        sched = oracle.schedule_node(msg, C)
        load = sched["send_load"]
        base = np.concatenate([[0], np.cumsum(load)[:-1]]).astype(np.int64)
        out = oracle.pack_node(M, N, d, T, k, RB, C, x, topk, lut, msg, sched, base, int(load.sum()))
        streams = _streams_from_x(M, N, d, T, k, RB, x, topk, lut)
        ch = sched["chunks"]
        rebuilt = {}
        for i in range(len(ch["size"])):
            key = (int(ch["g"][i]), int(ch["h"][i]))
            a = int(base[sched["rail"][i]] + sched["off"][i])
            rebuilt.setdefault(key, {})[int(ch["c"][i])] = out[a:a + int(ch["size"][i])].tobytes()
        assert set(rebuilt) == set(streams)
        for key, parts in rebuilt.items():
            assert b"".join(parts[c] for c in sorted(parts)) == streams[key]
        assert sum(len(v) for v in streams.values()) == int(load.sum()) == int(msg.sum())


# ------------------------------------------------------------------ NEXT f2: QP map
@pytest.mark.parametrize("ex", GOLD["qp_map"])
def test_qp_map_worked_examples(ex):
    # Alg. 2 step 4, SPEC S:304-312 examples and a hand-derived case
    order, rail, off, load = oracle.lpt(np.array(ex["sizes"], np.int64), ex["N"])
    qp = oracle.qp_map(order, rail, ex["N"], ex["qps_per_rail"])
    assert [int(qp[i]) for i in order] == ex["qp_in_assignment_order"]


def test_qp_map_matches_rail_offset_order():
    # independent of the visiting order: on one rail, offsets grow with assignment
    # order (sizes > 0), so the k-th chunk of rail j by OFFSET has QP k mod Q;
    # full chunk i (emission order) is the floor(i/N)-th chunk of rail i mod N
    rng = np.random.default_rng(34)
    for _ in range(60):
        N = int(rng.integers(1, 9))
        M = int(rng.integers(2, 5))
        C = int(rng.choice([64, 100, 4096]))
        Q = int(rng.choice([1, 2, 3, 64]))
        msg = rng.integers(0, 5 * C, size=(N, M * N)) * (rng.random((N, M * N)) < 0.8)
        msg[:, :N] = 0
        s = oracle.schedule_node(msg.astype(np.int64), C)
        qp = oracle.qp_map(s["order"], s["rail"], N, Q)
        for j in range(N):
            on_j = np.nonzero(s["rail"] == j)[0]
            by_off = on_j[np.argsort(s["off"][on_j], kind="stable")]
            assert np.all(np.diff(s["off"][by_off]) > 0)
            assert [int(qp[i]) for i in by_off] == [k % Q for k in range(len(by_off))]
        full = np.nonzero(s["chunks"]["size"] == C)[0]
        for i_em, i in enumerate(full):  # chunks are in emission order
            assert s["rail"][i] == i_em % N and qp[i] == (i_em // N) % Q


def test_qp_map_rejects_zero_qps():
    order, rail, off, load = oracle.lpt(np.array([3, 2], np.int64), 1)
    with pytest.raises(ValueError):
        oracle.qp_map(order, rail, 1, 0)


# ------------------------------------------------------------------ uniform policy (f3)
@pytest.mark.parametrize("ex", GOLD["uniform_hand"])
def test_uniform_hand_examples(ex):
    M, N = ex["M"], ex["N"]
    msg = _msg_from_entries(M, N, ex["messages"])
    u = oracle.eval_uniform(M, N, R2, msg)
    assert u["S_u"].tolist() == ex["S_u"] and u["R_u"].tolist() == ex["R_u"]
    assert u["maxload_u"] == ex["maxload_u"]
    assert u["T_u"] * R2 == pytest.approx(ex["maxload_u"], rel=1e-15)


def test_uniform_theorem3_and_bounds():
    # Thm 3: with every message a multiple of N, N*S_u[k][n] = row sum k
    # and N*R_u[f][n] = col sum f exactly, so T_u = T*; in general T_u >= T* (Thm 2),
    # bytes are conserved and a rail differs from the mean by < one byte per message
    rng = np.random.default_rng(16)
    for trial in range(120):
        M, N = int(rng.integers(2, 9)), int(rng.integers(1, 9))
        div = trial % 2 == 0
        msg = _random_msg(rng, M, N, p=0.4, hi=10000, mult=N if div else 1)
        _, ev = oracle.run_unit_matrix(M, N, 4096, R2, SEED, msg)
        u = oracle.eval_uniform(M, N, R2, msg)
        D2 = msg.reshape(M, N, M, N).sum(axis=(1, 3))
        rows, cols = D2.sum(axis=1), D2.sum(axis=0)
        assert (u["S_u"].sum(axis=1) == rows).all() and (u["R_u"].sum(axis=1) == cols).all()
        assert u["T_u"] >= ev["T_star"] * (1 - 1e-15)
        nmsg = (msg > 0).reshape(M, -1).sum(axis=1)
        assert (np.abs(N * u["S_u"] - rows[:, None]) <= N * nmsg[:, None]).all()
        if div:
            assert (u["S_u"] * N == rows[:, None]).all() and (u["R_u"] * N == cols[:, None]).all()
            assert u["T_u"] == pytest.approx(ev["T_star"], rel=1e-15)
        if ev["total"]:
            assert u["busbw_u"] == pytest.approx(ev["total"] / u["T_u"], rel=1e-15)
