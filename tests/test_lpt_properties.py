"""Properties of LPT that the CUDA fast paths rely on, checked on the oracle's plain
Alg. 2 -- not on the CUDA code (-m "not gpu")."""
import numpy as np

import oracle


def _replay_loads(w, N, order, rail):
    """Loads (per rail) before each assignment, replayed from the oracle schedule."""
    L = np.zeros(N, np.int64)
    before = []
    for i in order:
        before.append(L.copy())
        L[rail[i]] += w[i]
    return before


def test_full_chunks_round_robin_closed_form():
    # a node's full chunks (all size C, larger than every remainder) go to rail
    # i mod N at offset (i div N) * C: k_chunk_sort / eval / pack rely on it
    rng = np.random.default_rng(1)
    for _ in range(200):
        N = int(rng.integers(1, 9))
        C = int(rng.integers(2, 100))
        nf = int(rng.integers(0, 40))
        rem = list(rng.integers(1, C, size=int(rng.integers(0, 30))))
        w = np.array([C] * nf + sorted(rem, reverse=True), np.int64)
        order, rail, off, load = oracle.lpt(w, N)
        for i in range(nf):
            assert rail[i] == i % N and off[i] == (i // N) * C


def test_equal_run_cyclic_when_spread_below_w():
    # once max - min load < w, the next N items of size w go one per rail in
    # (load, rail) order and leave that order unchanged (lpt_group8 fast path)
    rng = np.random.default_rng(2)
    hits = 0
    for _ in range(400):
        N = int(rng.choice([2, 4, 8]))
        big = list(rng.integers(50, 400, size=int(rng.integers(0, 20))))
        wr = int(rng.integers(1, 50))
        r = int(rng.integers(N, 6 * N))
        w = np.array(sorted(big, reverse=True) + [wr] * r, np.int64)
        order, rail, off, load = oracle.lpt(w, N)
        before = _replay_loads(w, N, order, rail)
        start = len(big)
        p = start
        while p + N <= len(w):
            Lb = before[p]
            if Lb.max() - Lb.min() < wr:
                expect = sorted(range(N), key=lambda j: (Lb[j], j))
                got = [int(rail[order[p + t]]) for t in range(N)]
                assert got == expect
                for t in range(N):
                    assert off[order[p + t]] == Lb[expect[t]]
                hits += 1
            p += N
    assert hits > 100


def test_equal_run_merge_when_spread_below_2w():
    # N = 8, 8 equal items, spread < 2w: the picks are the 8 smallest (load, rail)
    # slots among {L_j, L_j + w} (lpt_merge8), checked against plain Alg. 2
    rng = np.random.default_rng(3)
    hits = 0
    for _ in range(1500):
        N = 8
        big = list(rng.integers(60, 500, size=int(rng.integers(0, 25))))
        wr = int(rng.integers(5, 60))
        w = np.array(sorted(big, reverse=True) + [wr] * 8, np.int64)
        order, rail, off, load = oracle.lpt(w, N)
        before = _replay_loads(w, N, order, rail)
        Lb = before[len(big)]
        if not (Lb.max() - Lb.min() < 2 * wr):
            continue
        cand = sorted([(int(Lb[j]), j) for j in range(N)] + [(int(Lb[j]) + wr, j) for j in range(N)])
        picks = cand[:8]
        got = [(int(off[order[len(big) + t]]), int(rail[order[len(big) + t]])) for t in range(8)]
        assert got == picks
        hits += 1
    assert hits > 100
