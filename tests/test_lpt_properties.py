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


def _keyspread_below(Lb, x):
    """max (load, rail) < min (load, rail) + (x, 0): the CUDA key test K[N-1] - K[0] < x << 5."""
    S = sorted((int(Lb[j]), j) for j in range(len(Lb)))
    return S[-1] < (S[0][0] + x, S[0][1])


def test_equal_run_cyclic_when_spread_below_w():
    # once the largest (load, rail) key is below the smallest key plus w, the next
    # N items of size w go one per rail in (load, rail) order and leave that order
    # unchanged (lpt_group8_v fast path)
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
            if _keyspread_below(Lb, wr):
                expect = sorted(range(N), key=lambda j: (Lb[j], j))
                got = [int(rail[order[p + t]]) for t in range(N)]
                assert got == expect
                for t in range(N):
                    assert off[order[p + t]] == Lb[expect[t]]
                hits += 1
            p += N
    assert hits > 100


def test_equal_run_cyclic_whole_run_closed_form():
    # lpt_run_cyclic: from the first item of an equal run at which the key test
    # holds, item t of the rest of the run goes to the (t mod N)-th rail in
    # (load, rail) order at that rail's load + (t div N) * w -- for the whole run
    rng = np.random.default_rng(4)
    hits = 0
    for _ in range(300):
        N = int(rng.choice([2, 4, 8, 16]))
        big = list(rng.integers(50, 400, size=int(rng.integers(0, 30))))
        wr = int(rng.integers(1, 50))
        r = int(rng.integers(1, 12 * N))
        small = list(rng.integers(1, wr + 1, size=int(rng.integers(0, 10))))
        w = np.array(sorted(big, reverse=True) + [wr] * r + sorted(small, reverse=True),
                     np.int64)
        order, rail, off, load = oracle.lpt(w, N)
        before = _replay_loads(w, N, order, rail)
        end = len(big) + r
        while end < len(w) and w[order[end]] == wr:  # equal smalls extend the run
            end += 1
        p = len(big)
        while p < end and not _keyspread_below(before[p], wr):
            p += 1
        if p == end:
            continue
        Lb = before[p]
        S = sorted(range(N), key=lambda j: (Lb[j], j))
        for t in range(end - p):
            i = order[p + t]
            assert rail[i] == S[t % N]
            assert off[i] == Lb[S[t % N]] + (t // N) * wr
        hits += 1
    assert hits > 150


def test_equal_run_merge_when_spread_below_2w():
    # N = 8, 8 equal items, key spread < 2w: the picks are the 8 smallest (load, rail)
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
        if not _keyspread_below(Lb, 2 * wr):
            continue
        cand = sorted([(int(Lb[j]), j) for j in range(N)] + [(int(Lb[j]) + wr, j) for j in range(N)])
        picks = cand[:8]
        got = [(int(off[order[len(big) + t]]), int(rail[order[len(big) + t]])) for t in range(8)]
        assert got == picks
        hits += 1
    assert hits > 100
