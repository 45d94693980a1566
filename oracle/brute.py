"""Exhaustive optimum for tiny atomic-flow instances -- TEST INFRASTRUCTURE ONLY.

The combinatorial program of PAPER.md section 4.6: assign every flow
to exactly one of N NICs; OPT makespan = min over all N^F assignments of
max_j L_j.  Guarded by N^F <= 1e7.  Pure Python on purpose:
it shares nothing with oracle.c or the CUDA path.
"""
from __future__ import annotations

import itertools


def brute_force_opt(weights, N):
    """Return (min makespan, min MSE-numerator) over all assignments.

    The MSE numerator is sum_j (N*L_j - sum w)^2 (exact integer); MSE = that / N^3.
    """
    F = len(weights)
    if N ** F > 10 ** 7:
        raise ValueError("instance too large for brute force")
    total = sum(weights)
    best_mk = None
    best_sq = None
    for assign in itertools.product(range(N), repeat=F):
        L = [0] * N
        for w, j in zip(weights, assign):
            L[j] += w
        mk = max(L)
        sq = sum((N * l - total) ** 2 for l in L)
        if best_mk is None or mk < best_mk:
            best_mk = mk
        if best_sq is None or sq < best_sq:
            best_sq = sq
    return best_mk, best_sq


def lower_bound(weights, N):
    """LB <= OPT: max(ceil(sum/N), w_max, w_(N) + w_(N+1)) (pigeonhole)."""
    ws = sorted(weights, reverse=True)
    lb = max(-(-sum(ws) // N), ws[0] if ws else 0)
    if len(ws) > N:
        lb = max(lb, ws[N - 1] + ws[N])
    return lb
