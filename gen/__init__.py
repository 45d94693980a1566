"""Seeded synthetic INPUT generators (routing, traffic matrices, payload).

Shared by the oracle side and the CUDA side: this module produces inputs only and
holds none of the method's arithmetic (no histogram, chunking, sort, LPT, eval or
pack).  Its splitmix64 is its own copy, used as a counter-based random source.

Recipes:
  * routing   -- Table 1 "Uniform" gating: top-k distinct experts per
                 token, destination node uniform, instance id f*E + e; LUT places
                 instance (f, e) on GPU f*N + (e mod N) (reading R#21).
  * receiver-skewed D^(1) -- Table 1 "Receiver-skewed" (uniform token input, Zipf
                 gating): Zipf(s) weights over a per-unit random ranking
                 of the G destination GPUs; every source GPU emits V bytes.
  * sender-skewed D^(1)   -- Table 1 "Sender-skewed".
  * uniform D^(1)         -- Table 1 "Uniform".
  * payload x  -- opaque 64-bit words from a counter hash (NaN encodings included).
Integer rounding of Zipf volumes: floor, remainder to the lowest-indexed remote
destination so each row sums to V exactly.

Everything is counter-based: any slice (unit, node range) can be regenerated
alone, on CPU or GPU, with identical values.
"""
from __future__ import annotations

import numpy as np
import torch

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def _s64(v: int) -> int:
    v &= M64
    return v - (1 << 64) if v >= (1 << 63) else v


def mix64_int(z: int) -> int:
    z = (z + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * _C1) & M64
    z = ((z ^ (z >> 27)) * _C2) & M64
    return z ^ (z >> 31)


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 viewed as uint64."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def mix64_t(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 output step on int64 tensors (two's-complement wraparound)."""
    z = z + _s64(GOLDEN)
    z = (z ^ _srl(z, 30)) * _s64(_C1)
    z = (z ^ _srl(z, 27)) * _s64(_C2)
    return z ^ _srl(z, 31)


def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
        return z ^ (z >> np.uint64(31))


def unit_seed(base: int, u: int) -> int:
    return mix64_int((base ^ u) & M64)


def draw31(sigma: int, ctr: torch.Tensor) -> torch.Tensor:
    """31-bit non-negative draw for counter ctr under unit seed sigma."""
    return _srl(mix64_t(ctr ^ _s64(sigma)), 33)


# ---------------------------------------------------------------- configs
KiB = 1024
MiB = 1024 * 1024

# BASELINE.json configs with the readings of DESIGN.md section 4 (R#22, R#23).
CONFIGS = {
    "c1": dict(kind="routing", M=4, N=4, T=4096, k=2, E=8, H=4096, C=64 * KiB, U=1),
    "c2": dict(kind="matrix", M=16, N=8, C=1 * MiB, U=1000, V=256 * MiB, zipf_s=1.2,
               skew="receiver"),
    "c3": dict(kind="routing", M=64, N=8, T=4096, k=2, E=8, H=4096, C=32 * KiB, U=1),
    "c4": dict(kind="routing", M=128, N=8, T=4096, k=2, E=8, H=6144, C=32 * KiB, U=32),
    "c5": dict(kind="matrix", M=256, N=8, C=None, U=1, V=256 * MiB, zipf_s=1.2,
               skew="receiver", C_sweep=[(4 * KiB) << i for i in range(11)]),
}
BASE_SEED = 0x2A115000
R2_DEFAULT = 5.0e10            # 400 Gb/s per rail per direction (R#9)
ECMP_SEED = 0x9E3779B97F4A7C15  # R#14


def config_seed(cfg_id: int) -> int:
    return BASE_SEED + cfg_id


# ---------------------------------------------------------------- routing
def inst_lut(M: int, N: int, E: int) -> torch.Tensor:
    """Instance (f, e) -> global GPU f*N + (e mod N) (R#21)."""
    f = torch.arange(M, dtype=torch.int64).repeat_interleave(E)
    e = torch.arange(E, dtype=torch.int64).repeat(M)
    return (f * N + (e % N)).to(torch.int32)


def routing(M: int, N: int, T: int, k: int, E: int, seed: int, u: int, d0: int = 0,
            nd: int | None = None, device="cpu") -> torch.Tensor:
    """Expert-instance ids int32 [nd][N][T][k] of nodes d0..d0+nd-1 in unit u.

    Token tau = (d*N + g)*T + t.  Distinct experts by a partial Fisher-Yates over
    E with draws r_i = draw31(sigma, 64*tau + i); destination node of slot s is
    draw31(sigma, 64*tau + 32 + s) mod M.
    """
    if nd is None:
        nd = M - d0
    assert 1 <= k <= E and k <= 32
    sigma = unit_seed(seed, u)
    dev = torch.device(device)
    out = torch.empty((nd, N, T, k), dtype=torch.int32, device=dev)
    step = max(1, (1 << 22) // (N * T))  # nodes per batch (bounded temporaries)
    for a in range(0, nd, step):
        b = min(nd, a + step)
        tau = (torch.arange((d0 + a) * N * T, (d0 + b) * N * T, dtype=torch.int64, device=dev))
        n = tau.numel()
        perm = torch.arange(E, dtype=torch.int64, device=dev).expand(n, E).clone()
        for i in range(k):
            r = draw31(sigma, tau * 64 + i)
            j = i + r % (E - i)
            pi = perm[:, i].clone()
            pj = perm.gather(1, j[:, None])[:, 0]
            perm[:, i] = pj
            perm.scatter_(1, j[:, None], pi[:, None])
        e = perm[:, :k]
        s_idx = torch.arange(k, dtype=torch.int64, device=dev)
        f = draw31(sigma, tau[:, None] * 64 + 32 + s_idx[None, :]) % M
        inst = (f * E + e).to(torch.int32)
        out[a:b] = inst.view(b - a, N, T, k)
    return out


def payload(M: int, N: int, T: int, row_bytes: int, seed: int, u: int, d0: int, nd: int,
            device="cpu", out: torch.Tensor | None = None) -> torch.Tensor:
    """Opaque token rows int64-words [nd][N][T][row_bytes/8] of nodes d0.. in unit u.

    Word = mix64(sigma_x ^ global word index); bit patterns include NaN encodings
    when viewed as bf16, which the pack must carry unchanged.
    """
    assert row_bytes % 8 == 0
    W = row_bytes // 8
    sigma = unit_seed(seed ^ 0x5A5A5A5A, u)
    dev = torch.device(device)
    if out is None:
        out = torch.empty((nd, N, T, W), dtype=torch.int64, device=dev)
    per_node = N * T * W
    for a in range(nd):
        base = ((d0 + a) * per_node)
        idx = torch.arange(base, base + per_node, dtype=torch.int64, device=dev)
        out[a] = mix64_t(idx ^ _s64(sigma)).view(N, T, W)
    return out


# ---------------------------------------------------------------- D^(1) matrices
def zipf_weights(s: float, n: int) -> np.ndarray:
    """w_r = r^-s / sum_{r'} r'^-s, r = 1..n."""
    r = np.arange(1, n + 1, dtype=np.float64)
    w = r ** (-s)
    return w / w.sum()


def _perm(sigma: int, n: int) -> np.ndarray:
    """Seeded permutation of range(n): argsort of counter-hash keys."""
    keys = mix64_np((np.arange(n, dtype=np.uint64) ^ np.uint64(sigma)))
    return np.argsort(keys, kind="stable")


def _remote_mask(M: int, N: int) -> np.ndarray:
    G = M * N
    d = np.arange(M)[:, None]
    f = (np.arange(G) // N)[None, :]
    return d != f  # [M][G]


def d1_receiver_skew(M: int, N: int, V: int, s: float, seed: int, u: int) -> np.ndarray:
    """int64 [M][N][G]; every source GPU sends V bytes, Zipf over a per-unit ranking
    of destination GPUs (common to all senders: incast onto hot receivers)."""
    G = M * N
    sigma = unit_seed(seed, u)
    pi = _perm(sigma, G)
    rank = np.empty(G, np.int64)
    rank[pi] = np.arange(1, G + 1)
    w = rank.astype(np.float64) ** (-s)
    rem = _remote_mask(M, N)                        # [M][G]
    Wd = (w[None, :] * rem).sum(axis=1)             # [M]
    D = np.floor((V * w[None, :]) / Wd[:, None]).astype(np.int64) * rem
    first = np.argmax(rem, axis=1)                  # lowest-indexed remote h
    D[np.arange(M), first] += V - D.sum(axis=1)
    return np.repeat(D[:, None, :], N, axis=1).copy()


def d1_sender_skew(M: int, N: int, V: int, s: float, seed: int, u: int) -> np.ndarray:
    """int64 [M][N][G]; node d's GPUs each send floor(M*V*z(d)) spread uniformly."""
    G = M * N
    sigma = unit_seed(seed, u)
    pi = _perm(sigma, M)
    rank = np.empty(M, np.int64)
    rank[pi] = np.arange(1, M + 1)
    z = zipf_weights(s, M)[rank - 1]
    Vd = np.floor(M * V * z).astype(np.int64)
    rem = _remote_mask(M, N)
    each = Vd // (G - N)
    D = each[:, None] * rem
    first = np.argmax(rem, axis=1)
    D[np.arange(M), first] += Vd - D.sum(axis=1)
    return np.repeat(D[:, None, :], N, axis=1).copy()


def d1_uniform(M: int, N: int, V: int) -> np.ndarray:
    G = M * N
    rem = _remote_mask(M, N)
    D = (V // (G - N)) * rem.astype(np.int64)
    first = np.argmax(rem, axis=1)
    D[np.arange(M), first] += V - D.sum(axis=1)
    return np.repeat(D[:, None, :], N, axis=1).copy()


def d1_sparse_topk(M: int, N: int, V: int, sparsity: float, K: int, seed: int, u: int) -> np.ndarray:
    """Table 1 "Sparse": floor(sparsity*M) seeded
    destination domains receive nothing; every source GPU picks K distinct active
    domains other than its own (seeded) and splits V equally over their N*K GPUs
    (floor, remainder to the first chosen GPU).  int64 [M][N][G]."""
    G = M * N
    sigma = unit_seed(seed, u)
    order = _perm(sigma, M)
    n_off = int(np.floor(sparsity * M))
    active = np.ones(M, bool)
    active[order[:n_off]] = False
    D = np.zeros((M, N, G), np.int64)
    for d in range(M):
        cand = np.nonzero(active & (np.arange(M) != d))[0]
        if len(cand) < K:
            raise ValueError("fewer active destination domains than K")
        for g in range(N):
            keys = mix64_np((cand.astype(np.uint64) * np.uint64(1000003)
                             + np.uint64((d * N + g) * 7919)) ^ np.uint64(sigma))
            pick = cand[np.argsort(keys, kind="stable")[:K]]
            dst = np.sort(np.concatenate([np.arange(f * N, (f + 1) * N) for f in pick]))
            each = V // len(dst)
            D[d, g, dst] = each
            D[d, g, dst[0]] += V - each * len(dst)
    return D


def d1_units(cfg: dict, seed: int, u0: int, U: int) -> np.ndarray:
    """Stack of D^(1) matrices int64 [U][M][N][G] for units u0..u0+U-1."""
    M, N, V = cfg["M"], cfg["N"], cfg["V"]
    out = np.empty((U, M, N, M * N), np.int64)
    for i in range(U):
        if cfg.get("skew") == "receiver":
            out[i] = d1_receiver_skew(M, N, V, cfg["zipf_s"], seed, u0 + i)
        elif cfg.get("skew") == "sender":
            out[i] = d1_sender_skew(M, N, V, cfg["zipf_s"], seed, u0 + i)
        elif cfg.get("skew") == "sparse":
            out[i] = d1_sparse_topk(M, N, V, cfg["sparsity"], cfg.get("K", 2), seed, u0 + i)
        else:
            out[i] = d1_uniform(M, N, V)
    return out


# ---------------------------------------------------------------- NEXT f1 inputs
def expert_outputs(shape, seed: int, u: int, device="cpu") -> torch.Tensor:
    """Finite bf16 expert-output rows as int16 bit patterns, `shape` = [..., H]:
    sign random, exponent 2^-8 .. 2^2, random 7-bit mantissa (no NaN/Inf, so the
    fp32 weighted sums are comparable bit for bit)."""
    sigma = unit_seed(seed ^ 0xE0E0E0, u)
    n = 1
    for s in shape:
        n *= s
    out = torch.empty(n, dtype=torch.int16, device=device)
    step = 1 << 26  # bounded int64 temporaries
    for a in range(0, n, step):
        b = min(n, a + step)
        idx = torch.arange(a, b, dtype=torch.int64, device=device)
        z = mix64_t(idx ^ _s64(sigma))
        sign = z & 1
        ex = 119 + (_srl(z, 1) % 11)
        mant = _srl(z, 8) & 0x7F
        bits = (sign << 15) | (ex << 7) | mant
        out[a:b] = (bits - ((bits >> 15) << 16)).to(torch.int16)
    return out.view(*shape)


def gate_weights(shape, seed: int, u: int, device="cpu") -> torch.Tensor:
    """Top-k gate weights in [0, 1), exactly representable in fp32 (24-bit grid)."""
    sigma = unit_seed(seed ^ 0x6A7E, u)
    n = 1
    for s in shape:
        n *= s
    idx = torch.arange(n, dtype=torch.int64, device=device)
    z = _srl(mix64_t(idx ^ _s64(sigma)), 40)
    return (z.to(torch.float64) / float(1 << 24)).to(torch.float32).view(*shape)
