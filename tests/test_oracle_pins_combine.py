"""Pins for the combine-round oracle, the compact schedule and the ECMP loads
(-m "not gpu").

The combine functions of oracle.c (orc_transpose, orc_recv_offsets,
orc_pack_combine_node, orc_unpack_combine; Alg. 1 step 4, readings
R#28-R#31) are the checker of tests/test_gpu_combine.py, so here they are pinned on
things other than themselves:
  * a hand-worked M = 2, N = 2 dispatch + combine round (tests/golden);
  * the composition dispatch pack -> delivery -> expert -> combine pack -> unpack
    returns each token's own row, scaled by its experts' known factors and the gate
    weights -- a wrong in_off ordering, slot order, chunk lookup or rank breaks it;
  * orc_transpose is an involution; orc_recv_offsets is an exclusive prefix sum.
orc_compact (R#19) is pinned by expanding the compact form through the closed form
of the full-chunk prefix and comparing with the per-chunk LPT result of orc_lpt;
the ECMP loads by a hand example on the pinned hash values (R#14).
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
R2 = 5.0e10
SEED = oracle.DEFAULT_ECMP_SEED


def _bf16(vals) -> np.ndarray:
    """bf16 bit patterns of values exactly representable in bf16."""
    f = np.asarray(vals, np.float32)
    b = (f.view(np.uint32) >> 16).astype(np.uint16)
    assert np.array_equal((b.astype(np.uint32) << 16).view(np.float32), f)
    return b


def _rows_bytes(rows) -> np.ndarray:
    """[rows][H] values -> [rows][2H] bytes (little-endian bf16)."""
    b = _bf16(rows)
    return b.view(np.uint8).reshape(b.shape[0], -1) if b.ndim == 2 else b.view(np.uint8)


def _excl(v):
    v = np.asarray(v, np.int64)
    return np.concatenate([[0], np.cumsum(v)[:-1]]).astype(np.int64)


# ------------------------------------------------------------------ small identities
def test_transpose_is_involution():
    rng = np.random.default_rng(40)
    for _ in range(50):
        M, N = int(rng.integers(2, 7)), int(rng.integers(1, 6))
        G = M * N
        msg = rng.integers(0, 1000, size=(M, N, G)).astype(np.int64)
        t = oracle.transpose(M, N, msg)
        # definition R#28 read elementwise: comb[b][a] = disp[a][b] on the flat G x G view
        assert np.array_equal(t.reshape(G, G), msg.reshape(G, G).T)
        assert np.array_equal(oracle.transpose(M, N, t), msg)


def test_recv_offsets_exclusive_prefix():
    rng = np.random.default_rng(41)
    for _ in range(50):
        rows = rng.integers(0, 50, size=int(rng.integers(1, 40)))
        off = oracle.recv_offsets(rows)
        assert off[0] == 0
        assert np.array_equal(np.diff(off), rows[:-1])


# ------------------------------------------------------------------ hand-worked round
def test_combine_hand_example_M2N2():
    ex = GOLD["combine_hand_M2N2"]
    M, N, T, k, RB, C = (ex[x] for x in ("M", "N", "T", "k", "RB", "C"))
    G = M * N
    lut = np.array(ex["lut"], np.int32)
    topk = np.array(ex["topk"], np.int32)  # [M][N][T][k]
    x = [_rows_bytes(r) for r in ex["x_rows_by_gpu"]]  # per GPU a: [T][RB]
    counts = np.zeros((G, G), np.int64)
    msg = np.zeros((M, N, G), np.int64)
    rank = np.zeros((M, N, T, k), np.int32)
    disp = []
    for d in range(M):
        c, m, r = oracle.histogram_node(M, N, d, T, k, topk[d], lut, RB)
        counts[d * N:(d + 1) * N] = c
        msg[d], rank[d] = m, r
        s = oracle.schedule_node(m, C)
        base = _excl(s["send_load"])
        xn = np.stack([x[d * N + g] for g in range(N)])
        disp.append((s, base, oracle.pack_node(M, N, d, T, k, RB, C, xn, topk[d], lut, m, s, base,
                                               int(s["send_load"].sum()))))
    assert counts.tolist() == ex["counts_ab"]
    assert rank.tolist() == ex["rank"]
    in_off = np.stack([oracle.recv_offsets(counts[:, b]) for b in range(G)])
    assert in_off.tolist() == ex["in_off_ba"]
    msg_t = oracle.transpose(M, N, msg)
    assert msg_t.tolist() == ex["combine_msg"]
    y = [_rows_bytes(r) for r in ex["y_rows_by_gpu"]]  # identity experts, hand-filled
    bufs, bases, firsts, scheds = [], [], [], []
    for f in range(M):
        s = oracle.schedule_node(msg_t[f], C)
        ch = s["chunks"]
        got = [[int(ch["g"][i]), int(ch["h"][i]), int(ch["c"][i]), int(ch["size"][i]),
                int(s["rail"][i]), int(s["off"][i])] for i in range(len(ch["size"]))]
        assert got == ex["combine_chunks"][f]
        assert s["send_load"].tolist() == ex["combine_send_load"][f]
        base = _excl(s["send_load"])
        buf = oracle.pack_combine_node(M, N, f, RB, C, [y[f * N + m] for m in range(N)],
                                       in_off[f * N:(f + 1) * N], msg_t[f], s, base,
                                       int(s["send_load"].sum()))
        assert np.array_equal(buf, _rows_bytes(ex["combine_buffer_rows"][f]).reshape(-1))
        bufs.append(buf); bases.append(base); scheds.append(s)
        firsts.append(oracle.first_chunk_table(N, G, s))
    for d in range(M):
        for g in range(N):
            out = oracle.unpack_combine(M, N, d, g, T, k, RB, C, topk[d, g], lut, rank[d, g],
                                        np.ones((T, k), np.float32),
                                        [y[d * N + m] for m in range(N)],
                                        in_off[d * N:(d + 1) * N], bufs, bases, firsts, scheds)
            assert out.tolist() == ex["out_by_gpu"][d * N + g]


# ------------------------------------------------------------------ round trip
def _deliver(M, N, T, k, RB, C, topk, lut, x, msg, counts, disp):
    """Expert-input buffers by R#29, rebuilt from what the dispatch put on the rails:
    GPU b's rows are its messages in ascending source GPU a, each in (t,s) order;
    a remote message is reassembled from the sender node's rail buffers chunk by
    chunk (chunk c = message bytes [c*C, c*C + size) at rail_base[rail] + off), an
    intra-node one is taken straight from x (it crosses NVLink, not a rail)."""
    G = M * N
    rows = [[None] * G for _ in range(G)]
    for d in range(M):
        s, base, out = disp[d]
        ch = s["chunks"]
        stream = {}
        for i in range(len(ch["size"])):
            key = (int(ch["g"][i]), int(ch["h"][i]))
            a = int(base[s["rail"][i]] + s["off"][i])
            stream.setdefault(key, {})[int(ch["c"][i])] = out[a:a + int(ch["size"][i])]
        for g in range(N):
            a = d * N + g
            for b in range(G):
                if b // N == d:
                    sel = [x[a][t] for t in range(T) for s_ in range(k)
                           if lut[topk[d, g, t, s_]] == b]
                    rows[a][b] = np.stack(sel) if sel else np.zeros((0, RB), np.uint8)
                elif msg[d, g, b] > 0:
                    parts = stream[(g, b)]
                    byt = np.concatenate([parts[c] for c in sorted(parts)])
                    assert len(byt) == msg[d, g, b]
                    rows[a][b] = byt.reshape(-1, RB)
                else:
                    rows[a][b] = np.zeros((0, RB), np.uint8)
                assert rows[a][b].shape[0] == counts[a, b]
    return [np.concatenate([rows[a][b] for a in range(G)]) if counts[:, b].sum()
            else np.zeros((0, RB), np.uint8) for b in range(G)]


@pytest.mark.parametrize("M,N,T,k,E,H,C,seed", [
    (2, 2, 6, 1, 2, 2, 4, 1),        # one row per chunk
    (3, 2, 20, 2, 4, 4, 12, 2),      # rows straddle chunks (C = 1.5 rows)
    (3, 3, 15, 2, 6, 8, 8, 3),       # C < RB: a row spans two chunks
    (4, 2, 25, 3, 4, 4, 64, 4),      # several rows per chunk, k = 3
    (2, 4, 30, 2, 8, 2, 20, 5),      # N = 4, C not a multiple of RB
])
def test_combine_round_trip_scaled_experts(M, N, T, k, E, H, C, seed):
    """dispatch -> expert -> combine -> unpack returns sum_s w[t][s] * 2^(h_s mod 3) * x_t.

    Expert GPU h multiplies every row it holds by 2^(h mod 3) (exact on small
    integers in bf16); gate weights are dyadic; so every product and sum is exact in
    fp32 and the expected value is computed in float64 from the routing alone."""
    rng = np.random.default_rng(100 + seed)
    G, RB = M * N, 2 * H
    lut = (np.arange(M * E) // E * N + (np.arange(M * E) % E) % N).astype(np.int32)
    topk = np.zeros((M, N, T, k), np.int32)
    for d in range(M):
        for g in range(N):
            for t in range(T):
                topk[d, g, t] = rng.choice(M * E, size=k, replace=False)
    vals = rng.integers(-60, 61, size=(G, T, H)).astype(np.float32)
    x = [_rows_bytes(vals[a]) for a in range(G)]
    w = rng.choice(np.array([0.25, 0.5, 1.0, 2.0], np.float32), size=(M, N, T, k))
    counts = np.zeros((G, G), np.int64)
    msg = np.zeros((M, N, G), np.int64)
    rank = np.zeros((M, N, T, k), np.int32)
    disp = []
    for d in range(M):
        c, m, r = oracle.histogram_node(M, N, d, T, k, topk[d], lut, RB)
        counts[d * N:(d + 1) * N] = c
        msg[d], rank[d] = m, r
        s = oracle.schedule_node(m, C)
        base = _excl(s["send_load"])
        xn = np.stack([x[d * N + g] for g in range(N)])
        disp.append((s, base, oracle.pack_node(M, N, d, T, k, RB, C, xn, topk[d], lut, m, s,
                                               base, int(s["send_load"].sum()))))
    recv = _deliver(M, N, T, k, RB, C, topk, lut, x, msg, counts, disp)
    # experts: GPU h scales its rows by 2^(h mod 3)
    y = []
    for b in range(G):
        v = (recv[b].view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        y.append(_rows_bytes(v * np.float32(2 ** (b % 3))) if len(v) else recv[b])
    in_off = np.stack([oracle.recv_offsets(counts[:, b]) for b in range(G)])
    msg_t = oracle.transpose(M, N, msg)
    bufs, bases, firsts, scheds = [], [], [], []
    for f in range(M):
        s = oracle.schedule_node(msg_t[f], C)
        base = _excl(s["send_load"])
        bufs.append(oracle.pack_combine_node(M, N, f, RB, C, [y[f * N + m] for m in range(N)],
                                             in_off[f * N:(f + 1) * N], msg_t[f], s, base,
                                             int(s["send_load"].sum())))
        bases.append(base); scheds.append(s)
        firsts.append(oracle.first_chunk_table(N, G, s))
    for d in range(M):
        for g in range(N):
            a = d * N + g
            out = oracle.unpack_combine(M, N, d, g, T, k, RB, C, topk[d, g], lut, rank[d, g],
                                        w[d, g], [y[d * N + m] for m in range(N)],
                                        in_off[d * N:(d + 1) * N], bufs, bases, firsts, scheds)
            for t in range(T):
                want = np.zeros(H, np.float64)
                for s_ in range(k):
                    h = int(lut[topk[d, g, t, s_]])
                    want += float(w[d, g, t, s_]) * 2.0 ** (h % 3) * vals[a, t].astype(np.float64)
                assert np.array_equal(out[t].astype(np.float64), want), (d, g, t)


# ------------------------------------------------------------------ compact form
def test_compact_matches_closed_form_expansion():
    """R#19 + a2: expanding the compact schedule chunk by chunk -- full chunk c of
    message m is node-global full chunk i = full_base[m] + c, on rail i mod N at
    offset floor(i/N)*C (every full chunk precedes every remainder in LPT order and
    they come in emission order, so LPT deals them round-robin); the remainder is at
    (rem_rail, rem_off) -- gives exactly orc_lpt's per-chunk (rail, offset)."""
    rng = np.random.default_rng(42)
    checked = 0
    for trial in range(240):
        M, N = int(rng.integers(2, 6)), int(rng.integers(1, 9))
        G = M * N
        C = int(rng.choice([1, 7, 16, 100, 4096]))
        kind = trial % 4
        if kind == 0:    # mixed, many zero-byte messages
            msg = rng.integers(0, 5 * C + 3, size=(N, G)) * (rng.random((N, G)) < 0.5)
        elif kind == 1:  # remainder-only messages (B < C) and exact multiples
            msg = np.where(rng.random((N, G)) < 0.5, rng.integers(0, C, size=(N, G)),
                           C * rng.integers(0, 4, size=(N, G)))
        elif kind == 2:  # a silent node except one message
            msg = np.zeros((N, G), np.int64)
            msg[int(rng.integers(0, N)), int(rng.integers(0, G))] = int(rng.integers(1, 9 * C + 1))
        else:            # equal sizes (tie-break path)
            msg = np.full((N, G), int(rng.integers(1, 3 * C + 1))) * (rng.random((N, G)) < 0.7)
        d = int(rng.integers(0, M))
        msg = msg.astype(np.int64)
        msg[:, d * N:(d + 1) * N] = 0  # intra-node bytes are never scheduled (R#2)
        s = oracle.schedule_node(msg, C)
        ch = s["chunks"]
        n_full_seen = 0
        for i in range(len(ch["size"])):
            g, h, c, size = int(ch["g"][i]), int(ch["h"][i]), int(ch["c"][i]), int(ch["size"][i])
            if c < msg[g, h] // C:
                gi = int(s["full_base"][g, h]) + c
                assert (int(s["rail"][i]), int(s["off"][i])) == (gi % N, (gi // N) * C)
                n_full_seen += 1
            else:
                assert size == msg[g, h] % C
                assert (int(s["rail"][i]), int(s["off"][i])) == \
                    (int(s["rem_rail"][g, h]), int(s["rem_off"][g, h]))
        assert n_full_seen == s["n_full"] == int((msg // C).sum())
        assert s["n_rem"] == int((msg % C > 0).sum())
        # full_base is the exclusive prefix of floor(B/C) in (g, h) order, also over
        # zero-byte and remainder-only messages
        assert np.array_equal(s["full_base"].reshape(-1), _excl((msg // C).reshape(-1)))
        assert np.array_equal(s["rem_rail"] >= 0, msg % C > 0)
        assert (s["rem_off"][msg % C == 0] == 0).all()
        checked += 1
    assert checked >= 200


# ------------------------------------------------------------------ ECMP loads
def test_ecmp_hand_example():
    ex = GOLD["ecmp_hand_M2N8"]
    M, N = ex["M"], ex["N"]
    msg = np.zeros((M, N, M * N), np.int64)
    for d, g, h, b in ex["messages"]:
        msg[d, g, h] = b
    _, ev = oracle.run_unit_matrix(M, N, 1 << 20, R2, SEED, msg)
    assert ev["S_e"][0].tolist() == ex["S_e_node0"]
    assert ev["S_e"][1].tolist() == [0] * N
    assert ev["R_e"][1].tolist() == ex["R_e_node1"]
    assert ev["R_e"][0].tolist() == [0] * N
    assert ev["maxload_e"] == ex["maxload_e"] and ev["total_e"] == ex["total_e"]
    assert ev["T_e"] * R2 == pytest.approx(ex["T_e_times_R2"], rel=1e-15)
    assert ev["busbw_e"] / R2 == pytest.approx(ex["busbw_e_over_R2"], rel=1e-15)


def test_busbw_zero_traffic_reading():
    # R#40: SPEC's busbw has "pre: cct_total > 0"; with no
    # inter-node byte T = 0, and the oracle reports busbw = 0 instead of 0/0
    M, N = 3, 2
    msg = np.zeros((M, N, M * N), np.int64)
    _, ev = oracle.run_unit_matrix(M, N, 64, R2, SEED, msg)
    assert ev["total"] == 0 and ev["T"] == 0.0 and ev["busbw"] == 0.0 and ev["busbw_e"] == 0.0
