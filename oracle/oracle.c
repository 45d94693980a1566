/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the RailS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path under
 * paper_2510_19262_b200/csrc; neither side includes or links the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (RailS, arXiv 2510.19262),
 * "S:n" = SPEC.md line n, "R#n" = reading n of DESIGN.md section 3 (the table of
 * readings where the paper is silent or ambiguous).
 *
 * Every function here follows the paper's definition or algorithm step by step,
 * in the paper's order, with no blocking, fusion or reordering:
 *   orc_histogram_node  D^(1) row block of node d, P:193 (Traffic Matrix), Alg.1
 *                       "Select input slices ... according to Gate" P:575;
 *                       stable rank = sequential counter (R#18).
 *   orc_split           fixed-size chunking, P:603 ("fixed-size data chunks");
 *                       S:274-282; R#3.
 *   orc_lpt             Alg. 2 steps 2-3: sort W by descending
 *                       weight, ties by GPU index (R#4), then
 *                       j* = argmin LoadState (lowest index on ties, R#5),
 *                       record (w_i, j*), LoadState[j*] += w_i.
 *   orc_compact         the compact schedule by its definition (R#19).
 *   orc_eval            Eq. 4-5 loads S and R via the rail pairing
 *                       NIC(k,n) -> NIC(f,n) (R#7); T (R#8);
 *                       T* (Thm 2 + Thm 3); busbw (R#10);
 *                       MSE Eq. 6 / Alg. 2 step 6, nMSE (R#12);
 *                       ECMP whole-message hash baseline (R#13, R#14).
 *   orc_eval_uniform    the uniform split P* = 1/N (Thm 3; R#41) on
 *                       the same load model.
 *   orc_pack_node       rail buffers by definition (R#18-R#20): message byte
 *                       stream = concatenation of rows in (t,s) order, chunk c of
 *                       message (g,h) copied to rail[j] + offset.
 *   orc_qp_map          NEXT f2: Alg. 2 step 4 round-robin QP index
 *                       per rail in assignment order (R#34).
 *
 * Parity pins live in tests/test_oracle_pins.py and tests/test_oracle_pins_combine.py
 * (worked examples from the paper / SPEC and hand-worked ones, closed forms,
 * invariants, round trips and brute force).  The ECMP hash is this build's
 * choice (R#14): "parity unpinned" beyond the splitmix64 textbook value and the
 * hand-computed pins listed in DESIGN.md.
 *
 * Integers are int64 throughout; floating point is IEEE binary64 with the exact
 * expressions of DESIGN.md section 3 (R#25).  Compile with -ffp-contract=off.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERANGE (-2)
#define ORC_ENOMEM (-3)

/* ---------------------------------------------------------------- ECMP hash */
/* R#14: one splitmix64 output step. */
uint64_t orc_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return z;
}

/* R#13/R#14: ECMP "binds flows to a single path via hashing": the whole
 * message from global source GPU src to global destination GPU dst goes on rail
 * (uint32)(mix64(key ^ seed) >> 32) mod N, key = (src << 32) | dst. */
int32_t orc_ecmp_rail(uint64_t seed, int64_t src, int64_t dst, int32_t N) {
    uint64_t key = ((uint64_t)src << 32) | (uint64_t)dst;
    uint32_t hi = (uint32_t)(orc_mix64(key ^ seed) >> 32);
    return (int32_t)(hi % (uint32_t)N);
}

/* ---------------------------------------------------------------- histogram */
/* One node d.  topk[g][t][s] are expert-instance ids, lut maps instance -> global
 * destination GPU h in [0, M*N).  counts[g][h] counts every (t,s) (intra-node too,
 * R#2); msg[g][h] = counts*RB for remote h and 0 for h on node d (R#2);
 * rank[g][t][s] = number of earlier (t',s') of GPU g with the same h, earlier in
 * the loop order g, t, s (R#18).  Returns ORC_ERANGE on an out-of-range id. */
int orc_histogram_node(int32_t M, int32_t N, int32_t d, int32_t T, int32_t k,
                       const int32_t *topk, const int32_t *lut, int32_t n_inst,
                       int64_t row_bytes, int32_t *counts, int64_t *msg,
                       int32_t *rank) {
    int64_t G = (int64_t)M * N;
    for (int64_t i = 0; i < (int64_t)N * G; i++) counts[i] = 0;
    for (int32_t g = 0; g < N; g++) {
        for (int32_t t = 0; t < T; t++) {
            for (int32_t s = 0; s < k; s++) {
                int64_t e = ((int64_t)g * T + t) * k + s;
                int32_t inst = topk[e];
                if (inst < 0 || inst >= n_inst) return ORC_ERANGE;
                int32_t h = lut[inst];
                if (h < 0 || h >= G) return ORC_ERANGE;
                if (rank) rank[e] = counts[(int64_t)g * G + h];
                counts[(int64_t)g * G + h] += 1;
            }
        }
    }
    for (int32_t g = 0; g < N; g++) {
        for (int64_t h = 0; h < G; h++) {
            int64_t f = h / N;
            msg[(int64_t)g * G + h] =
                (f == d) ? 0 : (int64_t)counts[(int64_t)g * G + h] * row_bytes;
        }
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- chunking */
/* P:603 / S:277 / R#3: message B -> floor(B/C) chunks of C bytes plus one chunk
 * of B mod C bytes when that is nonzero.  Zero-byte messages emit nothing. */
int64_t orc_chunk_count(int32_t N, int64_t G, const int64_t *msg, int64_t C) {
    int64_t F = 0;
    for (int64_t i = 0; i < (int64_t)N * G; i++) {
        int64_t B = msg[i];
        if (B <= 0) continue;
        F += B / C + ((B % C) > 0 ? 1 : 0);
    }
    return F;
}

/* Emission order: g ascending, then h ascending, then chunk index c ascending.
 * The chunk id is the emission index (R#4). */
int64_t orc_split(int32_t N, int64_t G, const int64_t *msg, int64_t C,
                  int32_t *ch_g, int32_t *ch_h, int64_t *ch_c, int64_t *ch_size) {
    int64_t F = 0;
    for (int32_t g = 0; g < N; g++) {
        for (int64_t h = 0; h < G; h++) {
            int64_t B = msg[(int64_t)g * G + h];
            if (B <= 0) continue;
            int64_t nfull = B / C;
            for (int64_t c = 0; c < nfull; c++) {
                ch_g[F] = g; ch_h[F] = (int32_t)h; ch_c[F] = c; ch_size[F] = C; F++;
            }
            if (B % C > 0) {
                ch_g[F] = g; ch_h[F] = (int32_t)h; ch_c[F] = nfull; ch_size[F] = B % C; F++;
            }
        }
    }
    return F;
}

/* ---------------------------------------------------------------- LPT */
static const int64_t *g_sort_w;  /* comparator context (single-threaded oracle) */

/* Alg. 2 step 2: descending weight; ties by GPU index, completed to
 * the total order (size desc, emission index asc) = (size desc, g, h, c) (R#4). */
static int cmp_desc_then_index(const void *a, const void *b) {
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    if (g_sort_w[i] > g_sort_w[j]) return -1;
    if (g_sort_w[i] < g_sort_w[j]) return 1;
    return (i < j) ? -1 : (i > j) ? 1 : 0;
}

/* Alg. 2 on F flows with weights w[0..F) given in tie-break order.
 * Outputs: order[p] = id of the p-th flow in LPT order; rail[i], off[i] per flow
 * id (off = LoadState[j*] before the update, R#19); load[N] = final LoadState. */
void orc_lpt(int64_t F, int32_t N, const int64_t *w, int64_t *order,
             int32_t *rail, int64_t *off, int64_t *load) {
    /* Initialization before each All-to-All: LoadState[1..N] <- 0. */
    for (int32_t j = 0; j < N; j++) load[j] = 0;
    /* Step 2: sort W by descending weight, break ties by GPU index. */
    for (int64_t i = 0; i < F; i++) order[i] = i;
    g_sort_w = w;
    qsort(order, (size_t)F, sizeof(int64_t), cmp_desc_then_index);
    /* Step 3: iterative allocation. */
    for (int64_t p = 0; p < F; p++) {
        int64_t i = order[p];
        int32_t jstar = 0;                      /* argmin, lowest index on ties (R#5) */
        for (int32_t j = 1; j < N; j++)
            if (load[j] < load[jstar]) jstar = j;
        rail[i] = jstar;                        /* record (w_i, j*) */
        off[i] = load[jstar];
        load[jstar] += w[i];                    /* LoadState[j*] += w_i */
    }
}

/* ---------------------------------------------------------------- compact form */
/* By definition (R#19): full_base[g][h] = number of full chunks (c < floor(B/C))
 * emitted before message (g,h) in emission order; rem_rail/rem_off = rail/offset
 * of the message's remainder chunk, -1/0 if none; n_full, n_rem = node totals. */
void orc_compact(int32_t N, int64_t G, const int64_t *msg, int64_t C, int64_t F,
                 const int32_t *ch_g, const int32_t *ch_h, const int64_t *ch_c,
                 const int64_t *ch_size, const int32_t *rail, const int64_t *off,
                 int64_t *full_base, int8_t *rem_rail, int64_t *rem_off,
                 int64_t *n_full, int32_t *n_rem) {
    for (int64_t i = 0; i < (int64_t)N * G; i++) {
        full_base[i] = 0; rem_rail[i] = -1; rem_off[i] = 0;
    }
    int64_t seen_full = 0;
    int32_t nr = 0;
    int64_t prev_msg = -1;
    for (int64_t i = 0; i < F; i++) {
        int64_t m = (int64_t)ch_g[i] * G + ch_h[i];
        int64_t B = msg[m];
        if (m != prev_msg) {
            /* every message between prev_msg and m (exclusive) has no chunks */
            for (int64_t q = prev_msg + 1; q < m; q++) full_base[q] = seen_full;
            full_base[m] = seen_full;
            prev_msg = m;
        }
        if (ch_c[i] < B / C) {
            seen_full++;
        } else {
            (void)ch_size;
            rem_rail[m] = (int8_t)rail[i];
            rem_off[m] = off[i];
            nr++;
        }
    }
    for (int64_t q = prev_msg + 1; q < (int64_t)N * G; q++) full_base[q] = seen_full;
    *n_full = seen_full;
    *n_rem = nr;
}

/* ---------------------------------------------------------------- eval */
/* Exact unsigned 128-bit value -> double, as DESIGN.md R#25 fixes it:
 * (double)hi * 2^64 + (double)lo, each step IEEE round-to-nearest. */
static double u128_to_double(unsigned __int128 v) {
    uint64_t hi = (uint64_t)(v >> 64), lo = (uint64_t)v;
    if (hi == 0) return (double)lo;
    return (double)hi * 18446744073709551616.0 + (double)lo;
}

/* MSE of one node's LoadState, Eq. 6 with T_opt = mean,
 * evaluated exactly as sum_j (N*L_j - sum L)^2 / N^3 (R#11). */
double orc_mse(int32_t N, const int64_t *L) {
    __int128 sum = 0;
    for (int32_t j = 0; j < N; j++) sum += L[j];
    unsigned __int128 sq = 0;
    for (int32_t j = 0; j < N; j++) {
        __int128 dev = (__int128)N * L[j] - sum;
        sq += (unsigned __int128)(dev * dev);
    }
    return u128_to_double(sq) / ((double)N * (double)N * (double)N);
}

/* Normalized MSE ("0-1 scale", R#12): MSE of L_j / sum L against 1/N
 * = mse / (sum L)^2, 0 when sum L = 0. */
double orc_nmse(int32_t N, const int64_t *L) {
    int64_t sum = 0;
    for (int32_t j = 0; j < N; j++) sum += L[j];
    if (sum == 0) return 0.0;
    double m = orc_mse(N, L);
    return m / ((double)sum * (double)sum);
}

/* One unit (one all-to-all round, R#6) over all M nodes.
 * msg: [M][N][G] message bytes (D^(1), intra-node zero).
 * Chunk list with any assignment: ch_d, ch_h (global dst GPU), ch_size, ch_rail.
 * Outputs (caller-allocated):
 *   S[M][N], R[M][N], S_e[M][N], R_e[M][N]            (int64)
 *   ints[6]  = maxload, maxload_e, total, rowmax, colmax, total_e
 *   dbl[5]   = T, T_e, T_star, busbw, busbw_e
 *   mse[M], nmse[M]
 */
void orc_eval(int32_t M, int32_t N, double R2, uint64_t ecmp_seed,
              const int64_t *msg, int64_t F, const int32_t *ch_d,
              const int32_t *ch_h, const int64_t *ch_size, const int32_t *ch_rail,
              int64_t *S, int64_t *R, int64_t *S_e, int64_t *R_e,
              int64_t *ints, double *dbl, double *mse, double *nmse) {
    int64_t G = (int64_t)M * N;
    for (int64_t i = 0; i < (int64_t)M * N; i++) { S[i] = R[i] = S_e[i] = R_e[i] = 0; }
    /* Eq. 4-5 on the discrete assignment: a chunk of node d on rail j bound for
     * domain f = h / N adds to S[d][j] and R[f][j] (rail pairing P:431, R#7). */
    for (int64_t i = 0; i < F; i++) {
        int64_t f = ch_h[i] / N;
        S[(int64_t)ch_d[i] * N + ch_rail[i]] += ch_size[i];
        R[f * N + ch_rail[i]] += ch_size[i];
    }
    /* ECMP baseline: each whole message on one hashed rail (R#13). */
    int64_t total_e = 0;
    for (int32_t d = 0; d < M; d++)
        for (int32_t g = 0; g < N; g++)
            for (int64_t h = 0; h < G; h++) {
                int64_t B = msg[((int64_t)d * N + g) * G + h];
                if (B <= 0) continue;
                int32_t e = orc_ecmp_rail(ecmp_seed, (int64_t)d * N + g, h, N);
                S_e[(int64_t)d * N + e] += B;
                R_e[(h / N) * N + e] += B;
                total_e += B;
            }
    /* T = most loaded NIC, sending or receiving, over R2. */
    int64_t maxload = 0, maxload_e = 0, total = 0;
    for (int64_t i = 0; i < (int64_t)M * N; i++) {
        if (S[i] > maxload) maxload = S[i];
        if (R[i] > maxload) maxload = R[i];
        if (S_e[i] > maxload_e) maxload_e = S_e[i];
        if (R_e[i] > maxload_e) maxload_e = R_e[i];
        total += S[i];
    }
    /* T* = max(max row sum, max column sum of D^(2)) / (N R2) (Thm 2 + Thm 3). */
    int64_t rowmax = 0, colmax = 0;
    for (int32_t d = 0; d < M; d++) {
        int64_t rs = 0;
        for (int64_t i = 0; i < (int64_t)N * G; i++) rs += msg[(int64_t)d * N * G + i];
        if (rs > rowmax) rowmax = rs;
    }
    for (int32_t f = 0; f < M; f++) {
        int64_t cs = 0;
        for (int32_t d = 0; d < M; d++)
            for (int32_t g = 0; g < N; g++)
                for (int32_t m = 0; m < N; m++)
                    cs += msg[((int64_t)d * N + g) * G + (int64_t)f * N + m];
        if (cs > colmax) colmax = cs;
    }
    ints[0] = maxload; ints[1] = maxload_e; ints[2] = total;
    ints[3] = rowmax; ints[4] = colmax; ints[5] = total_e;
    double T = (double)maxload / R2;
    double T_e = (double)maxload_e / R2;
    int64_t lb = rowmax > colmax ? rowmax : colmax;
    double T_star = (double)lb / ((double)N * R2);
    dbl[0] = T; dbl[1] = T_e; dbl[2] = T_star;
    /* busbw = total bytes / T (R#10); 0 when nothing crosses the rails */
    dbl[3] = (total > 0) ? (double)total / T : 0.0;
    dbl[4] = (total_e > 0) ? (double)total_e / T_e : 0.0;
    for (int32_t d = 0; d < M; d++) {
        mse[d] = orc_mse(N, S + (int64_t)d * N);
        nmse[d] = orc_nmse(N, S + (int64_t)d * N);
    }
}

/* Uniform policy (Theorem 3's continuous optimum P*_{k,f,n} = 1/N, P:452-455;
 * reading R#41): every message of B bytes is split over all N rails, rail j taking
 * floor(B/N) bytes plus one more when j < B mod N, on the same load model as the
 * LPT and ECMP assignments (Eq. 4-5, R#7).  Outputs: S_u[M][N], R_u[M][N],
 * *maxload_u, dbl[2] = T_u = maxload_u / R2, busbw_u = total / T_u (0 without
 * traffic, R#40). */
void orc_eval_uniform(int32_t M, int32_t N, double R2, const int64_t *msg, int64_t *S_u,
                      int64_t *R_u, int64_t *maxload_u, double *dbl) {
    int64_t G = (int64_t)M * N;
    int64_t total = 0;
    for (int64_t i = 0; i < (int64_t)M * N; i++) { S_u[i] = 0; R_u[i] = 0; }
    for (int32_t d = 0; d < M; d++)
        for (int32_t g = 0; g < N; g++)
            for (int64_t h = 0; h < G; h++) {
                int64_t B = msg[((int64_t)d * N + g) * G + h];
                if (B <= 0) continue;
                int64_t f = h / N;
                for (int32_t j = 0; j < N; j++) {
                    int64_t part = B / N + ((j < B % N) ? 1 : 0);
                    S_u[(int64_t)d * N + j] += part;
                    R_u[f * N + j] += part;
                }
                total += B;
            }
    int64_t mx = 0;
    for (int64_t i = 0; i < (int64_t)M * N; i++) {
        if (S_u[i] > mx) mx = S_u[i];
        if (R_u[i] > mx) mx = R_u[i];
    }
    *maxload_u = mx;
    double T_u = (double)mx / R2;
    dbl[0] = T_u;
    dbl[1] = (total > 0) ? (double)total / T_u : 0.0;
}

/* ---------------------------------------------------------------- pack */
/* Rail buffers of one node d by definition (R#18-R#20).
 * x: [N][T][RB] rows of node d; topk/lut as in the histogram; msg: [N][G].
 * Chunks in emission order with their LPT rail/offset.  out + rail_base[j] is
 * the start of rail j's buffer (rail_base[j] + S[d][j] <= out_cap is checked).
 * Step 1 builds the byte stream of each message (g,h): the rows x[g][t] of every
 * (t,s) with lut[topk[g][t][s]] = h, in ascending (t,s).  Step 2 copies chunk c
 * (bytes [c*C, c*C + size) of its stream) to out + rail_base[rail] + off. */
int orc_pack_node(int32_t M, int32_t N, int32_t d, int32_t T, int32_t k,
                  int64_t RB, int64_t C, const uint8_t *x, const int32_t *topk,
                  const int32_t *lut, const int64_t *msg, int64_t F,
                  const int32_t *ch_g, const int32_t *ch_h, const int64_t *ch_c,
                  const int64_t *ch_size, const int32_t *ch_rail,
                  const int64_t *ch_off, const int64_t *rail_base, uint8_t *out,
                  int64_t out_cap) {
    int64_t G = (int64_t)M * N;
    (void)d;
    uint8_t **stream = (uint8_t **)calloc((size_t)(N * G), sizeof(uint8_t *));
    int64_t *fill = (int64_t *)calloc((size_t)(N * G), sizeof(int64_t));
    if (!stream || !fill) { free(stream); free(fill); return ORC_ENOMEM; }
    int rc = ORC_OK;
    for (int64_t m = 0; m < (int64_t)N * G; m++) {
        if (msg[m] > 0) {
            stream[m] = (uint8_t *)malloc((size_t)msg[m]);
            if (!stream[m]) { rc = ORC_ENOMEM; goto done; }
        }
    }
    for (int32_t g = 0; g < N; g++)
        for (int32_t t = 0; t < T; t++)
            for (int32_t s = 0; s < k; s++) {
                int32_t h = lut[topk[((int64_t)g * T + t) * k + s]];
                int64_t m = (int64_t)g * G + h;
                if (msg[m] <= 0) continue;            /* intra-node: not sent (R#2) */
                memcpy(stream[m] + fill[m], x + ((int64_t)g * T + t) * RB, (size_t)RB);
                fill[m] += RB;
            }
    for (int64_t i = 0; i < F; i++) {
        int64_t m = (int64_t)ch_g[i] * G + ch_h[i];
        int64_t dst = rail_base[ch_rail[i]] + ch_off[i];
        if (dst < 0 || dst + ch_size[i] > out_cap) { rc = ORC_ERANGE; goto done; }
        memcpy(out + dst, stream[m] + ch_c[i] * C, (size_t)ch_size[i]);
    }
done:
    for (int64_t m = 0; m < (int64_t)N * G; m++) free(stream[m]);
    free(stream);
    free(fill);
    return rc;
}

/* ================================================================ NEXT f1: combine */
/* Combine all-to-all (Alg. 1 step 4): the expert outputs of every
 * dispatched row travel back from expert GPU h = f*N+m to the token's GPU (d,g);
 * it is a separate all-to-all round with its own LoadState (R#6).
 *
 * orc_transpose: combine traffic D_c[f][m][d*N+g] = D_d[d][g][f*N+m] (R#28). */
void orc_transpose(int32_t M, int32_t N, const int64_t *disp, int64_t *comb) {
    int64_t G = (int64_t)M * N;
    for (int64_t a = 0; a < G; a++)          /* a = d*N+g: dispatch source GPU */
        for (int64_t b = 0; b < G; b++)      /* b = f*N+m: dispatch destination */
            comb[b * G + a] = disp[a * G + b];
}

/* Expert-output buffer of GPU (f,m) (R#29): the rows it received in dispatch,
 * message by message in ascending source GPU a = d*N+g, each message's rows in
 * their dispatch order (rank rho).  rows_in[a] = dispatch counts[a][f*N+m]
 * (intra-node sources included: those rows came over NVLink).  Returns the
 * first row of message a in y: in_off[a] = sum_{a' < a} rows_in[a']. */
void orc_recv_offsets(int64_t G, const int64_t *rows_in, int64_t *in_off) {
    int64_t run = 0;
    for (int64_t a = 0; a < G; a++) { in_off[a] = run; run += rows_in[a]; }
}

/* Combine pack of sender node f by definition (R#29-R#30): combine message
 * (m, a) = rows [in_off_m[a], in_off_m[a] + cnt) of y_m, i.e. the bytes of the
 * expert outputs in dispatch order; chunk c of it (from the combine round's LPT
 * schedule, chunk list ch_* in emission order) is copied to
 * out + rail_base[rail] + off.  Intra-node messages (a on node f) are not sent.
 * y: [N] pointers to [rows][RB]; in_off: [N][G]; msgc: combine bytes [N][G]. */
int orc_pack_combine_node(int32_t M, int32_t N, int32_t f, int64_t RB, int64_t C,
                          const uint8_t *const *y, const int64_t *in_off,
                          const int64_t *msgc, int64_t F, const int32_t *ch_g,
                          const int32_t *ch_h, const int64_t *ch_c, const int64_t *ch_size,
                          const int32_t *ch_rail, const int64_t *ch_off,
                          const int64_t *rail_base, uint8_t *out, int64_t out_cap) {
    int64_t G = (int64_t)M * N;
    (void)f;
    for (int64_t i = 0; i < F; i++) {
        int32_t m = ch_g[i];
        int64_t a = ch_h[i];
        const uint8_t *stream = y[m] + in_off[(int64_t)m * G + a] * RB;
        int64_t dst = rail_base[ch_rail[i]] + ch_off[i];
        if (msgc[(int64_t)m * G + a] <= 0) return ORC_ERANGE;
        if (dst < 0 || dst + ch_size[i] > out_cap) return ORC_ERANGE;
        memcpy(out + dst, stream + ch_c[i] * C, (size_t)ch_size[i]);
    }
    return ORC_OK;
}

static float bf16_to_float(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float x;
    memcpy(&x, &u, 4);
    return x;
}

/* Unpack + top-k weighted combine on GPU (d,g) (Alg. 1 step 5 input; R#31):
 *   out[t][e] = sum_{s=0..k-1} w[t][s] * row(t,s)[e]      (e < H = RB/2 bf16 values)
 * accumulated in fp32 in the order s = 0..k-1 (each product and sum rounded to
 * fp32, no FMA).  row(t,s) is the expert output of slot (t,s): message
 * (h -> (d,g)) of the combine round, h = lut[topk[t][s]], at message row rho =
 * rank[t][s] (the dispatch rank).  If h is on node d the row never crossed a rail
 * and is read from y of GPU h (row in_off[h][d*N+g] + rho); otherwise from the
 * combine rail buffers of node f = h/N: chunk c = floor(rho*RB / C) ... located
 * through the chunk list of node f (first chunk of each message: first[m][a]).
 * rails_f: [M] pointers to node f's combine rail buffer block (rail_base applied
 * by the caller through rb[f][j]); ch_rail/ch_off/first: per node f arrays.
 * Returns ORC_ERANGE if a row is not found. */
int orc_unpack_combine(int32_t M, int32_t N, int32_t d, int32_t g, int32_t T, int32_t k,
                       int64_t RB, int64_t C, const int32_t *topk, const int32_t *lut,
                       const int32_t *rank, const float *w, const uint8_t *const *y_node_d,
                       const int64_t *in_off_node_d, const uint8_t *const *rails_f,
                       const int64_t *const *rb_f, const int64_t *const *first_f,
                       const int32_t *const *rail_f, const int64_t *const *off_f,
                       float *out) {
    int64_t G = (int64_t)M * N;
    int64_t H = RB / 2;
    int64_t a = (int64_t)d * N + g;
    uint8_t *row = (uint8_t *)malloc((size_t)RB);
    if (!row) return ORC_ENOMEM;
    for (int32_t t = 0; t < T; t++) {
        for (int64_t e = 0; e < H; e++) out[(int64_t)t * H + e] = 0.0f;
        for (int32_t s = 0; s < k; s++) {
            int64_t h = lut[topk[(int64_t)t * k + s]];
            int64_t rho = rank[(int64_t)t * k + s];
            int64_t fdst = h / N, m = h % N;
            if (fdst == d) {
                const uint8_t *src = y_node_d[m] + (in_off_node_d[m * G + a] + rho) * RB;
                memcpy(row, src, (size_t)RB);
            } else {
                /* gather the row piece by piece from node f's combine chunks */
                int64_t p = rho * RB, got = 0;
                while (got < RB) {
                    int64_t c = (p + got) / C;
                    int64_t in_c = (p + got) - c * C;
                    int64_t idx = first_f[fdst][m * G + a] + c;
                    int64_t len = C - in_c;
                    if (len > RB - got) len = RB - got;
                    int32_t j = rail_f[fdst][idx];
                    const uint8_t *src = rails_f[fdst] + rb_f[fdst][j] + off_f[fdst][idx] + in_c;
                    memcpy(row + got, src, (size_t)len);
                    got += len;
                }
            }
            float wt = w[(int64_t)t * k + s];
            for (int64_t e = 0; e < H; e++) {
                uint16_t b;
                memcpy(&b, row + 2 * e, 2);
                float prod = wt * bf16_to_float(b);
                out[(int64_t)t * H + e] = out[(int64_t)t * H + e] + prod;
            }
        }
    }
    free(row);
    return ORC_OK;
}

/* ================================================================ NEXT f2: QP map */
/* Alg. 2 step 4: "For each assignment (w_i, j*): select port p from
 * NIC j* by round-robin; map (j*, p) to a QP in NIC's QP set; bind w_i to the
 * chosen QP."  Reading R#34: one counter per rail, reset with the
 * LoadState at the start of the all-to-all round; the assignments are
 * visited in Step-3 order, and the chunk gets the rail's counter modulo
 * qps_per_rail, then the counter advances.
 *   order[p] = index of the p-th assigned chunk (orc_lpt), rail[i] = its rail;
 *   qp[i] = QP index of chunk i in [0, qps_per_rail). */
int orc_qp_map(int64_t F, int32_t N, const int64_t *order, const int32_t *rail,
               int64_t qps_per_rail, int64_t *qp) {
    if (qps_per_rail < 1) return ORC_ERANGE;
    int64_t *next = (int64_t *)calloc((size_t)N, sizeof(int64_t));
    if (!next) return ORC_ENOMEM;
    for (int64_t p = 0; p < F; p++) {
        int64_t i = order[p];
        int32_t j = rail[i];
        qp[i] = next[j] % qps_per_rail;
        next[j] += 1;
    }
    free(next);
    return ORC_OK;
}
