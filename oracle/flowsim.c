/*
 * flowsim.c -- plain CPU oracle for NEXT f4: the fluid (flow-level) simulator
 * with the RailS / uniform / ECMP / REPS / MinRTT policies and CCT percentiles.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as oracle.c): only tests/, smoke() and
 * bench.py's cpu legs may load it; it shares nothing with the CUDA path.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, R#n = DESIGN.md reading.
 * The paper's own experiments ran on Mininet + Soft-RoCE; SPEC's flowsim
 * module substitutes a fluid max-min model, and so do we (R#35-R#39).
 *
 *   Topology (R#35): M domains x N rails; NIC(k,n) attaches to
 *   leaf n; S spines fully connected to the leaves.  Directed links:
 *     GPU_UP(k,g,n)   gpu(k,g) -> nic(k,n), g != n        cap R1  (one per pair)
 *     NIC_UP(k,n)     nic(k,n) -> leaf(n)                 cap R2
 *     LEAF_SPINE(n,j) leaf(n) -> spine(j)                 cap Rs
 *     SPINE_LEAF(j,m) spine(j) -> leaf(m)                 cap Rs
 *     NIC_DOWN(f,m)   leaf(m) -> nic(f,m)                 cap R2
 *     GPU_DOWN(f,n,m) nic(f,n) -> gpu(f,m), m != n        cap R1
 *   rail_path: [GPU_UP(k,g,n)] NIC_UP(k,n) NIC_DOWN(f,n) [GPU_DOWN(f,n,m)];
 *   spine_path from the source GPU's own NIC g to the destination GPU's
 *   own NIC m: NIC_UP(k,g) LEAF_SPINE(g,j) SPINE_LEAF(j,m) NIC_DOWN(f,m), or the
 *   direct leaf path NIC_UP(k,g) NIC_DOWN(f,g) when g = m.
 *
 *   Policies (R#36): flows of one all-to-all round, messages in
 *   (d, g, h) order, B = msg[d][g][h] > 0:
 *     0 LPT      chunks of the node's LPT schedule (orc_split + orc_lpt), each on
 *                the rail path of its rail (Alg. 2);
 *     1 UNIFORM  continuous P* = 1/N (Theorem 3): N flows of B/N bytes,
 *                one per rail path;
 *     2 ECMP     one flow per message on the spine path, spine = the R#14 hash of
 *                (src GPU, dst GPU) mod S ("binds flows to a single path");
 *     3 REPS     one flow per message split evenly over the S spine paths (P:840
 *                "per-packet spraying" as a fluid split);
 *     4 MINRTT   the LPT chunks, each on the spine path (fixed source NIC g)
 *                minimising max over its links of backlog/capacity at decision
 *                time (t = 0, chunks in (d, g, h, c) order), lowest spine
 *                on ties; backlog += chunk bytes on the chosen links;
 *     5 PLB      as ECMP, but at every completion event a flow whose rate was set
 *                by a congested spine link (a LEAF_SPINE / SPINE_LEAF bottleneck)
 *                re-hashes its spine: attempt a -> spine hash with seed + a*phi,
 *                at most every other event ("switch paths during idle
 *                periods"; R#36).
 *
 *   Max-min rates (R#37): progressive filling over subflows with
 *   share-weights: level x* = min over links of (cap - frozen rates) / (sum of
 *   unfrozen weights); every unfrozen subflow crossing a link at that level
 *   (within 1e-12 relative) is frozen at rate w * x*; repeat.
 *
 *   Event loop (R#38): rates; dt = min remaining / rate; t += dt;
 *   remaining -= rate * dt; every flow whose own remaining / rate is within
 *   1e-9 relative of dt completes at t (a scale-free form of S:522's 1-byte
 *   clamp, so that S:529's volume scaling holds), its residual added to its links.
 *
 *   Results (R#39): completion time per message (max over its flows), T =
 *   max, per-link bytes, CCT mean / p80 / p95 / p99 over messages (nearest rank),
 *   busbw = total bytes / T, and the largest domain-pair rate over N*R2 seen at any
 *   event (Theorem 1 ceiling).
 *
 * Compile with -ffp-contract=off (plain IEEE binary64 expressions).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FS_OK 0
#define FS_EINVAL (-1)
#define FS_ENOMEM (-3)
#define FS_MAXL 4

/* from oracle.c */
int32_t orc_ecmp_rail(uint64_t seed, int64_t src, int64_t dst, int32_t N);
int64_t orc_chunk_count(int32_t N, int64_t G, const int64_t *msg, int64_t C);
int64_t orc_split(int32_t N, int64_t G, const int64_t *msg, int64_t C, int32_t *ch_g,
                  int32_t *ch_h, int64_t *ch_c, int64_t *ch_size);
void orc_lpt(int64_t F, int32_t N, const int64_t *w, int64_t *order, int32_t *rail,
             int64_t *off, int64_t *load);

typedef struct {
    int32_t M, N, S;
    double R1, R2, Rs;
} fs_topo;

/* ---------------------------------------------------------------- links */
static int64_t L_gpu_up(const fs_topo *t, int k, int g, int n) {
    return ((int64_t)k * t->N + g) * t->N + n;
}
static int64_t L_nic_up(const fs_topo *t, int k, int n) {
    return (int64_t)t->M * t->N * t->N + (int64_t)k * t->N + n;
}
static int64_t L_leaf_spine(const fs_topo *t, int n, int j) {
    return (int64_t)t->M * t->N * t->N + (int64_t)t->M * t->N + (int64_t)n * t->S + j;
}
static int64_t L_spine_leaf(const fs_topo *t, int j, int m) {
    return (int64_t)t->M * t->N * t->N + (int64_t)t->M * t->N + (int64_t)t->N * t->S +
           (int64_t)j * t->N + m;
}
static int64_t L_nic_down(const fs_topo *t, int f, int m) {
    return (int64_t)t->M * t->N * t->N + (int64_t)t->M * t->N + 2 * (int64_t)t->N * t->S +
           (int64_t)f * t->N + m;
}
static int64_t L_gpu_down(const fs_topo *t, int f, int n, int m) {
    return (int64_t)t->M * t->N * t->N + 2 * (int64_t)t->M * t->N + 2 * (int64_t)t->N * t->S +
           ((int64_t)f * t->N + n) * t->N + m;
}
int64_t orc_fs_nlinks(int32_t M, int32_t N, int32_t S) {
    return 2 * (int64_t)M * N * N + 2 * (int64_t)M * N + 2 * (int64_t)N * S;
}
static double link_cap(const fs_topo *t, int64_t l) {
    const int64_t a = (int64_t)t->M * t->N * t->N, b = (int64_t)t->M * t->N;
    const int64_t c = (int64_t)t->N * t->S;
    if (l < a) return t->R1;                 /* GPU_UP */
    if (l < a + b) return t->R2;             /* NIC_UP */
    if (l < a + b + 2 * c) return t->Rs;     /* LEAF_SPINE, SPINE_LEAF */
    if (l < a + 2 * b + 2 * c) return t->R2; /* NIC_DOWN */
    return t->R1;                            /* GPU_DOWN */
}

/* rail_path */
static int rail_path(const fs_topo *t, int k, int g, int f, int m, int n, int64_t *p) {
    int c = 0;
    if (g != n) p[c++] = L_gpu_up(t, k, g, n);
    p[c++] = L_nic_up(t, k, n);
    p[c++] = L_nic_down(t, f, n);
    if (m != n) p[c++] = L_gpu_down(t, f, n, m);
    return c;
}
/* spine_path from NIC g to NIC m through spine j */
static int spine_path(const fs_topo *t, int k, int g, int f, int m, int j, int64_t *p) {
    if (g == m) return rail_path(t, k, g, f, m, g, p);
    p[0] = L_nic_up(t, k, g);
    p[1] = L_leaf_spine(t, g, j);
    p[2] = L_spine_leaf(t, j, m);
    p[3] = L_nic_down(t, f, m);
    return 4;
}

/* ---------------------------------------------------------------- flows */
typedef struct {
    int64_t nflow, nsub;
    uint8_t *init;    /* [nsub] active at t = 0 (PLB's spare spine paths are not) */
    double *bytes;    /* [nflow] */
    int64_t *msg;     /* [nflow] message index d*N*G + g*G + h */
    int64_t *sub0;    /* [nflow+1] first subflow */
    double *w;        /* [nsub] share-weight */
    int32_t *nl;      /* [nsub] */
    int64_t *links;   /* [nsub][FS_MAXL] */
} fs_flows;

static void fs_free(fs_flows *F) {
    free(F->init); free(F->bytes); free(F->msg); free(F->sub0); free(F->w); free(F->nl);
    free(F->links);
    memset(F, 0, sizeof(*F));
}

static int fs_alloc(fs_flows *F, int64_t nflow, int64_t nsub) {
    F->nflow = 0;
    F->nsub = 0;
    F->bytes = (double *)calloc((size_t)(nflow + 1), sizeof(double));
    F->msg = (int64_t *)calloc((size_t)(nflow + 1), sizeof(int64_t));
    F->sub0 = (int64_t *)calloc((size_t)(nflow + 2), sizeof(int64_t));
    F->w = (double *)calloc((size_t)(nsub + 1), sizeof(double));
    F->nl = (int32_t *)calloc((size_t)(nsub + 1), sizeof(int32_t));
    F->links = (int64_t *)calloc((size_t)(nsub + 1) * FS_MAXL, sizeof(int64_t));
    F->init = (uint8_t *)calloc((size_t)(nsub + 1), 1);
    if (!F->init || !F->bytes || !F->msg || !F->sub0 || !F->w || !F->nl || !F->links) return FS_ENOMEM;
    return FS_OK;
}

static void add_flow(fs_flows *F, double bytes, int64_t msg) {
    F->bytes[F->nflow] = bytes;
    F->msg[F->nflow] = msg;
    F->sub0[F->nflow] = F->nsub;
    F->nflow++;
    F->sub0[F->nflow] = F->nsub;
}
static int64_t *add_sub(fs_flows *F, double w) {
    F->w[F->nsub] = w;
    F->init[F->nsub] = 1;
    F->nsub++;
    F->sub0[F->nflow] = F->nsub;
    return F->links + (F->nsub - 1) * FS_MAXL;
}

/* Materialise the policy's flows (R#36). */
static int build_flows(const fs_topo *t, int64_t C, uint64_t seed, int policy,
                       const int64_t *msg, fs_flows *F) {
    const int M = t->M, N = t->N, S = t->S;
    const int64_t G = (int64_t)M * N, L = orc_fs_nlinks(M, N, S);
    /* upper bounds on counts */
    int64_t nflow = 0, nsub = 0;
    for (int d = 0; d < M; d++) {
        const int64_t *md = msg + (int64_t)d * N * G;
        int64_t nch = orc_chunk_count(N, G, md, C);
        int64_t nm = 0;
        for (int64_t i = 0; i < N * G; i++) nm += md[i] > 0;
        nflow += nch > nm * N ? nch : nm * N;
        nsub += nch > nm * (N > S ? N : S) ? nch : nm * (N > S ? N : S);
    }
    int rc = fs_alloc(F, nflow, nsub);
    if (rc) return rc;
    double *backlog = (double *)calloc((size_t)L, sizeof(double));
    if (!backlog) return FS_ENOMEM;
    for (int d = 0; d < M; d++) {
        const int64_t *md = msg + (int64_t)d * N * G;
        if (policy == 0 || policy == 4) {
            int64_t nch = orc_chunk_count(N, G, md, C);
            int32_t *cg = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nch + 1));
            int32_t *chh = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nch + 1));
            int64_t *cc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nch + 1));
            int64_t *cs = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nch + 1));
            int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nch + 1));
            int32_t *rail = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nch + 1));
            int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nch + 1));
            int64_t *load = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1));
            if (!cg || !chh || !cc || !cs || !ord || !rail || !off || !load) return FS_ENOMEM;
            orc_split(N, G, md, C, cg, chh, cc, cs);
            if (policy == 0) orc_lpt(nch, N, cs, ord, rail, off, load);
            for (int64_t i = 0; i < nch; i++) {   /* chunks in (g, h, c) order */
                const int g = cg[i], h = chh[i], f = h / N, m = h % N;
                add_flow(F, (double)cs[i], (int64_t)d * N * G + (int64_t)g * G + h);
                int64_t *p = add_sub(F, 1.0);
                if (policy == 0) {
                    F->nl[F->nsub - 1] = rail_path(t, d, g, f, m, rail[i], p);
                } else {
                    /* MinRTT: min over spines of max backlog/cap on the path */
                    int64_t best[FS_MAXL];
                    int bn = 0;
                    double bscore = 0.0;
                    const int nj = (g == m) ? 1 : S;
                    for (int j = 0; j < nj; j++) {
                        int64_t q[FS_MAXL];
                        const int qn = spine_path(t, d, g, f, m, j, q);
                        double sc = 0.0;
                        for (int a = 0; a < qn; a++) {
                            const double v = backlog[q[a]] / link_cap(t, q[a]);
                            if (v > sc) sc = v;
                        }
                        if (j == 0 || sc < bscore) {
                            bscore = sc;
                            bn = qn;
                            memcpy(best, q, sizeof(best));
                        }
                    }
                    for (int a = 0; a < bn; a++) {
                        p[a] = best[a];
                        backlog[best[a]] += (double)cs[i];
                    }
                    F->nl[F->nsub - 1] = bn;
                }
            }
            free(cg); free(chh); free(cc); free(cs); free(ord); free(rail); free(off); free(load);
        } else {
            for (int g = 0; g < N; g++)
                for (int64_t h = 0; h < G; h++) {
                    const int64_t B = md[(int64_t)g * G + h];
                    if (B <= 0) continue;
                    const int f = (int)(h / N), m = (int)(h % N);
                    const int64_t mi = (int64_t)d * N * G + (int64_t)g * G + h;
                    if (policy == 1) {
                        for (int n = 0; n < N; n++) {
                            add_flow(F, (double)B / (double)N, mi);
                            int64_t *p = add_sub(F, 1.0);
                            F->nl[F->nsub - 1] = rail_path(t, d, g, f, m, n, p);
                        }
                    } else if (policy == 2) {
                        const int j = orc_ecmp_rail(seed, (int64_t)d * N + g, h, S);
                        add_flow(F, (double)B, mi);
                        int64_t *p = add_sub(F, 1.0);
                        F->nl[F->nsub - 1] = spine_path(t, d, g, f, m, j, p);
                    } else if (policy == 5) {
                        /* PLB: every spine path is a candidate; the ECMP one starts */
                        add_flow(F, (double)B, mi);
                        const int j0 = orc_ecmp_rail(seed, (int64_t)d * N + g, h, S);
                        const int nj = (g == m) ? 1 : S;
                        for (int j = 0; j < nj; j++) {
                            int64_t *p = add_sub(F, 1.0);
                            F->nl[F->nsub - 1] = spine_path(t, d, g, f, m, j, p);
                            F->init[F->nsub - 1] = (uint8_t)(nj == 1 || j == j0);
                        }
                    } else {
                        add_flow(F, (double)B, mi);
                        const int nj = (g == m) ? 1 : S;
                        for (int j = 0; j < nj; j++) {
                            int64_t *p = add_sub(F, 1.0 / (double)nj);
                            F->nl[F->nsub - 1] = spine_path(t, d, g, f, m, j, p);
                        }
                    }
                }
        }
    }
    free(backlog);
    return FS_OK;
}

/* ---------------------------------------------------------------- max-min */
/* Progressive filling (R#37) over the subflows with act[s] != 0.  rate[s] out. */
/* shit[s] (may be NULL): some bottleneck link of s's freezing step lies in the
 * spine layer [ls0, ls1) -- PLB's congestion signal. */
static void max_min(int64_t nsub, const int32_t *nl, const int64_t *links, const double *w,
                    const uint8_t *act, int64_t L, const double *cap, double *rate,
                    double *sumw, double *used, uint8_t *frozen, uint8_t *bott,
                    uint8_t *shit, int64_t ls0, int64_t ls1) {
    for (int64_t s = 0; s < nsub; s++) {
        frozen[s] = 0;
        rate[s] = 0.0;
    }
    for (;;) {
        for (int64_t l = 0; l < L; l++) { sumw[l] = 0.0; used[l] = 0.0; }
        int64_t left = 0;
        for (int64_t s = 0; s < nsub; s++) {
            if (!act[s]) continue;
            for (int a = 0; a < nl[s]; a++) {
                const int64_t l = links[s * FS_MAXL + a];
                if (frozen[s]) used[l] += rate[s];
                else sumw[l] += w[s];
            }
            left += !frozen[s];
        }
        if (left == 0) return;
        double xs = INFINITY;
        for (int64_t l = 0; l < L; l++) {
            if (sumw[l] <= 0.0) continue;
            double r = cap[l] - used[l];
            if (r < 0.0) r = 0.0;
            const double x = r / sumw[l];
            if (x < xs) xs = x;
        }
        for (int64_t l = 0; l < L; l++) {
            bott[l] = 0;
            if (sumw[l] <= 0.0) continue;
            double r = cap[l] - used[l];
            if (r < 0.0) r = 0.0;
            if (r / sumw[l] <= xs * (1.0 + 1e-12)) bott[l] = 1;
        }
        for (int64_t s = 0; s < nsub; s++) {
            if (!act[s] || frozen[s]) continue;
            int hit = 0, sp = 0;
            for (int a = 0; a < nl[s]; a++) {
                const int64_t l = links[s * FS_MAXL + a];
                hit |= bott[l];
                sp |= bott[l] && l >= ls0 && l < ls1;
            }
            if (hit) {
                rate[s] = w[s] * xs;
                frozen[s] = 1;
                if (shit) shit[s] = (uint8_t)sp;
            }
        }
    }
}

/* Exposed for the pins: rates of n subflows (links as [n][4], -1 padded). */
int orc_max_min(int64_t nsub, const int32_t *nl, const int64_t *links, const double *w,
                int64_t L, const double *cap, double *rate) {
    double *sumw = (double *)calloc((size_t)L + 1, sizeof(double));
    double *used = (double *)calloc((size_t)L + 1, sizeof(double));
    uint8_t *frozen = (uint8_t *)calloc((size_t)nsub + 1, 1);
    uint8_t *bott = (uint8_t *)calloc((size_t)L + 1, 1);
    uint8_t *act = (uint8_t *)malloc((size_t)nsub + 1);
    if (!sumw || !used || !frozen || !bott || !act) return FS_ENOMEM;
    memset(act, 1, (size_t)nsub + 1);
    max_min(nsub, nl, links, w, act, L, cap, rate, sumw, used, frozen, bott, NULL, 0, 0);
    free(sumw); free(used); free(frozen); free(bott); free(act);
    return FS_OK;
}

static int cmp_double(const void *a, const void *b) {
    const double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* ---------------------------------------------------------------- simulate */
/* msg int64 [M][N][G] (one round).  Outputs:
 *   msg_cct   double [M][N][G]  completion time of each message (0 if B = 0);
 *   link_bytes double [L];
 *   stats     double [10]: T, total bytes, busbw, CCT mean, p80, p95, p99,
 *             max domain-pair rate / (N*R2), events, flows. */
int orc_flowsim(int32_t M, int32_t N, int32_t S, double R1, double R2, double Rs, int64_t C,
                uint64_t seed, int32_t policy, const int64_t *msg, double *msg_cct,
                double *link_bytes, double *stats) {
    if (M < 2 || N < 1 || S < 1 || !(R1 > R2) || !(R2 > 0.0) || !(Rs > 0.0) || C < 1 ||
        policy < 0 || policy > 5)
        return FS_EINVAL;
    fs_topo t = {M, N, S, R1, R2, Rs};
    const int64_t G = (int64_t)M * N, L = orc_fs_nlinks(M, N, S);
    fs_flows F;
    memset(&F, 0, sizeof(F));
    int rc = build_flows(&t, C, seed, policy, msg, &F);
    if (rc) { fs_free(&F); return rc; }
    const int64_t nf = F.nflow, ns = F.nsub;
    double *cap = (double *)malloc(sizeof(double) * (size_t)L);
    double *sumw = (double *)calloc((size_t)L, sizeof(double));
    double *used = (double *)calloc((size_t)L, sizeof(double));
    uint8_t *bott = (uint8_t *)calloc((size_t)L, 1);
    double *rate = (double *)calloc((size_t)ns + 1, sizeof(double));
    uint8_t *frozen = (uint8_t *)calloc((size_t)ns + 1, 1);
    uint8_t *act = (uint8_t *)calloc((size_t)ns + 1, 1);
    double *rem = (double *)malloc(sizeof(double) * (size_t)(nf + 1));
    double *frate = (double *)calloc((size_t)nf + 1, sizeof(double));
    double *done = (double *)calloc((size_t)nf + 1, sizeof(double));
    double *pair = (double *)calloc((size_t)M * M, sizeof(double));
    uint8_t *fact = (uint8_t *)calloc((size_t)nf + 1, 1);
    uint8_t *shit = (uint8_t *)calloc((size_t)ns + 1, 1);
    int64_t *att = (int64_t *)calloc((size_t)nf + 1, sizeof(int64_t));
    int64_t *last = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nf + 1));
    if (!cap || !sumw || !used || !bott || !rate || !frozen || !act || !rem || !frate || !done ||
        !pair || !fact || !shit || !att || !last) {
        fs_free(&F);
        return FS_ENOMEM;
    }
    for (int64_t l = 0; l < L; l++) { cap[l] = link_cap(&t, l); link_bytes[l] = 0.0; }
    int64_t active = 0;
    for (int64_t i = 0; i < nf; i++) {
        rem[i] = F.bytes[i];
        fact[i] = 1;
        last[i] = -2;
        for (int64_t s = F.sub0[i]; s < F.sub0[i + 1]; s++) act[s] = F.init[s];
        active++;
    }
    double tnow = 0.0, maxpair = 0.0;
    int64_t events = 0;
    while (active > 0) {
        max_min(ns, F.nl, F.links, F.w, act, L, cap, rate, sumw, used, frozen, bott, shit,
                L_leaf_spine(&t, 0, 0), L_nic_down(&t, 0, 0));
        double dt = INFINITY;
        for (int64_t i = 0; i < nf; i++) {
            if (!fact[i]) continue;
            double r = 0.0;
            for (int64_t s = F.sub0[i]; s < F.sub0[i + 1]; s++) r += rate[s];
            frate[i] = r;
            const double x = rem[i] / r;
            if (x < dt) dt = x;
        }
        /* Theorem 1 ceiling: aggregate rate between two domains <= N*R2 */
        memset(pair, 0, sizeof(double) * (size_t)M * M);
        for (int64_t i = 0; i < nf; i++) {
            if (!fact[i]) continue;
            const int64_t mi = F.msg[i];
            const int d = (int)(mi / (N * G)), f = (int)((mi % G) / N);
            pair[(int64_t)d * M + f] += frate[i];
        }
        for (int64_t q = 0; q < (int64_t)M * M; q++)
            if (pair[q] / ((double)N * R2) > maxpair) maxpair = pair[q] / ((double)N * R2);
        tnow = tnow + dt;
        for (int64_t i = 0; i < nf; i++) {
            if (!fact[i]) continue;
            for (int64_t s = F.sub0[i]; s < F.sub0[i + 1]; s++) {
                const double b = rate[s] * dt;
                for (int a = 0; a < F.nl[s]; a++) link_bytes[F.links[s * FS_MAXL + a]] += b;
            }
            const double fin = rem[i] / frate[i];  /* this flow's own finish time */
            rem[i] = rem[i] - frate[i] * dt;
            if (fin <= dt * (1.0 + 1e-9)) {  /* finishes at this event (R#38) */
                /* the residual (|rem| < 1 byte) still crosses the links, in the
                 * subflows' rate proportions, so link bytes conserve the flow */
                for (int64_t s = F.sub0[i]; s < F.sub0[i + 1]; s++) {
                    const double b = rem[i] * (rate[s] / frate[i]);
                    for (int a = 0; a < F.nl[s]; a++) link_bytes[F.links[s * FS_MAXL + a]] += b;
                }
                done[i] = tnow;
                fact[i] = 0;
                for (int64_t s = F.sub0[i]; s < F.sub0[i + 1]; s++) act[s] = 0;
                active--;
            }
        }
        /* PLB (R#36): a flow held back by a spine bottleneck re-hashes its spine,
         * not at two consecutive events */
        if (policy == 5) {
            for (int64_t i = 0; i < nf; i++) {
                if (!fact[i] || F.sub0[i + 1] - F.sub0[i] < 2 || last[i] == events - 1) continue;
                int64_t cur = F.sub0[i];
                while (!act[cur]) cur++;
                if (!shit[cur]) continue;
                const int64_t mi = F.msg[i];
                const int64_t src = mi / G, dst = mi % G;
                att[i]++;
                const int j = orc_ecmp_rail(seed + (uint64_t)att[i] * 0x9E3779B97F4A7C15ULL, src,
                                            dst, S);
                last[i] = events;
                if (F.sub0[i] + j == cur) continue;
                act[cur] = 0;
                act[F.sub0[i] + j] = 1;
            }
        }
        events++;
    }
    /* per message completion = its last flow (R#39) */
    for (int64_t q = 0; q < (int64_t)M * N * G; q++) msg_cct[q] = 0.0;
    double total = 0.0, T = 0.0;
    for (int64_t i = 0; i < nf; i++) {
        if (done[i] > msg_cct[F.msg[i]]) msg_cct[F.msg[i]] = done[i];
        if (done[i] > T) T = done[i];
    }
    int64_t nm = 0;
    for (int64_t q = 0; q < (int64_t)M * N * G; q++)
        if (msg[q] > 0) { nm++; total += (double)msg[q]; }
    double *cs = (double *)malloc(sizeof(double) * (size_t)(nm + 1));
    int64_t k = 0;
    double sum = 0.0;
    for (int64_t q = 0; q < (int64_t)M * N * G; q++)
        if (msg[q] > 0) { cs[k++] = msg_cct[q]; sum += msg_cct[q]; }
    qsort(cs, (size_t)nm, sizeof(double), cmp_double);
    /* nearest rank: the ceil(p*n)-th smallest */
    const double ps[3] = {0.80, 0.95, 0.99};
    double pv[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < 3 && nm > 0; a++) {
        int64_t r = (int64_t)ceil(ps[a] * (double)nm);
        if (r < 1) r = 1;
        pv[a] = cs[r - 1];
    }
    stats[0] = T;
    stats[1] = total;
    stats[2] = T > 0.0 ? total / T : 0.0;
    stats[3] = nm > 0 ? sum / (double)nm : 0.0;
    stats[4] = pv[0];
    stats[5] = pv[1];
    stats[6] = pv[2];
    stats[7] = maxpair;
    stats[8] = (double)events;
    stats[9] = (double)nf;
    free(cs);
    free(cap); free(sumw); free(used); free(bott); free(rate); free(frozen); free(act);
    free(rem); free(frate); free(done); free(pair); free(fact); free(shit); free(att); free(last);
    fs_free(&F);
    return FS_OK;
}
