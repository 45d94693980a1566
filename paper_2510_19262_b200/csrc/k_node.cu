// k_node.cu -- a2-a5 fused: one CTA per (unit, node) computes the node's compact
// LPT schedule and its evaluation in ONE kernel (sm_100a).
//
// a2 (R#3): message B of (g,h) -> floor(B/C) full chunks + one remainder of
//    B mod C bytes.  Full chunks are never materialised: every full chunk (size C)
//    is larger than every remainder (< C) and full chunks are emitted in (g,h,c)
//    order, so under Alg. 2's sort (size desc, ties by GPU index, R#4) they form
//    the prefix of the sorted list in emission order, and LPT from all-zero loads
//     deals them round-robin: full chunk i -> rail i mod N at offset
//    floor(i/N)*C (lowest-index argmin, R#5).  Phase A writes full_base = exclusive
//    prefix of floor(B/C) in (g,h) order (one block scan per tile of messages) and
//    compacts the remainders (at most one per message) in (g,h) order.
// a3: phase B sorts the remainders by size descending with a stable
//    LSD radix sort on key = C-1-size over only the key bits that vary (radix.cuh
//    radix_sort_narrow: routing remainders are multiples of the row size, so C3's
//    keys vary in 2 bits and one 2-bit pass sorts them); stability keeps
//    (g,h) order among equal sizes = the tie-break R#4.  In shared memory when the
//    node fits (N*G <= 16384), else in a global scratch.
// a4: phase C, warp 0 runs the serial chain (lpt.cuh) over the sorted
//    list; results land in sorted order (shared memory when they fit); runs of equal
//    sizes are recorded as (start state, length) and written by the whole CTA at the
//    start of phase D.  Phase D expands the results to per-message rem_rail /
//    rem_off through the sort's inverse permutation (and the QP map of Alg. 2 step
//    4, R#34, when asked).
// a5 (EVAL): while warp 0 runs the chain, the other warps add the full chunks into
//    R_d[f][j] by the closed form (message block (g, f*N..f*N+N-1) holds the
//    node-global full chunks [P_gf, P_g,f+1); rail j receives cnt_j(b) - cnt_j(a),
//    cnt_j(x) = floor(x/N) + (j < x mod N)); phase A already added the ECMP bytes
//    (R#13-R#14) and the uniform split (R#41) per destination node; phase D adds
//    the remainders.  S[d] is the chain's LoadState (Eq. 4); R_d is added into a
//    per-unit accumulator (int64 atomics: exact, order-free); MSE/nMSE as Eq. 6.
//    The last CTA of a unit to arrive (arrival counter) moves the accumulator into
//    red_sum / red_max, re-zeroes it, and -- when the call holds every node of the
//    unit -- finalizes T, T*, busbw (Thm 2 + 3); the last CTA of the
//    grid computes the rail offsets.  So a whole single-rank schedule + evaluation
//    is one launch, and the workspace is left zeroed for the next call.
#include "common.cuh"
#ifdef RAILS_NODE_TIMING
__device__ unsigned long long g_node_t[32];
__device__ unsigned long long g_node_cta[4][512];  // per CTA: start A, C, D, F (first 512)
// chain instrumentation (off unless asked for: each adds work to the timed chain):
// -DRAILS_LPT_CLK sums clock64 cycles of the chain's parts in registers (slots 25..28),
// -DRAILS_LPT_COUNT counts its paths (slots 20..23: runs, single steps, windows, groups)
#ifdef RAILS_LPT_CLK
#define LPT_CLK() clock64()
#define LPT_ACC_DECL long long lpt_acc_[4] = {0, 0, 0, 0};
#define LPT_ACC(k, t0) lpt_acc_[k] += clock64() - (t0)
#define LPT_ACC_FLUSH                                                \
  if (blockIdx.x == 0 && threadIdx.x == 0) {                         \
    for (int k_ = 0; k_ < 4; ++k_) g_node_t[25 + k_] = lpt_acc_[k_]; \
  }
#endif
#ifdef RAILS_LPT_COUNT
#define LPT_COUNT(i)                                                   \
  do {                                                                 \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_node_t[20 + (i)] += 1; \
  } while (0)
#endif
#endif
#include "eval.cuh"
#include "lpt.cuh"
#include "radix.cuh"

#ifdef RAILS_NODE_TIMING
// phase timestamps of CTA 0 (globaltimer ns), debug builds only (tools/node_timing.py)
#define NODE_T(i)                                                         \
  do {                                                                    \
    if (blockIdx.x == 0 && threadIdx.x == 0) g_node_t[i] = globaltimer_ns(); \
  } while (0)
#define NODE_TL(i)                              \
  do {                                          \
    if (threadIdx.x == 0) g_node_t[i] = globaltimer_ns(); \
  } while (0)
#define NODE_TC(k)                                                         \
  do {                                                                     \
    if (threadIdx.x == 0 && blockIdx.x < 512) g_node_cta[k][blockIdx.x] = globaltimer_ns(); \
  } while (0)
#define NODE_TW(i)                                                         \
  do {                                                                     \
    if (blockIdx.x == 0 && threadIdx.x == 32) g_node_t[i] = globaltimer_ns(); \
  } while (0)
extern "C" int rails_debug_node_reset() {
  unsigned long long z[32] = {0};
  return cudaMemcpyToSymbol(g_node_t, z, sizeof(z)) == cudaSuccess ? 0 : -5;
}
extern "C" int rails_debug_node_cta(unsigned long long* host2048) {
  return cudaMemcpyFromSymbol(host2048, g_node_cta, 2048 * sizeof(unsigned long long)) ==
                 cudaSuccess
             ? 0
             : -5;
}
extern "C" int rails_debug_node_times(unsigned long long* host32) {
  return cudaMemcpyFromSymbol(host32, g_node_t, 32 * sizeof(unsigned long long)) == cudaSuccess
             ? 0
             : -5;
}
#else
#define NODE_T(i) \
  do {            \
  } while (0)
#define NODE_TL(i) \
  do {             \
  } while (0)
#define NODE_TW(i) \
  do {             \
  } while (0)
#define NODE_TC(k) \
  do {             \
  } while (0)
#endif

namespace rails {

constexpr int NODE_MAX_THREADS = 512;
constexpr int NODE_MAX_RUNS = 32;  // deferred cyclic runs per chain (lpt.cuh RunList)
constexpr long long NODE_SMEM_ITEMS = 16384;  // N*G kept in shared memory

struct NodeArgs {
  const int64_t* msg;
  long long NG;
  int M, N, d0, nd, U;
  long long C;
  int cshift, nbits;
  uint64_t seed;
  double R2;
  rails_sched_t s;
  int32_t* rem_qp;
  int Q;
  uint64_t* res_g;     // [nseg][NG] chain results when not in shared memory
  uint32_t* qp_g;      // [nseg][NG] QP of each sorted remainder (QP map only)
  uint8_t* scratch;    // sort buffers when !SMEM
  rails_eval_t e;
  int64_t* acc;        // [U][rsl + RAILS_RED_MAX_LEN], zero between calls
  unsigned* cnt;       // [U + 1] arrival counters, zero between calls
  rails_final_t fin;
  int do_final;
  int64_t* rail_base;
  int64_t* rail_total;
  size_t res_off;      // byte offset of the shared result buffer (res_smem)
  size_t ev_off;       // byte offset of the eval arrays in shared memory
  int res_smem;        // chain results in shared memory, else res_g
  int* err;
};

// number of the node-global full chunks 0..x-1 that land on rail j (i mod N == j)
__device__ __forceinline__ long long full_on_rail(long long x, int N, int j) {
  long long q;
  int r;
  divmod_n(x, N, q, r);
  return q + (j < r ? 1 : 0);
}

template <typename KeyT, int NT, bool SMEM, bool EVAL>
__global__ void __launch_bounds__(NODE_MAX_THREADS) k_node(NodeArgs a) {
  using IdxT = typename std::conditional<SMEM, uint16_t, uint32_t>::type;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ long long scan_scratch[33];
  __shared__ int hist[(NODE_MAX_THREADS / 32) * 256];
  __shared__ int sc[256];
  __shared__ uint32_t red32[64];
  __shared__ long long sL[32], sSe[32], sSu[32];
  __shared__ int s_last;
  __shared__ RunDesc s_runs[NODE_MAX_RUNS];
  __shared__ int s_nrun;

  const long long seg = blockIdx.x;
  const long long NG = a.NG;
  const int N = NT ? NT : a.N;
  const int M = a.M;
  const long long C = a.C;
  const ChunkDiv cd{C, a.cshift};
  const int64_t* __restrict__ mg = a.msg + seg * NG;
  const long long G = NG / N;
  const long long u = seg / a.nd;
  const int d = a.d0 + (int)(seg % a.nd);
  const long long MN = (long long)M * N;

  KeyT *kA, *kB;
  IdxT *iA, *iB;
  {
    uint8_t* base;
    if constexpr (SMEM) base = smem;
    else base = a.scratch + seg * (NG * (2 * sizeof(KeyT) + 2 * sizeof(IdxT)) + 64);
    kA = (KeyT*)base;
    kB = kA + NG;
    iA = (IdxT*)(kB + NG);
    iB = iA + NG;
  }
  // eval arrays (EVAL): block starts P[G+1] (int64), then u32 arrays of MN:
  // R lo/hi (full chunks + remainders), ECMP lo/hi, uniform remainder histogram
  // cU[f][r]; then uniform quotient sums lo/hi per destination node [M]
  long long* sP = nullptr;
  unsigned *aRlo = nullptr, *aRhi = nullptr, *aElo = nullptr, *aEhi = nullptr, *cU = nullptr,
           *aQlo = nullptr, *aQhi = nullptr;
  uint8_t* sPr = nullptr;  // r of each block start (phase C)
  if constexpr (EVAL) {
    sP = (long long*)(smem + a.ev_off);
    aRlo = (unsigned*)(sP + G + 1);
    aRhi = aRlo + MN;
    aElo = aRhi + MN;
    aEhi = aElo + MN;
    cU = aEhi + MN;
    aQlo = cU + MN;
    aQhi = aQlo + M;
    sPr = reinterpret_cast<uint8_t*>(aQhi + M);
    for (long long i = threadIdx.x; i < MN; i += blockDim.x) aElo[i] = aEhi[i] = cU[i] = 0u;
    for (int i = threadIdx.x; i < M; i += blockDim.x) aQlo[i] = aQhi[i] = 0u;
    __syncthreads();
  }
  // launched with programmatic stream serialization: everything above overlapped the
  // histogram kernel's tail; its outputs (msg) are read from here on
  NODE_T(0);
  pdl_wait();

  NODE_T(1);
  NODE_TC(0);
  // ---- phase A: full_base scan + remainder compaction (+ ECMP and uniform sums)
  // Tiles of blockDim * IPT messages, each thread owning IPT consecutive messages:
  // its loads are all in flight at once, one block scan per tile.
  constexpr int IPT = 8;
  long long carry_full = 0;
  int carry_rem = 0;
  KeyT kor = 0, kand = (KeyT)~(KeyT)0;
  const int lo = d * N, hi = d * N + N;  // the source node's own GPUs (R#2)
  int64_t* __restrict__ fbg = a.s.full_base + seg * NG;
  const bool vec = aligned32(mg) && aligned32(fbg);  // 256-bit accesses (ld8/st8_s64)
  bool bad_range = false, bad_ovf = false;  // flagged once after the pass
  for (long long t0 = 0; t0 < NG; t0 += (long long)blockDim.x * IPT) {
    const long long m0 = t0 + (long long)threadIdx.x * IPT;
    const bool whole = vec && m0 + IPT <= NG;
    long long B[IPT];
    if (whole) {
      ld8_s64(mg + m0, B);
    } else {
#pragma unroll
      for (int j = 0; j < IPT; ++j) B[j] = m0 + j < NG ? mg[m0 + j] : 0;
    }
    long long snf = 0;
    int srem = 0;
    long long nfv[IPT];
    // destination GPU h = m mod G and source GPU g = m div G of the first item, then
    // stepped (one division per thread and tile instead of one per message)
    const int h0 = (int)((unsigned long long)m0 % (unsigned long long)G);
    const int g0 = (int)((unsigned long long)m0 / (unsigned long long)G);
    int h = h0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      // negative bytes, or bytes to a GPU of the source node (R#2), are invalid
      const bool inval = B[j] < 0 || (B[j] != 0 && h >= lo && h < hi);
      bad_range |= inval;
      if (inval) B[j] = 0;
      if (++h >= G) h -= (int)G;
      nfv[j] = cd.div(B[j]);
      bad_ovf |= nfv[j] >= (1LL << 40);
      snf += nfv[j];
      srem += (B[j] - nfv[j] * C) > 0;
    }
    if (t0 == 0) NODE_T(14);
    long long tot;
    const long long ex = block_excl_scan((snf << 16) | srem, scan_scratch, &tot);
    if (t0 == 0) NODE_T(15);
    long long fb = carry_full + (ex >> 16);
    int pos = carry_rem + (int)(ex & 0xffff);
    h = h0;
    int g = g0;
    long long fbv[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const long long m = m0 + j;
      if (m >= NG) break;
      const long long nf = nfv[j];
      const long long rem = B[j] - nf * C;
      fbv[j] = fb;
      if (!whole) fbg[m] = fb;
      if constexpr (EVAL) {
        if (h % N == 0) sP[m / N] = fb;  // block (g, f = h/N) starts here
        if (B[j] > 0) {  // own-node and invalid entries were zeroed above
          // the ECMP rail (R#13-R#14) and the uniform split (R#41) of the message,
          // as fire-and-forget split shared sums (add_split20)
          const int f = h / N;
          const int e = ecmp_rail(a.seed, (long long)d * N + g, h, N);
          add_split20(&aElo[f * N + e], &aEhi[f * N + e], (unsigned long long)B[j]);
          long long qb;
          int rb;
          divmod_n(B[j], N, qb, rb);
          if (qb) add_split20(&aQlo[f], &aQhi[f], (unsigned long long)qb);
          if (rb) atomicAdd(&cU[f * N + rb], 1u);
        }
      }
      fb += nf;
      if (rem > 0) {
        const KeyT key = (KeyT)(C - 1 - rem);
        kA[pos] = key;
        iA[pos] = (IdxT)m;
        kor |= key;
        kand &= key;
        ++pos;
      }
      if (++h >= G) {
        h -= (int)G;
        ++g;
      }
    }
    if (whole) st8_s64(fbg + m0, fbv);
    carry_full += tot >> 16;
    carry_rem += (int)(tot & 0xffff);
  }
  if (bad_range) flag_error(a.err, ERR_RANGE);
  if (bad_ovf) flag_error(a.err, ERR_OVERFLOW);
  NODE_T(16);
  {
    uint32_t o = kor, an = kand;
    block_reduce_or_and(o, an, red32);
    kor = (KeyT)o;
    kand = (KeyT)an;
  }
  NODE_T(17);
  const long long nf_node = carry_full;
  const int n = carry_rem;
  if (threadIdx.x == 0) {
    a.s.n_full[seg] = nf_node;
    a.s.n_rem[seg] = n;
    if constexpr (EVAL) sP[G] = nf_node;
  }
  __syncthreads();

  NODE_T(2);
  // ---- phase B: stable radix sort of the remainder keys
  const int which =
      radix_sort_narrow<KeyT, IdxT>(kA, iA, kB, iB, n, kor, kand, a.nbits, hist, sc);
  const KeyT* ks = which ? kB : kA;
  const IdxT* is = which ? iB : iA;
  IdxT* inv = which ? iA : iB;  // inverse permutation: message -> sorted position
  constexpr IdxT NONE = (IdxT)~(IdxT)0;
  for (int m = threadIdx.x; m < (int)NG; m += blockDim.x) inv[m] = NONE;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) inv[is[i]] = (IdxT)i;

  NODE_T(3);
  NODE_TC(1);
  // ---- phase C: warp 0 runs the LPT chain; the other warps add the full chunks
  uint64_t* res = a.res_smem ? (uint64_t*)(smem + a.res_off) : a.res_g + seg * NG;
  if (threadIdx.x < 32) {
    NODE_T(4);
    if constexpr (NT != 0) {
#ifdef RAILS_CHAIN_TWICE  // debug: the same chain code twice (cold, then warm i-cache)
#pragma unroll 1
      for (int rep = 0; rep < 2; ++rep) {
        if (rep == 1) NODE_T(24);
        lpt_chain_net<NT, KeyT>(ks, n, C, nf_node, res, sL,
                                RunList{s_runs, NODE_MAX_RUNS, &s_nrun});
        __syncwarp();
      }
#else
      lpt_chain_net<NT, KeyT>(ks, n, C, nf_node, res, sL,
                              RunList{s_runs, NODE_MAX_RUNS, &s_nrun});
#endif
    } else {
      const long long L = lpt_chain_generic<KeyT>(ks, n, N, C, nf_node, res, a.err);
      if (threadIdx.x < N) sL[threadIdx.x] = L;
    }
    __syncwarp();
    NODE_T(9);
    if (threadIdx.x < N) a.s.send_load[seg * N + threadIdx.x] = sL[threadIdx.x];
  } else if constexpr (EVAL) {
    // full chunks: block boundary t (= g*M + f) starts at node-global full index
    // sP[t] = q*N + r; rail j of block t receives (q_b - q_a) + [j < r_b] - [j < r_a]
    for (int t = threadIdx.x - 32; t <= (int)G; t += blockDim.x - 32) {
      long long q;
      int r;
      divmod_n(sP[t], N, q, r);
      sP[t] = q;
      sPr[t] = (uint8_t)r;
    }
    asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x - 32) : "memory");  // workers only
    NODE_TW(13);  // workers' block starts converted
    if constexpr (NT != 0) {
      // thread per destination node f: the q difference is the same for every rail,
      // the [j < r] terms for all NT rails in registers
      for (int f = threadIdx.x - 32; f < M; f += blockDim.x - 32) {
        long long qs = 0;
        int cnt[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) cnt[j] = 0;
        if (f != d) {
          for (int g = 0; g < NT; ++g) {
            const long long ia = (long long)g * M + f;
            qs += sP[ia + 1] - sP[ia];
            const int rb = sPr[ia + 1], ra = sPr[ia];
#pragma unroll
            for (int j = 0; j < NT; ++j) cnt[j] += (j < rb ? 1 : 0) - (j < ra ? 1 : 0);
          }
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const unsigned long long v = f != d ? (unsigned long long)((qs + cnt[j]) * C) : 0ull;
          aRlo[f * NT + j] = (unsigned)(v & 0xFFFFFull);
          aRhi[f * NT + j] = (unsigned)(v >> 20);
        }
      }
    } else {
      for (long long t = threadIdx.x - 32; t < MN; t += blockDim.x - 32) {
        const int f = (int)(t / N), j = (int)(t - (long long)f * N);
        long long full = 0;
        if (f != d) {
          for (int g = 0; g < N; ++g) {
            const long long ia = (long long)g * M + f;
            full += (sP[ia + 1] - sP[ia]) + (j < sPr[ia + 1] ? 1 : 0) - (j < sPr[ia] ? 1 : 0);
          }
        }
        const unsigned long long v = (unsigned long long)(full * C);
        aRlo[t] = (unsigned)(v & 0xFFFFFull);
        aRhi[t] = (unsigned)(v >> 20);
      }
    }
  }
  __syncthreads();

  NODE_T(5);
  NODE_TC(2);
  // ---- phase D: the chain's deferred runs, QP map (optional), expand, remainders
  // into R_d
  if constexpr (NT != 0) {
    lpt_runs_expand<NT>(s_runs, s_nrun, res);
    __syncthreads();
  }
  if (a.rem_qp) qp_rank_block(N, a.Q, nf_node, n, res, a.qp_g + seg * NG);
  const unsigned NGu = (unsigned)NG, Gu = (unsigned)G;  // N*G < 2^26 (M*N <= 2^20, N <= 32)
  for (unsigned m = threadIdx.x; m < NGu; m += blockDim.x) {
    const IdxT p = inv[m];
    int8_t r = -1;
    long long o = 0;
    int32_t q = -1;
    if (p != NONE) {
      const uint64_t v = res[p];
      r = (int8_t)(v >> 56);
      o = (long long)(v & (uint64_t)OFF_MASK);
      if (a.rem_qp) q = (int32_t)a.qp_g[seg * NG + p];
      if constexpr (EVAL) {
        const int f = (int)((m % Gu) / (unsigned)N);
        add_split20(&aRlo[f * N + r], &aRhi[f * N + r],
                    (unsigned long long)(C - 1 - (long long)ks[p]));
      }
    }
    a.s.rem_rail[seg * NG + m] = r;
    a.s.rem_off[seg * NG + m] = o;
    if (a.rem_qp) a.rem_qp[seg * NG + m] = q;
  }
  if constexpr (!EVAL) return;

  NODE_T(6);
  // ---- phase E: this node's receive contributions into the unit's accumulator
  __syncthreads();
  const long long rsl = RAILS_RED_SUM_LEN(M, N);
  const long long rec = rsl + RAILS_RED_MAX_LEN;
  const RedLayout RL{MN, M};
  unsigned long long* acc = (unsigned long long*)(a.acc + u * rec);
  // thread per (f, j): R, R_e, R_u into the unit's accumulator.  When N divides the
  // block, every thread keeps one rail j (register partials of S_e, S_u, reduced
  // below); when N divides 32, the N rails of one f sit in consecutive lanes and the
  // column sum is a shuffle reduction.  Otherwise shared split atomics / a loop.
  const bool jfix = (blockDim.x % N) == 0;
  const bool wlanes = (32 % N) == 0;
  __shared__ unsigned sEU[4][32];  // S_e lo/hi, S_u lo/hi when !jfix
  if (threadIdx.x < 32) sEU[0][threadIdx.x] = sEU[1][threadIdx.x] = sEU[2][threadIdx.x] =
      sEU[3][threadIdx.x] = 0u;
  __syncthreads();
  unsigned long long pe = 0, pu = 0;
  for (int t0 = 0; t0 < (int)MN; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    const bool act = t < (int)MN;
    const int f = act ? t / N : 0, j = act ? t - f * N : 0;
    unsigned long long R = 0, Re = 0, Ru = 0;
    if (act) {
      R = get_split20(aRlo[t], aRhi[t]);
      Re = get_split20(aElo[t], aEhi[t]);
      Ru = get_split20(aQlo[f], aQhi[f]);
      for (int r = j + 1; r < N; ++r) Ru += cU[f * N + r];
      if (R) atomicAdd(acc + RL.R() + t, R);
      if (Re) atomicAdd(acc + RL.Re() + t, Re);
      if (Ru) atomicAdd(acc + RL.Ru() + t, Ru);
    }
    if (jfix) {
      pe += Re;
      pu += Ru;
    } else if (act) {
      if (Re) add64_split(&sEU[0][j], &sEU[1][j], Re);
      if (Ru) add64_split(&sEU[2][j], &sEU[3][j], Ru);
    }
    if (wlanes) {
      unsigned long long v = R;
      for (int o = 1; o < N; o <<= 1) v += __shfl_xor_sync(FULL, v, o);
      if (act && j == 0 && v) atomicAdd(acc + RL.col() + f, v);
    }
  }
  if (!wlanes) {
    for (int f = threadIdx.x; f < M; f += blockDim.x) {
      unsigned long long cf = 0;
      for (int j = 0; j < N; ++j)
        cf += get_split20(aRlo[f * N + j], aRhi[f * N + j]);
      if (cf) atomicAdd(acc + RL.col() + f, cf);
    }
  }
  unsigned long long* part = reinterpret_cast<unsigned long long*>(hist);  // free after the sort
  if (jfix) {
    part[threadIdx.x] = pe;
    part[NODE_MAX_THREADS + threadIdx.x] = pu;
  }
  __syncthreads();
  if (threadIdx.x < N) {  // S_e, S_u of this node per rail j
    const int j = threadIdx.x;
    unsigned long long se = 0, su = 0;
    if (jfix) {
      for (int t = j; t < (int)blockDim.x; t += N) {
        se += part[t];
        su += part[NODE_MAX_THREADS + t];
      }
    } else {
      se = ((unsigned long long)sEU[1][j] << 32) | sEU[0][j];
      su = ((unsigned long long)sEU[3][j] << 32) | sEU[2][j];
    }
    sSe[j] = (long long)se;
    sSu[j] = (long long)su;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const long long s = lane < N ? sL[lane] : 0, se = lane < N ? sSe[lane] : 0,
                    su = lane < N ? sSu[lane] : 0;
    if (lane < N) {
      a.e.S[seg * N + lane] = s;
      a.e.S_e[seg * N + lane] = se;
      a.e.S_u[seg * N + lane] = su;
    }
    const long long total = warp_sum(s), total_e = warp_sum(se);
    const long long mx = warp_max(s), mxe = warp_max(se), mxu = warp_max(su);
    double mse, nmse;
    warp_mse(s, N, total, &mse, &nmse);
    if (lane == 0) {
      a.e.mse[seg] = mse;
      a.e.nmse[seg] = nmse;
      if (total) atomicAdd(acc + RL.tot(), (unsigned long long)total);
      if (total_e) atomicAdd(acc + RL.tot() + 1, (unsigned long long)total_e);
      long long* am = (long long*)acc + rsl;
      atomicMax(am + RMAX_S, mx);
      atomicMax(am + RMAX_SE, mxe);
      atomicMax(am + RMAX_ROW, total);  // row sum of node d = its inter-node bytes
      atomicMax(am + RMAX_SU, mxu);
    }
  }

  NODE_T(7);
  NODE_TC(3);
  // ---- phase F: the unit's last CTA publishes (and finalizes); the grid's last
  // CTA computes the rail offsets
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // release: this CTA's accumulator adds (ordered by the barrier)
    const bool last = atomicAdd(&a.cnt[u], 1u) == (unsigned)(a.nd - 1);
    if (last) __threadfence();  // acquire: every CTA's adds, for the whole CTA (barrier)
    s_last = last;
  }
  __syncthreads();
  if (s_last) {
    NODE_TL(12);
    NODE_TL(18);
    // publish the unit's record (red_sum / red_max), re-zero the accumulator, and
    // take the maxima the finalize needs in the same pass
    int64_t* rs = a.e.red_sum + u * rsl;
    int64_t* rm = a.e.red_max + u * RAILS_RED_MAX_LEN;
    long long mx[4] = {0, 0, 0, 0};  // max R, R_e, R_u, colsum
    for (long long i0 = threadIdx.x; i0 < rec; i0 += 4LL * blockDim.x) {
      long long v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long i = i0 + (long long)q * blockDim.x;
        v[q] = i < rec ? (long long)__ldcg((const long long*)acc + i) : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long i = i0 + (long long)q * blockDim.x;
        if (i >= rec) break;
        if (i < rsl) rs[i] = v[q];
        else rm[i - rsl] = v[q];
        acc[i] = 0;
        const int cls = i < MN ? 0 : i < 2 * MN ? 1 : i < 3 * MN ? 2 : i < 3 * MN + M ? 3 : 4;
        if (cls < 4) mx[cls] = max(mx[cls], v[q]);
      }
    }
    if (threadIdx.x == 0) a.cnt[u] = 0;
    NODE_TL(19);
    __shared__ long long s_mx[4][NODE_MAX_THREADS / 32];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long w = warp_max(mx[q]);
      if ((threadIdx.x & 31) == 0) s_mx[q][threadIdx.x >> 5] = w;
    }
    __syncthreads();
    NODE_TL(30);
    if (threadIdx.x == 0 && a.do_final) {
      // (the record's maxima and totals as this CTA just stored them; a four-warp
      // finalize from a shared copy measured ~1 us slower)
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
#pragma unroll
        for (int q = 0; q < 4; ++q) s_mx[q][0] = max(s_mx[q][0], s_mx[q][w]);
      long long rmv[RAILS_RED_MAX_LEN];
#pragma unroll
      for (int q = 0; q < RAILS_RED_MAX_LEN; ++q) rmv[q] = rm[q];
      finalize_unit(u, N, a.R2, s_mx[0][0], s_mx[1][0], s_mx[2][0], s_mx[3][0], rmv,
                    rs[RL.tot()], rs[RL.tot() + 1], a.fin);
    }
    NODE_TL(10);
    if (a.rail_base && (int)gridDim.x == a.nd) {  // one unit: this CTA is also the grid's last
      block_rail_offsets<true>((long long)gridDim.x * N, a.s.send_load, a.rail_base,
                               a.rail_total);
      NODE_TL(11);
    }
  }
  if (a.rail_base && (int)gridDim.x != a.nd) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const bool last = atomicAdd(&a.cnt[a.U], 1u) == (unsigned)(gridDim.x - 1);
      if (last) __threadfence();
      s_last = last;
    }
    __syncthreads();
    if (s_last) {
      block_rail_offsets<true>((long long)gridDim.x * N, a.s.send_load, a.rail_base,
                               a.rail_total);
      if (threadIdx.x == 0) a.cnt[a.U] = 0;
      NODE_TL(11);
    }
  }
  NODE_T(8);
}

// ---------------------------------------------------------------- host side
static int ceil_log2(long long x) {  // bits needed for values 0..x-1
  int b = 0;
  while ((1LL << b) < x) ++b;
  return b;
}

struct NodePlan {
  bool smem_sort, k16, res_smem, eval_fused;
  int threads;
  size_t sort_bytes, res_off, ev_off, smem;
};

// Shared-memory plan of the fused kernel for N*G messages per node.
static NodePlan node_plan(int M, int N, long long C, bool eval, long long nseg, int num_sms) {
  const long long G = (long long)M * N, NG = (long long)N * G;
  NodePlan p{};
  constexpr size_t DYN_LIMIT = 200 * 1024;  // + ~20 KiB static stays under 227 KiB
  const size_t ev_bytes = (size_t)(G + 1) * 8 + (size_t)G * 4 * 5 + (size_t)M * 8 + (size_t)G + 16;
  p.eval_fused = eval && ev_bytes <= 96 * 1024;
  const bool k16 = C <= 65536;
  const size_t sort_smem = (size_t)NG * 2 * ((k16 ? 2 : 4) + 2);
  p.smem_sort = NG <= NODE_SMEM_ITEMS &&
                sort_smem + (p.eval_fused ? ev_bytes + 32 : 0) <= DYN_LIMIT;
  p.k16 = p.smem_sort && k16;
  // few segments (C3: 64 on 148 SMs): the node's latency is the step's, so give each
  // CTA the most threads; many segments: 256 (128 registers each -> 2 CTAs per SM)
  p.threads = NG <= 1024 ? 128 : (NG <= 8192 ? 256 : NODE_MAX_THREADS);
  if (nseg <= num_sms && NG >= 2048) p.threads = NODE_MAX_THREADS;
  p.sort_bytes = p.smem_sort ? sort_smem : 0;
  size_t off = (p.sort_bytes + 15) & ~(size_t)15;
  if (p.eval_fused) {
    p.ev_off = off;
    off = (off + ev_bytes + 15) & ~(size_t)15;
  }
  // chain results in shared memory when the CTA still fits twice per SM
  const size_t res_bytes = (size_t)NG * 8;
  p.res_smem = off + res_bytes <= 110 * 1024;
  if (p.res_smem) {
    p.res_off = off;
    off += res_bytes;
  }
  p.smem = off;
  if (p.smem < 16) p.smem = 16;
  return p;
}

// workspace: [256 B header][acc: U x rec int64][counters: U + 1 u32, 256-aligned]
//            [res_g u64: nseg x NG][qp_g u32][w_g u32][inv_g i32 (k_chains)]
//            [sort spill when N*G > 4096]
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct NodeWs {
  int64_t* acc;
  unsigned* cnt;
  uint64_t* res_g;
  uint32_t* qp_g;
  uint32_t* w_g;    // k_chains: sorted sizes
  int32_t* inv_g;   // k_chains: inverse permutation
  uint8_t* scratch;
  size_t bytes;
};

static NodeWs node_ws(void* ws, int U, int nd, int M, int N) {
  const long long NG = (long long)N * M * N, nseg = (long long)U * nd;
  const long long rec = RAILS_RED_SUM_LEN(M, N) + RAILS_RED_MAX_LEN;
  uint8_t* b = (uint8_t*)ws;
  NodeWs w{};
  size_t o = 256;
  w.acc = (int64_t*)(b + o);
  o = al256(o + (size_t)U * rec * 8);
  w.cnt = (unsigned*)(b + o);
  o = al256(o + (size_t)(U + 1) * 4);
  w.res_g = (uint64_t*)(b + o);
  o = al256(o + (size_t)nseg * NG * 8);
  w.qp_g = (uint32_t*)(b + o);
  o = al256(o + (size_t)nseg * NG * 4);
  w.w_g = (uint32_t*)(b + o);
  o = al256(o + (size_t)nseg * NG * 4);
  w.inv_g = (int32_t*)(b + o);
  o = al256(o + (size_t)nseg * NG * 4);
  w.scratch = b + o;
  if (NG > NODE_SMEM_ITEMS / 4) o += (size_t)nseg * (NG * (2 * 4 + 2 * 4) + 64);
  w.bytes = o;
  return w;
}

void schedule_workspace_ptrs(void* ws, int U, int nd, int M, int N, int64_t** acc,
                             unsigned** cnt, uint64_t** res) {
  const NodeWs w = node_ws(ws, U, nd, M, N);
  *acc = w.acc;
  *cnt = w.cnt;
  *res = w.res_g;
}

size_t schedule_workspace_bytes(int U, int nd, int M, int N) {
  return node_ws(nullptr, U, nd, M, N).bytes;
}

template <typename KeyT, int NT, bool SMEM, bool EVAL>
static cudaError_t launch_k(const LaunchCtx& c, const NodePlan& p, unsigned grid,
                            const NodeArgs& a) {
  auto kern = k_node<KeyT, NT, SMEM, EVAL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)p.smem);
  if (e != cudaSuccess) return e;
  // PDL: the CTAs may be scheduled while the previous kernel (the histogram) runs and
  // wait for it in pdl_wait(), hiding this launch's latency
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(p.threads);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, a);
  count_launch(1);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <bool EVAL>
static cudaError_t launch_eval_t(const LaunchCtx& c, const NodePlan& p, unsigned grid,
                                 const NodeArgs& a, int N) {
  const bool net = N == 8 && a.C < (1LL << 23);
  if (p.smem_sort) {
    if (p.k16)
      return net ? launch_k<uint16_t, 8, true, EVAL>(c, p, grid, a)
                 : launch_k<uint16_t, 0, true, EVAL>(c, p, grid, a);
    return net ? launch_k<uint32_t, 8, true, EVAL>(c, p, grid, a)
               : launch_k<uint32_t, 0, true, EVAL>(c, p, grid, a);
  }
  if constexpr (EVAL) {
    return cudaErrorInvalidConfiguration;  // the fused evaluation needs the sort in smem
  } else {
    return net ? launch_k<uint32_t, 8, false, false>(c, p, grid, a)
               : launch_k<uint32_t, 0, false, false>(c, p, grid, a);
  }
}

// rails_lpt_schedule[_qp] (ev == nullptr) and rails_schedule_eval.  Returns
// *fused = false when the evaluation could not be fused (the caller then runs
// rails_eval's kernel).
cudaError_t launch_node(const LaunchCtx& c, int U, int nd, int d0, int M, int N, long long C,
                        uint64_t seed, double R2, const int64_t* msg, const rails_sched_t& s,
                        void* ws, int32_t* rem_qp, int qps_per_rail, const rails_eval_t* ev,
                        const rails_final_t* fin, int64_t* rail_base, int64_t* rail_total,
                        bool* fused) {
  const long long NG = (long long)N * M * N, nseg = (long long)U * nd;
  const NodeWs w = node_ws(ws, U, nd, M, N);
  const int cshift = (C & (C - 1)) == 0 ? ceil_log2(C) : -1;
  const int nbits = ceil_log2(C > 1 ? C - 1 : 1) + 1;
  if (fused) *fused = false;
  if (nseg > 2LL * c.num_sms) {
    // many segments (C2's 16 000, a C4 iteration's 4 096): per-phase kernels at their
    // own occupancy measured faster than one CTA walking every phase (k_chains.cu)
    // With an evaluation (and no QP map) the expand pass runs inside it: one pass over
    // the messages instead of two.
    const bool ex = ev != nullptr && rem_qp == nullptr;
    cudaError_t e = launch_chains(c, U, nd, d0, M, N, C, msg, s, w.res_g, w.qp_g, w.w_g,
                                  w.inv_g, w.scratch, rem_qp, qps_per_rail, cshift, nbits, ex);
    if (e != cudaSuccess || !ex) return e;
    if ((e = launch_eval(c, U, nd, d0, M, N, C, seed, msg, s, *ev, w.inv_g, w.res_g)) !=
        cudaSuccess)
      return e;
    if (fin && (e = launch_finalize(c, U, M, N, R2, ev->red_sum, ev->red_max, *fin)) !=
                   cudaSuccess)
      return e;
    if (rail_base &&
        (e = launch_rail_offsets(c, (long long)U * nd * N, s.send_load, rail_base,
                                 rail_total)) != cudaSuccess)
      return e;
    if (fused) *fused = true;  // evaluated (and finalized / offset) here
    return cudaSuccess;
  }
  NodePlan p = node_plan(M, N, C, ev != nullptr, nseg, c.num_sms);
  if (p.eval_fused && !p.smem_sort) {
    // the sort would spill to global memory to make room for the evaluation: the
    // schedule alone (sort in shared memory) plus rails_eval's kernel measured faster
    p = node_plan(M, N, C, false, nseg, c.num_sms);
  }
  if (fused) *fused = p.eval_fused;
  NodeArgs a{};
  a.msg = msg;
  a.NG = NG;
  a.M = M;
  a.N = N;
  a.d0 = d0;
  a.nd = nd;
  a.U = U;
  a.C = C;
  a.cshift = cshift;
  a.nbits = nbits;
  a.seed = seed;
  a.R2 = R2;
  a.s = s;
  a.rem_qp = rem_qp;
  a.Q = qps_per_rail;
  a.res_g = w.res_g;
  a.qp_g = w.qp_g;
  a.scratch = w.scratch;
  a.acc = w.acc;
  a.cnt = w.cnt;
  a.res_off = p.res_off;
  a.res_smem = p.res_smem ? 1 : 0;
  a.ev_off = p.ev_off;
  a.err = c.err;
  if (p.eval_fused) {
    a.e = *ev;
    if (fin) {
      a.fin = *fin;
      a.do_final = 1;
    }
    a.rail_base = rail_base;
    a.rail_total = rail_total;
    return launch_eval_t<true>(c, p, (unsigned)nseg, a, N);
  }
  return launch_eval_t<false>(c, p, (unsigned)nseg, a, N);
}

}  // namespace rails
