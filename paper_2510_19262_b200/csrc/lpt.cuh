// lpt.cuh -- a4: the LPT assignment chain of one (unit, node) (Alg. 2 step 3,
// P:634-640), run by one warp over the node's remainder chunks already sorted by
// size descending (R#4), and the QP map of Alg. 2 step 4 (qp_rank_block).  Included
// by k_node.cu and k_chains.cu.
//
// Full chunks are never materialised (k_node.cu header): they form the prefix of
// the LPT order and are dealt round-robin, so the chain starts from the closed-form
// LoadState after n_full chunks: rails 0..r-1 hold C*(q+1), the others C*q
// (q = n_full div N, r = n_full mod N).  Each remainder goes to the lowest-index
// argmin rail (R#5) at offset LoadState[j*] (R#19), then LoadState[j*] += w.
//
// Two chains:
//  * lpt_chain_net (N in {2,4,8,16}, C < 2^23): every lane holds the N rail keys
//    (rel << 5) | rail SORTED in registers, so the argmin is K[0] (lowest rail on
//    ties: the rail is the low key bits) and an assignment is one compare/select
//    merge.  Loads are relative to an exact int64 `base`, rebased when the minimum
//    passes 2^23.  Runs of equal sizes (routing traffic has only C / row_bytes
//    distinct remainder sizes) are dealt by an exact closed form: written by all 32
//    lanes, or -- given a RunList (the fused node kernel) -- recorded as (start
//    state, length) and written by the whole CTA after the chain; aligned groups of
//    8 equal sizes by a warp scan; other items 8 at a time.
//  * lpt_chain_generic (any N <= 32, any C): lane j holds rail j's load; the
//    argmin with lowest-index tie is one redux.sync.min on (rel << 5) | j when
//    C < 2^26, else a 64-bit butterfly over (load, lane).
// Results are written in SORTED order, packed rail << 56 | offset.
#pragma once

#include <climits>

#include "common.cuh"

#ifndef LPT_CLK
#define LPT_CLK() 0LL  // debug builds: clock64(), sums in registers (k_node.cu)
#define LPT_ACC(k, t0) \
  do {                 \
  } while (0)
#define LPT_ACC_DECL
#define LPT_ACC_FLUSH
#endif
#ifndef LPT_COUNT
#define LPT_COUNT(i) \
  do {               \
  } while (0)
#endif

namespace rails {

constexpr long long OFF_MASK = (1LL << 56) - 1;
__device__ __forceinline__ uint64_t pack_res(unsigned rail, long long off) {
  return ((uint64_t)rail << 56) | ((uint64_t)off & (uint64_t)OFF_MASK);
}

// One network step: K sorted ascending holds the N rail keys (rel << 5) | rail; the
// chunk of size w goes to K[0]'s rail at offset base + rel, and K[0] + (w << 5) is
// merged back.
template <int NT>
__device__ __forceinline__ uint64_t lpt_step_v(uint32_t (&K)[NT], uint32_t w, long long base) {
  const uint32_t head = K[0];
  const uint32_t x = head + (w << 5);
  const uint64_t res = pack_res(head & 31u, base + (long long)(head >> 5));
  bool cprev = true;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const bool c = (j < NT - 1) ? (K[j + 1] < x) : false;
    const uint32_t a = (j < NT - 1) ? K[j + 1] : 0u;
    const uint32_t b = (j > 0) ? K[j] : 0u;
    K[j] = c ? a : (cprev ? x : b);
    cprev = c;
  }
  return res;
}

// eight packed results -> four 16-byte stores (out is 64-byte aligned)
__device__ __forceinline__ void store8(uint64_t* __restrict__ out, const uint64_t (&r)[8]) {
  ulonglong2* o = reinterpret_cast<ulonglong2*>(out);
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = make_ulonglong2(r[2 * q], r[2 * q + 1]);
}

template <int NT>
__device__ __forceinline__ void lpt_rebase(uint32_t (&K)[NT], long long& base) {
  const uint32_t mrel = K[0] >> 5;
  if (mrel > (1u << 23)) {
#pragma unroll
    for (int j = 0; j < NT; ++j) K[j] -= mrel << 5;
    base += mrel;
  }
}

__device__ __forceinline__ void cas_u32(uint32_t& a, uint32_t& b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

// NT = 8, 8 equal items, key spread K[7] - K[0] < 2w << 5.  The picks are the 8
// smallest slots (value, rail) among every rail's next slots rel + t*w; a rail's
// third slot is at key >= K[0] + 2(w << 5) > K[7], so the 8 smallest lie in
// {K_i} U {K_i + w}: a bitonic half-cleaner (K ascending against K + w descending)
// selects them, an 8-wide bitonic merge orders them.  K_i was taken iff
// K_i < K_{7-i} + w, and K_i + w iff K_i + w < K_{7-i}; the new keys
// K_i + (takes)*w are re-sorted (Batcher, 19 CAS).
__device__ __forceinline__ void lpt_merge8(uint32_t (&K)[8], uint32_t w,
                                           uint64_t (&out)[8], long long base) {
  const uint32_t W = w << 5;
  uint32_t L[8];
  int c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t a = K[i], b = K[7 - i] + W;
    L[i] = min(a, b);
    c[i] = (a < b) ? 1 : 0;  // K_i taken
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] += (K[i] + W < K[7 - i]) ? 1 : 0;  // K_i + w taken
#pragma unroll
  for (int i = 0; i < 4; ++i) cas_u32(L[i], L[i + 4]);
  cas_u32(L[0], L[2]); cas_u32(L[1], L[3]); cas_u32(L[4], L[6]); cas_u32(L[5], L[7]);
  cas_u32(L[0], L[1]); cas_u32(L[2], L[3]); cas_u32(L[4], L[5]); cas_u32(L[6], L[7]);
#pragma unroll
  for (int p = 0; p < 8; ++p) out[p] = pack_res(L[p] & 31u, base + (long long)(L[p] >> 5));
#pragma unroll
  for (int i = 0; i < 8; ++i) K[i] += (uint32_t)c[i] * W;
  cas_u32(K[0], K[1]); cas_u32(K[2], K[3]); cas_u32(K[4], K[5]); cas_u32(K[6], K[7]);
  cas_u32(K[0], K[2]); cas_u32(K[1], K[3]); cas_u32(K[4], K[6]); cas_u32(K[5], K[7]);
  cas_u32(K[1], K[2]); cas_u32(K[5], K[6]);
  cas_u32(K[0], K[4]); cas_u32(K[1], K[5]); cas_u32(K[2], K[6]); cas_u32(K[3], K[7]);
  cas_u32(K[2], K[4]); cas_u32(K[3], K[5]);
  cas_u32(K[1], K[2]); cas_u32(K[3], K[4]); cas_u32(K[5], K[6]);
}

// Eight consecutive sorted items.  If the largest key is below the smallest key plus
// w (K[NT-1] - K[0] < w << 5) and the 8 sizes are equal, LPT deals them one per rail
// in the current (load, rail) order -- after k of them the assigned rails sit at
// keys K_i + (w << 5) > K[NT-1] >= every unassigned key -- and the order is
// unchanged afterwards, all loads having grown by w.  So item p goes to K[p mod NT]
// at rel + (p div NT)*w and base += (8/NT)*w.  Keys stay below 2^32: rel < 2^23
// after a rebase, spread < 2w < 2^24, at most 8 network steps between rebases.
template <int NT>
__device__ __forceinline__ void lpt_group8_v(uint32_t (&K)[NT], const uint32_t (&w8)[8],
                                             uint64_t (&r)[8], long long& base) {
  const uint32_t w = w8[0];
  const uint32_t kspread = K[NT - 1] - K[0];
  if ((8 % NT) == 0 && w8[7] == w && kspread < (w << 5)) {
#pragma unroll
    for (int p = 0; p < 8; ++p)
      r[p] = pack_res(K[p % NT] & 31u,
                      base + (long long)(K[p % NT] >> 5) + (long long)(p / NT) * w);
    base += (long long)(8 / NT) * w;
  } else if (NT == 8 && w8[7] == w && kspread < (w << 6)) {
    lpt_merge8(reinterpret_cast<uint32_t(&)[8]>(K), w, r, base);
  } else {
#pragma unroll
    for (int p = 0; p < 8; ++p) r[p] = lpt_step_v<NT>(K, w8[p], base);
  }
  lpt_rebase<NT>(K, base);
}

// A whole run of n equal sizes w once K[NT-1] - K[0] < w << 5 (the cyclic case
// above, repeated): item t of the run goes to K[t mod NT] at rel + (t div NT)*w,
// so the warp writes the run in parallel, lane l taking t = l, l + 32, ... (NT
// divides 32, so t mod NT = l mod NT).  Afterwards rail K_i carries q = n div NT
// more items, plus one for i < n mod NT: the sorted keys become K[rr..NT-1] + q*w,
// K[0..rr-1] + (q+1)*w (still sorted, spread still < w).
template <int NT>
__device__ __forceinline__ void lpt_run_advance(uint32_t (&K)[NT], uint32_t w, int n,
                                                long long& base) {
  base += (long long)(n / NT) * w;
  // rotate left by s = n mod NT, the wrapped keys + w: composed from rotations by
  // 1, 2, 4, ... (each key wraps at most once since s < NT)
  const uint32_t W = w << 5;
  const int s = n % NT;
#pragma unroll
  for (int b = 1; b < NT; b <<= 1) {
    if (s & b) {
      uint32_t R[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) R[j] = (j < NT - b) ? K[j + b] : K[j + b - NT] + W;
#pragma unroll
      for (int j = 0; j < NT; ++j) K[j] = R[j];
    }
  }
  lpt_rebase<NT>(K, base);
}

template <int NT>
__device__ __forceinline__ void lpt_run_cyclic(uint32_t (&K)[NT], uint32_t w, int n, int lane,
                                               uint64_t* __restrict__ out, long long& base) {
  uint32_t kl = K[0];
#pragma unroll
  for (int j = 1; j < NT; ++j)
    if ((lane % NT) == j) kl = K[j];
  const long long lb = base + (long long)(kl >> 5);
  for (int t = lane; t < n; t += 32) out[t] = pack_res(kl & 31u, lb + (long long)(t / NT) * w);
  lpt_run_advance<NT>(K, w, n, base);
}

// A cyclic run whose writes are deferred: the chain records the run's start state
// (K, base) and moves on; afterwards the whole CTA writes the run by the same closed
// form (lpt_runs_expand), so the serial chain only pays for the runs' boundaries.
struct RunDesc {
  int start, n;
  uint32_t w, pad;
  long long base;
  uint32_t K[8];
};
struct RunList {
  RunDesc* d;  // shared memory, cap entries
  int cap;
  int* count;  // written by lane 0 when the chain ends
};

// Called by every thread of the block after the chain (and a barrier).
template <int NT>
__device__ __forceinline__ void lpt_runs_expand(const RunDesc* rl, int nrun,
                                                uint64_t* __restrict__ out) {
  for (int r = 0; r < nrun; ++r) {
    const int start = rl[r].start, n = rl[r].n;
    const uint32_t w = rl[r].w;
    const long long base = rl[r].base;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const uint32_t kl = rl[r].K[t % NT];
      out[start + t] = pack_res(kl & 31u, base + (long long)(kl >> 5) + (long long)(t / NT) * w);
    }
  }
}

// Sorted remainder sizes: w(i) = C - 1 - key[i] (keys ascending = sizes descending).
template <typename KeyT>
struct SortedSizes {
  const KeyT* key;
  uint32_t cm1;  // C - 1 (C < 2^32 on every chain that reads 32-bit sizes)
  __device__ __forceinline__ uint32_t operator()(int i) const { return cm1 - (uint32_t)key[i]; }
};

// First index >= i whose key differs from key[i] (the keys are sorted): 32-ary
// search by the warp, a prefix of the probes compares equal.
template <typename KeyT>
__device__ __forceinline__ int run_end(const KeyT* key, int i, int n, int lane) {
  const KeyT k0 = key[i];
  int lo = i + 1, hi = n;
  while (lo < hi) {
    const int step = (hi - lo + 31) >> 5;
    const int p = lo + lane * step;
    const bool eq = p < hi && key[p] == k0;
    const int c = __popc(__ballot_sync(FULL, eq));
    if (c == 0) break;  // key[lo] differs
    const int nhi = min(hi, lo + c * step);
    lo = lo + (c - 1) * step + 1;
    hi = nhi;
  }
  return lo;
}

// The sorted-register chain (one warp, every lane holds the same state).
template <int NT, typename KeyT>
__device__ void lpt_chain_net(const KeyT* __restrict__ key, int nr, long long C, long long nf,
                              uint64_t* __restrict__ res, long long* __restrict__ load_out,
                              RunList rl = RunList{nullptr, 0, nullptr}) {
  static_assert(NT <= 8, "RunDesc holds at most 8 rail keys");
  LPT_ACC_DECL
  int nrun = 0;
  const int lane = threadIdx.x & 31;
  const SortedSizes<KeyT> W{key, (uint32_t)(C - 1)};
  const long long q = nf / NT;
  const int r = (int)(nf - q * NT);
  long long base = C * q;
  uint32_t K[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {  // sorted by (load, rail): rails r..NT-1 (rel 0), then 0..r-1
    const int rail = (i < NT - r) ? (r + i) : (i - (NT - r));
    K[i] = (((i < NT - r) ? 0u : (uint32_t)C) << 5) | (uint32_t)rail;
  }
  int i = 0;
  const long long tchain = LPT_CLK();
  while (i < nr) {
    const uint32_t w = W(i);
    if (i + 32 <= nr && W(i + 31) == w) {
      // a run [i, e) of equal sizes: single steps until the cyclic condition holds,
      // then the closed form written by all lanes
      LPT_COUNT(0);
      long long tc = LPT_CLK();
      const int e = run_end(key, i, nr, lane);
      LPT_ACC(0, tc);
      tc = LPT_CLK();
      while (i < e && K[NT - 1] - K[0] >= (w << 5)) {
        LPT_COUNT(1);
        const uint64_t rv = lpt_step_v<NT>(K, w, base);
        if (lane == 0) res[i] = rv;
        lpt_rebase<NT>(K, base);
        ++i;
      }
      LPT_ACC(1, tc);
      tc = LPT_CLK();
      if (i < e) {
        if (nrun < rl.cap) {
          if (lane == 0) {
            RunDesc& R = rl.d[nrun];
            R.start = i;
            R.n = e - i;
            R.w = w;
            R.base = base;
#pragma unroll
            for (int j = 0; j < NT; ++j) R.K[j] = K[j];
          }
          ++nrun;
          lpt_run_advance<NT>(K, w, e - i, base);
        } else {
          lpt_run_cyclic<NT>(K, w, e - i, lane, res + i, base);
        }
      }
      LPT_ACC(2, tc);
      i = e;
    } else if ((8 % NT) == 0 && (i & 7) == 0 && i + 8 <= nr && W(i + 7) == w &&
               K[NT - 1] - K[0] < (w << 5)) {
      // window of up to 32 aligned groups, lane l taking group i + 8l: while every
      // group is 8 equal sizes w_l with K[NT-1] - K[0] < w_l << 5, each is dealt
      // cyclically, K is unchanged and base grows by (8/NT)*w_l, so the groups'
      // bases are an exclusive scan of those increments
      LPT_COUNT(2);
      const int at = i + 8 * lane;
      uint32_t a = 0, b = 0;
      if (at + 8 <= nr) {
        a = W(at);
        b = W(at + 7);
      }
      const bool ok = at + 8 <= nr && a == b && K[NT - 1] - K[0] < (a << 5);
      const unsigned bad = __ballot_sync(FULL, !ok);
      const int nok = bad ? __ffs(bad) - 1 : 32;  // >= 1: lane 0's group passed above
      const uint32_t inc = lane < nok ? (uint32_t)(8 / NT) * a : 0u;
      uint32_t ex = inc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, ex, o);
        if (lane >= o) ex += t;
      }
      const uint32_t tot = __shfl_sync(FULL, ex, 31);
      ex -= inc;
      if (lane < nok) {
        uint64_t rr[8];
        const long long bl = base + (long long)ex;
#pragma unroll
        for (int p = 0; p < 8; ++p)
          rr[p] = pack_res(K[p % NT] & 31u,
                           bl + (long long)(K[p % NT] >> 5) + (long long)(p / NT) * a);
        store8(res + at, rr);
      }
      base += (long long)tot;
      i += 8 * nok;
    } else if (i + 8 <= nr && (i & 7) == 0) {
      LPT_COUNT(3);
      uint32_t g8[8];
      uint64_t rr[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) g8[p] = W(i + p);
      lpt_group8_v<NT>(K, g8, rr, base);
      if (lane == 0) store8(res + i, rr);
      i += 8;
    } else {
      LPT_COUNT(1);
      const uint64_t rv = lpt_step_v<NT>(K, w, base);
      if (lane == 0) res[i] = rv;
      lpt_rebase<NT>(K, base);
      ++i;
    }
  }
  LPT_ACC(3, tchain);
  LPT_ACC_FLUSH
  if (lane == 0) {  // final LoadState by rail (K holds every rail once)
#pragma unroll
    for (int j = 0; j < NT; ++j) load_out[K[j] & 31u] = base + (long long)(K[j] >> 5);
    if (rl.count) *rl.count = nrun;
  }
}

// The generic chain: lane j < N holds rail j's load.  Returns lane's final load
// (lanes >= N: undefined).
template <typename KeyT>
__device__ long long lpt_chain_generic(const KeyT* __restrict__ key, int nr, int N, long long C,
                                       long long nf, uint64_t* __restrict__ res, int* err) {
  const int lane = threadIdx.x & 31;
  const long long q = nf / N;
  const int r = (int)(nf - q * N);
  if (C < (1LL << 26)) {
    // relative loads (spread <= C < 2^26 throughout), single redux.sync per step
    long long base = C * q;
    uint32_t rel = (lane < r) ? (uint32_t)C : 0u;
    for (int i0 = 0; i0 < nr; i0 += 32) {
      uint32_t wv = 0;
      if (i0 + lane < nr) wv = (uint32_t)(C - 1 - (long long)key[i0 + lane]);
      const int cnt = min(32, nr - i0);
      for (int b = 0; b < cnt; ++b) {
        const uint32_t wb = __shfl_sync(FULL, wv, b);
        const uint32_t kk = (lane < N) ? ((rel << 5) | (uint32_t)lane) : 0xffffffffu;
        const uint32_t kmin = __reduce_min_sync(FULL, kk);
        const int j = (int)(kmin & 31u);
        const uint32_t mrel = kmin >> 5;
        if (lane == j) {
          rel += wb;
          res[i0 + b] = pack_res((unsigned)j, base + mrel);
        }
        rel -= mrel;
        base += mrel;
      }
    }
    return base + rel;
  }
  // 64-bit loads, butterfly argmin over (load, lane)
  long long L = (lane < N) ? C * (q + (lane < r ? 1 : 0)) : LLONG_MAX;
  for (int i0 = 0; i0 < nr; i0 += 32) {
    long long wv = 0;
    if (i0 + lane < nr) wv = C - 1 - (long long)key[i0 + lane];
    const int cnt = min(32, nr - i0);
    for (int b = 0; b < cnt; ++b) {
      const long long wb = __shfl_sync(FULL, wv, b);
      long long v = L;
      int ix = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const long long ov = __shfl_xor_sync(FULL, v, o);
        const int oi = __shfl_xor_sync(FULL, ix, o);
        if (ov < v || (ov == v && oi < ix)) {
          v = ov;
          ix = oi;
        }
      }
      if (lane == ix) {
        res[i0 + b] = pack_res((unsigned)ix, v);
        L += wb;
      }
    }
  }
  if (lane < N && L < 0) flag_error(err, ERR_OVERFLOW);
  return L;
}

constexpr int QP_MAX_WARPS = 16;

// Alg. 2 step 4 (R#34): per-rail round-robin QP index in assignment
// order.  The chain results are in sorted (= assignment) order, so the QP of the
// p-th remainder is (full chunks on its rail + remainders on its rail before p) mod
// Q, full chunks being assigned first (i mod N).  Warp w owns a contiguous slice:
// pass 1 counts the slice's items per rail; the per-warp starting counters are an
// exclusive scan over warps (plus rail j's full chunks); pass 2 ranks each 32-item
// batch by rail with a ballot multi-split and advances the counters.
__device__ inline void qp_rank_block(int N, int Q, long long nf, int nr, const uint64_t* res,
                              uint32_t* out) {
  __shared__ unsigned cnt[QP_MAX_WARPS][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int per = (((nr + W - 1) / W) + 31) & ~31;
  const int beg = wid * per, end = min(nr, beg + per);
  const unsigned lt = lanemask_lt();
  cnt[wid][lane] = 0;
  __syncwarp();
  for (int p0 = beg; p0 < end; p0 += 32) {
    const int p = p0 + lane;
    const unsigned r = p < end ? (unsigned)(res[p] >> 56) : 0u;
    const unsigned peers = warp_match_nb<5>(r, p < end);
    if (p < end && (peers & lt) == 0) cnt[wid][r] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const unsigned q = (unsigned)Q;
  if (threadIdx.x < 32) {  // counters are kept modulo Q from here on (32-bit math)
    const int j = threadIdx.x;
    unsigned run = (unsigned)((nf / N + ((long long)j < nf % N ? 1 : 0)) % Q);
    for (int w = 0; w < W; ++w) {
      const unsigned c = cnt[w][j] % q;
      cnt[w][j] = run;
      run = (run + c) % q;
    }
  }
  __syncthreads();
  for (int p0 = beg; p0 < end; p0 += 32) {
    const int p = p0 + lane;
    const unsigned r = p < end ? (unsigned)(res[p] >> 56) : 0u;
    const unsigned peers = warp_match_nb<5>(r, p < end);
    if (p < end) out[p] = (cnt[wid][r] + __popc(peers & lt)) % q;
    __syncwarp();
    if (p < end && (peers & lt) == 0) cnt[wid][r] = (cnt[wid][r] + __popc(peers)) % q;
    __syncwarp();
  }
  __syncthreads();
}

}  // namespace rails
