// k_sched.cu -- a2 chunking, a3 segmented radix sort, a4 LPT chain (sm_100a).
//
// a2 (R#3): message B of (g,h) -> floor(B/C) full chunks + one remainder of
//    B mod C bytes.  Full chunks are never materialised: every full chunk (size C)
//    is larger than every remainder (< C) and full chunks are emitted in (g,h,c)
//    order, so under Alg. 2's sort (size desc, ties by GPU index, R#4) they form
//    the prefix of the sorted list in emission order, and LPT with all-zero start
//    loads deals them round-robin: full chunk i -> rail i mod N at offset
//    floor(i/N)*C (lowest-index argmin, R#5).  k_chunk_sort emits
//    full_base = exclusive prefix of floor(B/C) in (g,h) order and compacts the
//    remainders (at most one per message) into a list in (g,h) order.
// a3: the remainder list is sorted by size descending with a stable
//    LSD radix sort on key = C-1-size (8-bit digits, passes whose digit is constant
//    over the segment are skipped).  Stability keeps (g,h) order among equal sizes,
//    which is exactly the tie-break R#4.  One CTA per (unit, node); the segment
//    lives in shared memory when it fits (generic pointers, global otherwise).
// a4: one warp per (unit, node) runs the serial chain over the sorted
//    remainders.  Default (N in {2,4,8,16}, C < 2^23): k_lpt_wstage -- every lane
//    holds the N rail keys (rel << 5) | rail sorted in registers (argmin = K[0],
//    lowest rail on ties), runs of equal sizes are dealt by the exact cyclic
//    closed form with all 32 lanes writing, and the sorted size list is staged
//    through shared memory one batch ahead.  Otherwise k_lpt_chain: lane j holds
//    rail j's load relative to a running base and argmin-with-lowest-index-tie is
//    one redux.sync.min.u32 on (rel << 5) | j.  Offsets are base + rel of the
//    chosen rail before the add (R#19).  Results are written in sorted order and
//    expanded to per-message rem_rail / rem_off through the inverse permutation.
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "radix.cuh"

namespace rails {

// ---------------------------------------------------------------- a2 + a3
constexpr int SORT_THREADS = 512;
constexpr int SORT_SMEM_ITEMS = 16384;  // items per CTA kept in shared memory

// KeyT: uint16_t when every key C-1-size fits 16 bits (C <= 65536), else uint32_t;
// IdxT: uint16_t message index when N*G <= 65536.  Smaller items -> more CTAs per SM.
// SMEM: the segment's sort buffers are in shared memory (known at compile time, so
// the radix passes use shared-memory instructions instead of generic ones).
template <typename KeyT, typename IdxT, int THREADS, bool SMEM>
__global__ void __launch_bounds__(THREADS)
    k_chunk_sort(const int64_t* __restrict__ msg, long long NG, int N, int d0, int nd,
                 long long C, int cshift, int nbits, int64_t* __restrict__ full_base,
                 int32_t* __restrict__ ws_inv, int64_t* __restrict__ n_full_out,
                 int32_t* __restrict__ n_rem_out, uint32_t* __restrict__ ws_w,
                 uint8_t* __restrict__ ws_scratch, int use_smem,
                 int* err) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ long long scan_scratch[33];
  __shared__ int hist[(THREADS / 32) * 256];
  __shared__ int sc[256];
  __shared__ uint32_t red32[32];

  const long long seg = blockIdx.x;
  const ChunkDiv cd{C, cshift};
  const int64_t* __restrict__ mg = msg + seg * NG;
  const long long G = NG / N;
  const int d = d0 + (int)(seg % nd);

  KeyT *kA, *kB;
  IdxT *iA, *iB;
  {
    const long long cap = NG;
    uint8_t* base;
    if constexpr (SMEM) base = smem;
    else base = ws_scratch + seg * (cap * (8 + 2 * sizeof(IdxT)) + 64);
    kA = (KeyT*)base;
    kB = kA + cap;
    iA = (IdxT*)(kB + cap);
    iB = iA + cap;
  }

  // Pass over the messages in tiles of THREADS * IPT, each thread owning IPT
  // consecutive messages: its loads are all in flight at once and one block scan
  // per tile gives the running (full chunks, remainders) prefix.
  constexpr int IPT = 8;
  long long carry_full = 0;
  int carry_rem = 0;
  KeyT kor = 0, kand = (KeyT)~(KeyT)0;
  for (long long t0 = 0; t0 < NG; t0 += (long long)THREADS * IPT) {
    const long long m0 = t0 + (long long)threadIdx.x * IPT;
    long long B[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) B[j] = m0 + j < NG ? mg[m0 + j] : 0;
    long long snf = 0;
    int srem = 0;
    long long nfv[IPT];
    // destination GPU h = m mod G of the first item, then stepped (one division
    // per thread and tile instead of one per message)
    int h = (int)((unsigned long long)m0 % (unsigned long long)G);
    const int lo = d * N, hi = d * N + N;  // the source node's own GPUs (R#2)
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      // negative bytes, or bytes to a GPU of the source node (R#2), are invalid
      if (B[j] < 0 || (B[j] != 0 && h >= lo && h < hi)) {
        flag_error(err, ERR_RANGE);
        B[j] = 0;
      }
      if (++h >= G) h -= G;
      nfv[j] = cd.div(B[j]);
      if (nfv[j] >= (1LL << 40)) flag_error(err, ERR_OVERFLOW);
      snf += nfv[j];
      srem += (B[j] - nfv[j] * C) > 0;
    }
    long long tot;
    const long long ex = block_excl_scan((snf << 16) | srem, scan_scratch, &tot);
    long long fb = carry_full + (ex >> 16);
    int pos = carry_rem + (int)(ex & 0xffff);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const long long m = m0 + j;
      if (m >= NG) break;
      const long long nf = nfv[j];
      const long long rem = B[j] - nf * C;
      full_base[seg * NG + m] = fb;
      fb += nf;
      if (rem > 0) {
        const KeyT key = (KeyT)(C - 1 - rem);
        kA[pos] = key;
        iA[pos] = (IdxT)m;
        kor |= key;
        kand &= key;
        ++pos;
      }
    }
    carry_full += tot >> 16;
    carry_rem += (int)(tot & 0xffff);
  }
  kor = (KeyT)block_reduce_or((uint32_t)kor, red32);
  kand = (KeyT)block_reduce_and((uint32_t)kand, red32);
  if (threadIdx.x == 0) {
    n_full_out[seg] = carry_full;
    n_rem_out[seg] = carry_rem;
  }
  __syncthreads();
  const int n = carry_rem;
  const int which = radix_sort<KeyT, IdxT>(kA, iA, kB, iB, n, kor, kand, nbits, hist, sc);
  const KeyT* ks = which ? kB : kA;
  const IdxT* is = which ? iB : iA;
  // inverse permutation in the free index buffer, then written out coalesced
  // (message m -> sorted position of its remainder, -1 if none)
  IdxT* inv = which ? iA : iB;
  constexpr IdxT NONE = (IdxT)~(IdxT)0;
  for (long long m = threadIdx.x; m < NG; m += THREADS) inv[m] = NONE;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += THREADS) {
    ws_w[seg * NG + i] = (uint32_t)(C - 1 - (long long)ks[i]);
    inv[is[i]] = (IdxT)i;
  }
  __syncthreads();
  for (long long m = threadIdx.x; m < NG; m += THREADS)
    ws_inv[seg * NG + m] = inv[m] == NONE ? -1 : (int32_t)inv[m];
}

// ---------------------------------------------------------------- a4 chain
constexpr int CHAIN_WARPS = 4;

// Chain results are written in SORTED order (sequential per chain: full sectors,
// no read-modify-write), packed as rail << 56 | offset; k_expand_rem then writes
// rem_rail / rem_off per message, coalesced, through the sort's inverse permutation.
constexpr long long OFF_MASK = (1LL << 56) - 1;
__device__ __forceinline__ uint64_t pack_res(unsigned rail, long long off) {
  return ((uint64_t)rail << 56) | ((uint64_t)off & (uint64_t)OFF_MASK);
}

__global__ void __launch_bounds__(CHAIN_WARPS * 32)
    k_lpt_chain(long long nseg, int N, long long C, long long NG,
                const int64_t* __restrict__ n_full, const int32_t* __restrict__ n_rem,
                const uint32_t* __restrict__ ws_w, uint64_t* __restrict__ ws_res,
                int64_t* __restrict__ send_load, int* err) {
  const int lane = threadIdx.x & 31;
  const long long seg = (long long)blockIdx.x * CHAIN_WARPS + (threadIdx.x >> 5);
  if (seg >= nseg) return;
  const long long nf = n_full[seg];
  const long long q = nf / N;
  const int r = (int)(nf - q * N);
  const int nr = n_rem[seg];
  const uint32_t* __restrict__ sw = ws_w + seg * NG;
  uint64_t* __restrict__ res = ws_res + seg * NG;

  if (C < (1LL << 26)) {
    // Fast path: relative loads, single redux.sync per step.
    long long base = C * q;  // current minimum load (full-chunk closed form)
    uint32_t rel = (lane < r) ? (uint32_t)C : 0u;
    for (int i0 = 0; i0 < nr; i0 += 32) {
      uint32_t wv = 0;
      if (i0 + lane < nr) wv = sw[i0 + lane];
      const int cnt = min(32, nr - i0);
      for (int b = 0; b < cnt; ++b) {
        const uint32_t wb = __shfl_sync(FULL, wv, b);
        const uint32_t key = (lane < N) ? ((rel << 5) | (uint32_t)lane) : 0xffffffffu;
        const uint32_t kmin = __reduce_min_sync(FULL, key);
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
    if (lane < N) send_load[seg * N + lane] = base + rel;
  } else {
    // General path: 64-bit loads, butterfly argmin over (load, lane).
    long long L = (lane < N) ? C * (q + (lane < r ? 1 : 0)) : LLONG_MAX;
    for (int i0 = 0; i0 < nr; i0 += 32) {
      uint32_t wv = 0;
      if (i0 + lane < nr) wv = sw[i0 + lane];
      const int cnt = min(32, nr - i0);
      for (int b = 0; b < cnt; ++b) {
        const uint32_t wb = __shfl_sync(FULL, wv, b);
        long long v = L;
        int ix = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          long long ov = __shfl_xor_sync(FULL, v, o);
          int oi = __shfl_xor_sync(FULL, ix, o);
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
    if (lane < N) {
      if (L < 0) flag_error(err, ERR_OVERFLOW);
      send_load[seg * N + lane] = L;
    }
  }
}



// LPT network step shared by the chain kernels: K sorted ascending holds the N
// rail keys (rel << 5) | rail; the chunk of size w goes to K[0]'s rail (argmin,
// lowest rail on ties) at offset base + rel, and K[0] + (w << 5) is merged back.
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

template <int NT>
__device__ __forceinline__ void lpt_step(uint32_t (&K)[NT], uint32_t w, uint64_t* __restrict__ res_i,
                                         long long base) {
  *res_i = lpt_step_v<NT>(K, w, base);
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

// Eight consecutive sorted items.  Exact fast path for a run of equal sizes w: if
// the largest key is below the smallest key plus w, compared as (load, rail) keys
// (K[NT-1] - K[0] < w << 5), LPT deals the next NT items of size w one per rail in
// the current (load, rail) order -- after k of them the assigned rails sit at keys
// K_i + (w << 5) > K[NT-1] >= every unassigned key -- and the sorted order is
// unchanged afterwards, all loads having grown by w.  So 8 equal items (8 a
// multiple of NT) go to K[p mod NT] at rel + (p div NT)*w and base += (8/NT)*w,
// with no compare network.  Otherwise: eight network steps.
__device__ __forceinline__ void cas_u32(uint32_t& a, uint32_t& b) {
  const uint32_t lo = min(a, b), hi = max(a, b);
  a = lo;
  b = hi;
}

// NT = 8, 8 equal items, key spread K[7] - K[0] < 2w << 5.  The picks are the 8
// smallest slots (value, rail) among every rail's next slots rel + t*w; a rail's
// third slot is at key >= K[0] + 2(w << 5) > K[7], so the 8 smallest lie in
// {K_i} U {K_i + w}: a bitonic
// half-cleaner (K ascending against K + w descending) selects them, an 8-wide
// bitonic merge orders them.  K_i was taken iff K_i < K_{7-i} + w, and K_i + w iff
// K_i + w < K_{7-i}; the new keys K_i + (takes)*w are re-sorted (Batcher, 19 CAS).
__device__ __forceinline__ void lpt_merge8(uint32_t (&K)[8], uint32_t w,
                                           uint64_t* __restrict__ out, long long base) {
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
  // L is bitonic: merge 8
#pragma unroll
  for (int i = 0; i < 4; ++i) cas_u32(L[i], L[i + 4]);
  cas_u32(L[0], L[2]); cas_u32(L[1], L[3]); cas_u32(L[4], L[6]); cas_u32(L[5], L[7]);
  cas_u32(L[0], L[1]); cas_u32(L[2], L[3]); cas_u32(L[4], L[5]); cas_u32(L[6], L[7]);
#pragma unroll
  for (int p = 0; p < 8; ++p) out[p] = pack_res(L[p] & 31u, base + (long long)(L[p] >> 5));
#pragma unroll
  for (int i = 0; i < 8; ++i) K[i] += (uint32_t)c[i] * W;
  // Batcher odd-even merge sort of 8
  cas_u32(K[0], K[1]); cas_u32(K[2], K[3]); cas_u32(K[4], K[5]); cas_u32(K[6], K[7]);
  cas_u32(K[0], K[2]); cas_u32(K[1], K[3]); cas_u32(K[4], K[6]); cas_u32(K[5], K[7]);
  cas_u32(K[1], K[2]); cas_u32(K[5], K[6]);
  cas_u32(K[0], K[4]); cas_u32(K[1], K[5]); cas_u32(K[2], K[6]); cas_u32(K[3], K[7]);
  cas_u32(K[2], K[4]); cas_u32(K[3], K[5]);
  cas_u32(K[1], K[2]); cas_u32(K[3], K[4]); cas_u32(K[5], K[6]);
}

// Keys stay below 2^32: rel < 2^23 after a rebase, spread < 2w < 2^24 on the fast
// paths, at most 8 network steps between rebases (C < 2^23).
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

template <int NT>
__device__ __forceinline__ void lpt_group8(uint32_t (&K)[NT], const uint32_t (&w8)[8],
                                           uint64_t* __restrict__ out, long long& base) {
  uint64_t r[8];
  lpt_group8_v<NT>(K, w8, r, base);
  store8(out, r);
}

// A whole run of n equal sizes w once K[NT-1] - K[0] < w << 5 (the cyclic case
// above, repeated): item t of the run goes to K[t mod NT] at rel + (t div NT)*w,
// so the warp writes the run in parallel, lane l taking t = l, l + 32, ... (NT
// divides 32, so t mod NT = l mod NT).  Afterwards rail K_i carries
// q = n div NT more items, plus one for i < n mod NT: the sorted keys become
// K[rr..NT-1] + q*w, K[0..rr-1] + (q+1)*w (still sorted, spread still < w).
template <int NT>
__device__ __forceinline__ void lpt_run_cyclic(uint32_t (&K)[NT], uint32_t w, int n, int lane,
                                               uint64_t* __restrict__ out, long long& base) {
  uint32_t kl = K[0];
#pragma unroll
  for (int j = 1; j < NT; ++j)
    if ((lane % NT) == j) kl = K[j];
  const long long lb = base + (long long)(kl >> 5);
  for (int t = lane; t < n; t += 32) out[t] = pack_res(kl & 31u, lb + (long long)(t / NT) * w);
  base += (long long)(n / NT) * w;
  const uint32_t W = w << 5;
  for (int s = n % NT; s > 0; --s) {
    const uint32_t h = K[0] + W;
#pragma unroll
    for (int j = 0; j < NT - 1; ++j) K[j] = K[j + 1];
    K[NT - 1] = h;
  }
  lpt_rebase<NT>(K, base);
}

// Few long chains (C3: 64, C5: 256): one chain per warp.  All 32 lanes stream the
// sorted remainder list through a double-buffered shared-memory stage with
// coalesced loads, one batch ahead, and all run the same (warp-uniform) register
// state.  A run of >= 32 equal sizes -- routing traffic has only C / row_bytes
// distinct remainder sizes -- is assigned by single network steps until the
// cyclic condition holds, then written by the whole warp (lpt_run_cyclic); other
// items go eight at a time through lpt_group8_v with lane 0 storing.
constexpr int WS_WARPS = 4;
constexpr int WS_BATCH = 256;

template <int NT>
__global__ void __launch_bounds__(WS_WARPS * 32)
    k_lpt_wstage(long long nseg, long long C, long long NG, const int64_t* __restrict__ n_full,
                 const int32_t* __restrict__ n_rem, const uint32_t* __restrict__ ws_w,
                 uint64_t* __restrict__ ws_res, int64_t* __restrict__ send_load) {
  __shared__ uint32_t sW[WS_WARPS][2][WS_BATCH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long seg = (long long)blockIdx.x * WS_WARPS + wid;
  if (seg >= nseg) return;
  const long long nf = n_full[seg];
  const long long q = nf / NT;
  const int r = (int)(nf - q * NT);
  const int nr = n_rem[seg];
  const uint32_t* __restrict__ gw = ws_w + seg * NG;
  uint64_t* __restrict__ res = ws_res + seg * NG;
  long long base = C * q;
  uint32_t K[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int rail = (i < NT - r) ? (r + i) : (i - (NT - r));
    K[i] = (((i < NT - r) ? 0u : (uint32_t)C) << 5) | (uint32_t)rail;
  }
  constexpr int PL = WS_BATCH / 32;
  uint32_t pw[PL];
#pragma unroll
  for (int p = 0; p < PL; ++p) {
    const int i = p * 32 + lane;
    pw[p] = i < nr ? gw[i] : 0u;
  }
  int cur = 0;
  for (int b0 = 0; b0 < nr; b0 += WS_BATCH) {
    uint32_t cw[PL];
#pragma unroll
    for (int p = 0; p < PL; ++p) {
      sW[wid][cur][p * 32 + lane] = pw[p];
      cw[p] = pw[p];
    }
    __syncwarp();
    const int nb = b0 + WS_BATCH;  // prefetch the next batch while this one is assigned
#pragma unroll
    for (int p = 0; p < PL; ++p) {
      const int i = nb + p * 32 + lane;
      pw[p] = i < nr ? gw[i] : 0u;
    }
    const int cnt = min(WS_BATCH, nr - b0);
    const uint32_t* w_ = sW[wid][cur];
    uint64_t* rb = res + b0;
    // the next group's sizes (and the size 31 ahead, the run test) are read from
    // shared memory before the current group is assigned
    uint32_t w8[8], w31;
    auto load8 = [&](int at) {
#pragma unroll
      for (int p = 0; p < 8; ++p) w8[p] = w_[(at + p) & (WS_BATCH - 1)];
      w31 = w_[(at + 31) & (WS_BATCH - 1)];
    };
    int i = 0;
    load8(0);
    while (i < cnt) {
      const uint32_t w = w8[0];
      if (i + 32 <= cnt && w31 == w) {
        // run [i, e) of equal sizes inside this batch (the list is sorted, so the
        // equal entries at or after i are contiguous)
        int e = i;
#pragma unroll
        for (int p = 0; p < PL; ++p) {
          const int j = p * 32 + lane;
          e += __popc(__ballot_sync(0xffffffffu, j >= i && j < cnt && cw[p] == w));
        }
        while (i < e && K[NT - 1] - K[0] >= (w << 5)) {
          const uint64_t r = lpt_step_v<NT>(K, w, base);
          if (lane == 0) rb[i] = r;
          lpt_rebase<NT>(K, base);
          ++i;
        }
        if (i < e) lpt_run_cyclic<NT>(K, w, e - i, lane, rb + i, base);
        i = e;
        load8(i);
      } else if ((8 % NT) == 0 && (i & 7) == 0 && i + 8 <= cnt && w8[7] == w &&
                 K[NT - 1] - K[0] < (w << 5)) {
        // window of up to 32 aligned groups, lane l taking group i + 8l: while
        // every group is 8 equal sizes w_l with K[NT-1] - K[0] < w_l << 5, each is
        // dealt cyclically, K is unchanged and base grows by (8/NT)*w_l, so the
        // groups' bases are an exclusive scan of those increments
        const int at = i + 8 * lane;
        uint32_t a = 0, b = 0;
        if (at + 8 <= cnt) {
          a = w_[at];
          b = w_[at + 7];
        }
        const bool ok = at + 8 <= cnt && a == b && K[NT - 1] - K[0] < (a << 5);
        const unsigned bad = __ballot_sync(0xffffffffu, !ok);
        const int nok = bad ? __ffs(bad) - 1 : 32;  // >= 1: lane 0's group passed above
        const uint32_t inc = lane < nok ? (uint32_t)(8 / NT) * a : 0u;
        uint32_t ex = inc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, ex, o);
          if (lane >= o) ex += t;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, ex, 31);
        ex -= inc;
        if (lane < nok) {
          uint64_t r[8];
          const long long bl = base + (long long)ex;
#pragma unroll
          for (int p = 0; p < 8; ++p)
            r[p] = pack_res(K[p % NT] & 31u,
                            bl + (long long)(K[p % NT] >> 5) + (long long)(p / NT) * a);
          store8(rb + at, r);
        }
        base += (long long)tot;
        i += 8 * nok;
        load8(i);
      } else if (i + 8 <= cnt && (i & 7) == 0) {
        uint32_t g8[8];
        uint64_t r[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) g8[p] = w8[p];
        load8(i + 8);
        lpt_group8_v<NT>(K, g8, r, base);
        if (lane == 0) store8(rb + i, r);
        i += 8;
      } else {
        const uint64_t r = lpt_step_v<NT>(K, w, base);
        if (lane == 0) rb[i] = r;
        lpt_rebase<NT>(K, base);
        ++i;
        load8(i);
      }
    }
    __syncwarp();
    cur ^= 1;
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NT; ++j)
      send_load[seg * NT + (K[j] & 31u)] = base + (long long)(K[j] >> 5);
  }
}

// Thread-per-chain variant (N = NT in {2, 4, 8, 16}, C < 2^23): the N rail keys
// (rel << 5) | rail live in registers kept SORTED ascending, so the argmin of
// Alg. 2 step 3 is simply K[0] (lowest rail on equal load because the rail index
// is the low key bits, R#5).  Assigning w moves K[0] to K[0] + (w << 5), which is
// merged back into K[1..NT-1] by a branch-free compare/select network.  Loads are
// kept relative to `base` (an exact int64) and rebased when the minimum exceeds
// 2^23; with at most 8 steps between rebases and C < 2^23, rel < 2^23 + 9*C < 2^27,
// so keys stay below 2^32.
// Chains are spread cpw per warp (cpw <= 32, chosen from the SM count) so that a
// few long chains (C3: 64, C5: 256) occupy many SMs instead of sharing one LSU.
template <int NT>
__global__ void __launch_bounds__(128)
    k_lpt_thread(long long nseg, int cpw, long long C, long long NG,
                 const int64_t* __restrict__ n_full, const int32_t* __restrict__ n_rem,
                 const uint32_t* __restrict__ ws_w, uint64_t* __restrict__ ws_res,
                 int64_t* __restrict__ send_load) {
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long seg = gw * cpw + lane;
  if (lane >= cpw || seg >= nseg) return;
  const long long nf = n_full[seg];
  const long long q = nf / NT;
  const int r = (int)(nf - q * NT);
  const int nr = n_rem[seg];
  const uint32_t* __restrict__ sw = ws_w + seg * NG;
  uint64_t* __restrict__ res = ws_res + seg * NG;
  // full-chunk closed form: rails 0..r-1 hold C*(q+1), the rest C*q.  Sorted by
  // (load, rail): rails r..NT-1 (rel 0) first, then rails 0..r-1 (rel C).
  long long base = C * q;
  uint32_t K[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const int rail = (i < NT - r) ? (r + i) : (i - (NT - r));
    const uint32_t rel = (i < NT - r) ? 0u : (uint32_t)C;
    K[i] = (rel << 5) | (uint32_t)rail;
  }
  constexpr int PF = 8;
  int i = 0;
  // batches of 8 as two 16-byte loads per array (chain lists start 16-B aligned:
  // N*G is a multiple of 4 for even N)
  auto ld8 = [](const uint32_t* p, uint32_t (&o)[PF]) {
    const uint4 a = __ldg((const uint4*)p), b = __ldg((const uint4*)p + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
  };
  uint32_t wv[PF];
  if (PF <= nr) ld8(sw, wv);
  for (; i + PF <= nr; i += PF) {
    uint32_t wn[PF];  // next batch in flight while this one is assigned
    if (i + 2 * PF <= nr) ld8(sw + i + PF, wn);
    lpt_group8<NT>(K, wv, res + i, base);
#pragma unroll
    for (int p = 0; p < PF; ++p) wv[p] = wn[p];
  }
  for (; i < nr; ++i) {
    lpt_step<NT>(K, __ldg(sw + i), res + i, base);
    lpt_rebase<NT>(K, base);
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) send_load[seg * NT + (K[j] & 31u)] = base + (long long)(K[j] >> 5);
}

// LPT chain implementation: 0 = thread-per-chain when N allows (default),
// 1 = warp-per-chain (RAILS_CHAIN_IMPL=1, kept as the reference path).
// RAILS_CHAIN_IMPL: 1 = generic warp chain, 2 = warp-staged (the default),
// 3 = thread-per-chain (measurement overrides)
static int chain_impl() {
  const char* e = getenv("RAILS_CHAIN_IMPL");
  return (e && e[0] >= '1' && e[0] <= '3') ? e[0] - '0' : 0;
}

static int ceil_log2(long long x) {  // bits needed for values 0..x-1
  int b = 0;
  while ((1LL << b) < x) ++b;
  return b;
}

// Expand the sorted-order chain results into per-message rem_rail / rem_off,
// coalesced: message m of segment seg has a remainder iff ws_inv[m] >= 0 (the
// sorted position written by k_chunk_sort).
__global__ void __launch_bounds__(256)
    k_expand_rem(long long NG, const int32_t* __restrict__ ws_inv,
                 const uint64_t* __restrict__ ws_res, int8_t* __restrict__ rem_rail,
                 int64_t* __restrict__ rem_off, const uint32_t* __restrict__ ws_qp,
                 int32_t* __restrict__ rem_qp) {
  const long long seg = blockIdx.y;
  const long long m = (long long)blockIdx.x * 256 + threadIdx.x;
  if (m >= NG) return;
  const int pos = ws_inv[seg * NG + m];
  int8_t r = -1;
  long long o = 0;
  int32_t q = -1;
  if (pos >= 0) {
    const uint64_t v = ws_res[seg * NG + pos];
    r = (int8_t)(v >> 56);
    o = (long long)(v & (uint64_t)OFF_MASK);
    if (rem_qp) q = (int32_t)ws_qp[seg * NG + pos];
  }
  rem_rail[seg * NG + m] = r;
  rem_off[seg * NG + m] = o;
  if (rem_qp) rem_qp[seg * NG + m] = q;
}

// k_expand_rem with 4 consecutive messages per thread (NG % 4 == 0, aligned
// outputs): one 16-byte load of the inverse permutation, four gathers in flight,
// 4-byte rail / 16-byte offset stores.  The one-per-thread kernel is latency-bound
// (two dependent loads per thread: ncu long-scoreboard stalls); this keeps 4x the
// loads in flight per warp.  Segments beyond gridDim.y are looped.
__global__ void __launch_bounds__(256)
    k_expand_rem4(long long NG, long long nseg, const int32_t* __restrict__ ws_inv,
                  const uint64_t* __restrict__ ws_res, int8_t* __restrict__ rem_rail,
                  int64_t* __restrict__ rem_off, const uint32_t* __restrict__ ws_qp,
                  int32_t* __restrict__ rem_qp) {
  const long long m = ((long long)blockIdx.x * 256 + threadIdx.x) * 4;
  if (m >= NG) return;
  for (long long seg = blockIdx.y; seg < nseg; seg += gridDim.y) {
    const long long b = seg * NG;
    const int4 pos = *(const int4*)(ws_inv + b + m);
    const int p[4] = {pos.x, pos.y, pos.z, pos.w};
    uint64_t v[4];
    uint32_t qv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = p[i] >= 0 ? ws_res[b + p[i]] : 0ull;
    if (rem_qp) {
#pragma unroll
      for (int i = 0; i < 4; ++i) qv[i] = p[i] >= 0 ? ws_qp[b + p[i]] : 0u;
    }
    char4 r;
    r.x = p[0] >= 0 ? (signed char)(v[0] >> 56) : (signed char)-1;
    r.y = p[1] >= 0 ? (signed char)(v[1] >> 56) : (signed char)-1;
    r.z = p[2] >= 0 ? (signed char)(v[2] >> 56) : (signed char)-1;
    r.w = p[3] >= 0 ? (signed char)(v[3] >> 56) : (signed char)-1;
    *(char4*)(rem_rail + b + m) = r;
    longlong2 o0, o1;
    o0.x = p[0] >= 0 ? (long long)(v[0] & (uint64_t)OFF_MASK) : 0;
    o0.y = p[1] >= 0 ? (long long)(v[1] & (uint64_t)OFF_MASK) : 0;
    o1.x = p[2] >= 0 ? (long long)(v[2] & (uint64_t)OFF_MASK) : 0;
    o1.y = p[3] >= 0 ? (long long)(v[3] & (uint64_t)OFF_MASK) : 0;
    *(longlong2*)(rem_off + b + m) = o0;
    *(longlong2*)(rem_off + b + m + 2) = o1;
    if (rem_qp) {
      int4 q;
      q.x = p[0] >= 0 ? (int32_t)qv[0] : -1;
      q.y = p[1] >= 0 ? (int32_t)qv[1] : -1;
      q.z = p[2] >= 0 ? (int32_t)qv[2] : -1;
      q.w = p[3] >= 0 ? (int32_t)qv[3] : -1;
      *(int4*)(rem_qp + b + m) = q;
    }
  }
}

// Same as k_expand_rem with one CTA per (unit, node): the segment's n_rem chain
// results are first copied into shared memory (coalesced), so the per-message
// gather through the inverse permutation hits shared memory instead of 32-byte
// global sectors for 8-byte values.
constexpr int EXP_THREADS = 512;
__global__ void __launch_bounds__(EXP_THREADS)
    k_expand_seg(long long NG, const int32_t* __restrict__ n_rem,
                 const int32_t* __restrict__ ws_inv, const uint64_t* __restrict__ ws_res,
                 int8_t* __restrict__ rem_rail, int64_t* __restrict__ rem_off,
                 const uint32_t* __restrict__ ws_qp, int32_t* __restrict__ rem_qp) {
  extern __shared__ __align__(16) uint64_t sres[];
  const long long seg = blockIdx.x;
  const int nr = n_rem[seg];
  const uint64_t* __restrict__ res = ws_res + seg * NG;
  for (int p = threadIdx.x; p < nr; p += EXP_THREADS) sres[p] = res[p];
  __syncthreads();
  const int32_t* __restrict__ inv = ws_inv + seg * NG;
  for (long long m = threadIdx.x; m < NG; m += EXP_THREADS) {
    const int pos = inv[m];
    int8_t r = -1;
    long long o = 0;
    int32_t q = -1;
    if (pos >= 0) {
      const uint64_t v = sres[pos];
      r = (int8_t)(v >> 56);
      o = (long long)(v & (uint64_t)OFF_MASK);
      if (rem_qp) q = (int32_t)ws_qp[seg * NG + pos];
    }
    rem_rail[seg * NG + m] = r;
    rem_off[seg * NG + m] = o;
    if (rem_qp) rem_qp[seg * NG + m] = q;
  }
}

// NEXT f2, Alg. 2 step 4 (R#34): per-rail round-robin QP index in
// assignment order.  The chain results are already in sorted (= assignment)
// order, so the QP of the p-th remainder is (full chunks on its rail + remainders
// on its rail before p) mod Q, full chunks being assigned first (i mod N).  One
// CTA per (unit, node); warp w owns a contiguous slice of the sorted list.
// Pass 1 counts each slice's items per rail; thread j < N turns the counts into
// per-warp starting counters (exclusive over warps, plus rail j's full chunks);
// pass 2 ranks each 32-item batch by rail with a ballot multi-split (5 ballots,
// rails < 32) and advances the warp's counters from the group leaders.
constexpr int QP_WARPS = 8;

__global__ void __launch_bounds__(QP_WARPS * 32)
    k_qp_rank(int N, int Q, long long NG, const int64_t* __restrict__ n_full,
              const int32_t* __restrict__ n_rem, const uint64_t* __restrict__ ws_res,
              uint32_t* __restrict__ ws_qp) {
  __shared__ unsigned cnt[QP_WARPS][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long seg = blockIdx.x;
  const long long nf = n_full[seg];
  const int nr = n_rem[seg];
  const uint64_t* __restrict__ res = ws_res + seg * NG;
  uint32_t* __restrict__ out = ws_qp + seg * NG;
  const int per = (((nr + QP_WARPS - 1) / QP_WARPS) + 31) & ~31;
  const int beg = wid * per, end = min(nr, beg + per);
  const unsigned lt = lanemask_lt();
  cnt[wid][lane] = 0;
  __syncwarp();
  for (int p0 = beg; p0 < end; p0 += 32) {  // pass 1: per-rail counts of the slice
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
    for (int w = 0; w < QP_WARPS; ++w) {
      const unsigned c = cnt[w][j] % q;
      cnt[w][j] = run;
      run = (run + c) % q;
    }
  }
  __syncthreads();
  for (int p0 = beg; p0 < end; p0 += 32) {  // pass 2: QP = counter + rank, mod Q
    const int p = p0 + lane;
    const unsigned r = p < end ? (unsigned)(res[p] >> 56) : 0u;
    const unsigned peers = warp_match_nb<5>(r, p < end);
    if (p < end) out[p] = (cnt[wid][r] + __popc(peers & lt)) % q;
    __syncwarp();
    if (p < end && (peers & lt) == 0) cnt[wid][r] = (cnt[wid][r] + __popc(peers)) % q;
    __syncwarp();
  }
}

// workspace: [256 B header][ws_res u64 (nseg*NG)][ws_w u32][ws_qp u32][ws_inv i32]
//            [sort spill scratch when N*G > SORT_SMEM_ITEMS]
size_t schedule_workspace_bytes(int U, int nd, long long NG) {
  const long long nseg = (long long)U * nd;
  size_t lists = (size_t)nseg * NG * (8 + 4 + 4 + 4);
  size_t scratch = (NG <= SORT_SMEM_ITEMS) ? 0 : (size_t)nseg * (NG * (8 + 2 * 4) + 64);
  return 256 + lists + scratch;
}

cudaError_t launch_schedule(const LaunchCtx& c, int U, int nd, int d0, int M, int N, long long C,
                            const int64_t* msg, const rails_sched_t& s, void* ws,
                            int32_t* rem_qp, int qps_per_rail) {
  const long long nseg = (long long)U * nd;
  const long long NG = (long long)N * M * N;
  int cshift = -1;
  if ((C & (C - 1)) == 0) cshift = ceil_log2(C);
  const int nbits = ceil_log2(C > 1 ? C - 1 : 1) + 1;
  uint8_t* w8 = (uint8_t*)ws;
  uint64_t* ws_res = (uint64_t*)(w8 + 256);
  uint32_t* ws_w = (uint32_t*)(ws_res + nseg * NG);
  uint32_t* ws_qp = ws_w + nseg * NG;
  int32_t* ws_inv = (int32_t*)(ws_qp + nseg * NG);
  uint8_t* scratch = (uint8_t*)(ws_inv + nseg * NG);
  cudaError_t e;
  if (NG <= SORT_SMEM_ITEMS) {
    // CTA size by segment size (128 / 256 / 512 threads) and 16-bit keys when
    // C <= 65536, so that several CTAs fit per SM (shared memory per item: 2 keys
    // + 2 indices).
    const bool k16 = C <= 65536;
    const size_t smem = (size_t)NG * (2 * (k16 ? 2 : 4) + 2 * sizeof(uint16_t));
    const int thr = NG <= 2048 ? 128 : (NG <= 8192 ? 256 : SORT_THREADS);
    void (*kern)(const int64_t*, long long, int, int, int, long long, int, int, int64_t*,
                 int32_t*, int64_t*, int32_t*, uint32_t*, uint8_t*, int, int*);
    if (k16)
      kern = thr == 128 ? k_chunk_sort<uint16_t, uint16_t, 128, true>
           : thr == 256 ? k_chunk_sort<uint16_t, uint16_t, 256, true>
                        : k_chunk_sort<uint16_t, uint16_t, SORT_THREADS, true>;
    else
      kern = thr == 128 ? k_chunk_sort<uint32_t, uint16_t, 128, true>
           : thr == 256 ? k_chunk_sort<uint32_t, uint16_t, 256, true>
                        : k_chunk_sort<uint32_t, uint16_t, SORT_THREADS, true>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)nseg, thr, smem, c.stream>>>(
        msg, NG, N, d0, nd, C, cshift, nbits, s.full_base, ws_inv, s.n_full, s.n_rem, ws_w,
        nullptr, 1, c.err);
  } else {
    k_chunk_sort<uint32_t, uint32_t, SORT_THREADS, false><<<(unsigned)nseg, SORT_THREADS, 0, c.stream>>>(
        msg, NG, N, d0, nd, C, cshift, nbits, s.full_base, ws_inv, s.n_full, s.n_rem, ws_w,
        scratch, 0, c.err);
  }
  count_launch(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int ci = chain_impl();
  const bool nt_ok = C < (1LL << 23) && (N == 2 || N == 4 || N == 8 || N == 16);
  // warp-staged chains by default: measured faster than thread-per-chain for few
  // long chains (C3, C5) and for many (C2: 16 000, C4: 4 096), since runs of
  // equal sizes are written by whole warps and the list staging hides latency
  if (nt_ok && (ci == 0 || ci == 2)) {
    const unsigned wgrid = (unsigned)((nseg + WS_WARPS - 1) / WS_WARPS);
#define RAILS_WS_CHAIN(NT)                                                                  \
  if (N == NT)                                                                              \
    k_lpt_wstage<NT><<<wgrid, WS_WARPS * 32, 0, c.stream>>>(nseg, C, NG, s.n_full, s.n_rem, \
                                                           ws_w, ws_res, s.send_load);
    RAILS_WS_CHAIN(2)
    RAILS_WS_CHAIN(4)
    RAILS_WS_CHAIN(8)
    RAILS_WS_CHAIN(16)
#undef RAILS_WS_CHAIN
  } else if (nt_ok && ci != 1) {
    // chains per warp: fill ~8 warps per SM before packing lanes (LSU sharing)
    long long cpw = nseg / ((long long)c.num_sms * 8);
    cpw = cpw < 1 ? 1 : (cpw > 32 ? 32 : cpw);
    const long long nwarp = (nseg + cpw - 1) / cpw;
    const unsigned tgrid = (unsigned)((nwarp + 3) / 4);
#define RAILS_THREAD_CHAIN(NT)                                                            \
  if (N == NT)                                                                            \
    k_lpt_thread<NT><<<tgrid, 128, 0, c.stream>>>(nseg, (int)cpw, C, NG, s.n_full, s.n_rem, \
                                                  ws_w, ws_res, s.send_load);
    RAILS_THREAD_CHAIN(2)
    RAILS_THREAD_CHAIN(4)
    RAILS_THREAD_CHAIN(8)
    RAILS_THREAD_CHAIN(16)
#undef RAILS_THREAD_CHAIN
  } else {
    const unsigned grid = (unsigned)((nseg + CHAIN_WARPS - 1) / CHAIN_WARPS);
    k_lpt_chain<<<grid, CHAIN_WARPS * 32, 0, c.stream>>>(nseg, N, C, NG, s.n_full, s.n_rem, ws_w,
                                                         ws_res, s.send_load, c.err);
  }
  count_launch(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (rem_qp) {
    k_qp_rank<<<(unsigned)nseg, QP_WARPS * 32, 0, c.stream>>>(N, qps_per_rail, NG, s.n_full,
                                                              s.n_rem, ws_res, ws_qp);
    count_launch(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const size_t esm = (size_t)NG * 8;
  const char* xv = getenv("RAILS_EXPAND_IMPL");
  // Expand kernel: 4 messages per thread when the outputs are aligned (C2 chunk ->
  // expand 94 -> ~60 us, C4 schedule 0.620 -> 0.605 ms against the staged kernel);
  // else the segment-staged gather for long segments (C4: 183 -> ~110 us against
  // one message per thread), else one message per thread.  RAILS_EXPAND_IMPL=1|2
  // forces one per thread, 3 the staged kernel (where it fits).
  const bool x1 = xv && (xv[0] == '1' || xv[0] == '2'), x3 = xv && xv[0] == '3';
  const bool al4 = NG % 4 == 0 && ((uintptr_t)ws_inv & 15) == 0 &&
                   ((uintptr_t)s.rem_rail & 3) == 0 && ((uintptr_t)s.rem_off & 15) == 0 &&
                   ((uintptr_t)rem_qp & 15) == 0;
  if (al4 && !x1 && !x3) {
    const long long gy = nseg < 65535 ? nseg : 65535;
    k_expand_rem4<<<dim3((unsigned)((NG / 4 + 255) / 256), (unsigned)gy), 256, 0, c.stream>>>(
        NG, nseg, ws_inv, ws_res, s.rem_rail, s.rem_off, rem_qp ? ws_qp : nullptr, rem_qp);
  } else if (esm <= 160 * 1024 && !x1 && (x3 || NG >= 8192)) {
    if (esm > 48 * 1024 &&
        (e = cudaFuncSetAttribute(k_expand_seg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)esm)) != cudaSuccess)
      return e;
    k_expand_seg<<<(unsigned)nseg, EXP_THREADS, esm, c.stream>>>(
        NG, s.n_rem, ws_inv, ws_res, s.rem_rail, s.rem_off, rem_qp ? ws_qp : nullptr, rem_qp);
  } else {
    if (nseg > 65535) return cudaErrorInvalidConfiguration;
    k_expand_rem<<<dim3((unsigned)((NG + 255) / 256), (unsigned)nseg), 256, 0, c.stream>>>(
        NG, ws_inv, ws_res, s.rem_rail, s.rem_off, rem_qp ? ws_qp : nullptr, rem_qp);
  }
  count_launch(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- generic assign
// One CTA per flow set: stable radix sort of ~w (64-bit keys) then the 64-bit
// argmin chain on warp 0.  Workspace holds the per-set key/index buffers.
__global__ void __launch_bounds__(SORT_THREADS)
    k_assign(int N, const int64_t* __restrict__ seg_off, const int64_t* __restrict__ w,
             int32_t* __restrict__ rail, int64_t* __restrict__ off, int64_t* __restrict__ load,
             uint64_t* kA, uint64_t* kB, uint32_t* iA, uint32_t* iB, int* err) {
  __shared__ int hist[(SORT_THREADS / 32) * 256];
  __shared__ int sc[256];
  __shared__ uint64_t red64[32];
  const int s = blockIdx.x;
  const long long b0 = seg_off[s], b1 = seg_off[s + 1];
  const int n = (int)(b1 - b0);
  kA += b0;
  kB += b0;
  iA += b0;
  iB += b0;
  uint64_t kor = 0, kand = ~0ull;
  for (int i = threadIdx.x; i < n; i += SORT_THREADS) {
    long long wi = w[b0 + i];
    if (wi < 0) {
      flag_error(err, ERR_RANGE);
      wi = 0;
    }
    const uint64_t key = ~(uint64_t)wi;
    kA[i] = key;
    iA[i] = (uint32_t)i;
    kor |= key;
    kand &= key;
  }
  kor = block_reduce_or(kor, red64);
  kand = block_reduce_and(kand, red64);
  __syncthreads();
  const int which = radix_sort<uint64_t, uint32_t>(kA, iA, kB, iB, n, kor, kand, 64, hist, sc);
  const uint64_t* ks = which ? kB : kA;
  const uint32_t* is = which ? iB : iA;
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  long long L = (lane < N) ? 0 : LLONG_MAX;
  for (int i0 = 0; i0 < n; i0 += 32) {
    long long wv = 0;
    uint32_t mv = 0;
    if (i0 + lane < n) {
      wv = (long long)(~ks[i0 + lane]);
      mv = is[i0 + lane];
    }
    const int cnt = min(32, n - i0);
    for (int b = 0; b < cnt; ++b) {
      const long long wb = __shfl_sync(FULL, wv, b);
      const uint32_t mb = __shfl_sync(FULL, mv, b);
      long long v = L;
      int ix = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        long long ov = __shfl_xor_sync(FULL, v, o);
        int oi = __shfl_xor_sync(FULL, ix, o);
        if (ov < v || (ov == v && oi < ix)) {
          v = ov;
          ix = oi;
        }
      }
      if (lane == ix) {
        rail[b0 + mb] = ix;
        off[b0 + mb] = v;
        if (L > LLONG_MAX - wb) flag_error(err, ERR_OVERFLOW);
        L += wb;
      }
    }
  }
  if (lane < N) load[(long long)s * N + lane] = L;
}

size_t assign_workspace_bytes(int n_seg, long long F) {
  (void)n_seg;
  return 256 + (size_t)F * (8 + 8 + 4 + 4) + 64;
}

cudaError_t launch_assign(const LaunchCtx& c, int N, int n_seg, const int64_t* seg_off,
                          long long F, const int64_t* w, int32_t* rail, int64_t* off,
                          int64_t* load, void* ws) {
  uint8_t* w8 = (uint8_t*)ws + 256;
  uint64_t* kA = (uint64_t*)w8;
  uint64_t* kB = kA + F;
  uint32_t* iA = (uint32_t*)(kB + F);
  uint32_t* iB = iA + F;
  k_assign<<<(unsigned)n_seg, SORT_THREADS, 0, c.stream>>>(N, seg_off, w, rail, off, load, kA,
                                                           kB, iA, iB, c.err);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace rails
