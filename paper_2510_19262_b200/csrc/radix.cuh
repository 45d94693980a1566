// radix.cuh -- CTA-wide stable LSD radix sort on (key, index) pairs and block
// reductions, shared by the schedule (k_sched.cu) and the fluid simulator
// (k_flowsim.cu).  Buffers are generic pointers (shared or global memory).
#pragma once

#include "common.cuh"

namespace rails {

// ---------------------------------------------------------------- block radix pass
// Stable counting pass over n items on digit (key >> shift) & 255.  Warp w owns
// the contiguous item range [w*seg, (w+1)*seg); per-warp digit counters in
// shared memory `hist` ([W][256] int32), `sc` >= 16 ints of scratch.
// Requires blockDim.x >= 256 and a multiple of 32.
template <typename KeyT, typename IdxT>
__device__ void radix_pass(const KeyT* kin, const IdxT* iin, KeyT* kout, IdxT* iout, int n,
                           int shift, int* hist, int* sc) {
  const int W = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = (((n + W - 1) / W) + 31) & ~31;
  const int beg = wid * seg, end = min(n, beg + seg);
  for (int i = threadIdx.x; i < W * 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  int* my = hist + wid * 256;
  for (int base = beg; base < end; base += 32) {
    int i = base + lane;
    if (i < end) atomicAdd(&my[(unsigned)((kin[i] >> shift) & 255)], 1);  // warp-private
  }
  __syncthreads();
  // digit totals -> exclusive digit bases -> per-warp starting positions
  // digit totals (any block size), exclusive scan of the 256 totals by warp 0
  // (8 digits per lane), then per-warp starting positions per digit.
  // sc: >= 256 ints of shared scratch.
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    int tot = 0;
    for (int w = 0; w < W; ++w) tot += hist[w * 256 + b];
    sc[b] = tot;
  }
  __syncthreads();
  if (wid == 0) {
    int v[8], s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i] = sc[lane * 8 + i];
      s += v[i];
    }
    int run = warp_incl_scan(s) - s;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sc[lane * 8 + i] = run;
      run += v[i];
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += blockDim.x) {
    int run = sc[b];
    for (int w = 0; w < W; ++w) {
      const int c = hist[w * 256 + b];
      hist[w * 256 + b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int base = beg; base < end; base += 32) {
    int i = base + lane;
    const unsigned dg = (i < end) ? (unsigned)((kin[i] >> shift) & 255) : 0u;
    const unsigned peers = warp_match_nb<8>(dg, i < end);
    int pos = 0;
    if (i < end) pos = my[dg] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (i < end && lane == __ffs(peers) - 1) my[dg] += __popc(peers);
    __syncwarp();
    if (i < end) {
      kout[pos] = kin[i];
      iout[pos] = iin[i];
    }
  }
  __syncthreads();
}

// Sort n (key, idx) pairs ascending by key, stably.  Returns 0 if the result is in
// the A buffers, 1 if in the B buffers.  kor/kand: OR and AND of all keys.
template <typename KeyT, typename IdxT>
__device__ int radix_sort(KeyT* kA, IdxT* iA, KeyT* kB, IdxT* iB, int n, KeyT kor, KeyT kand,
                          int nbits, int* hist, int* sc) {
  int cur = 0;
  if (n <= 1) return 0;
  const KeyT diff = kor ^ kand;
  for (int shift = 0; shift < nbits; shift += 8) {
    if (((diff >> shift) & 255) == 0) continue;  // digit constant: pass is identity
    if (cur == 0)
      radix_pass<KeyT, IdxT>(kA, iA, kB, iB, n, shift, hist, sc);
    else
      radix_pass<KeyT, IdxT>(kB, iB, kA, iA, n, shift, hist, sc);
    cur ^= 1;
  }
  return cur;
}

// ---------------------------------------------------------------- narrow digits
// The same stable counting pass on an NB-bit digit (NB <= 8, a compile-time width:
// NB ballots per 32 keys, 2^NB bins), and the sort that covers only the key bits that
// vary (kor ^ kand) in windows of <= 8 bits ending on a varying bit.  Routing traffic
// has few remainder sizes (multiples of the row size), so its keys vary in a few bits
// (C4: 3, C3: 2) and one narrow pass replaces an 8-bit one.  Used by the schedule's
// sorts (k_node.cu, k_chains.cu); radix_sort above keeps 8-bit passes (k_sched.cu's
// 64-bit flow keys, the fluid simulator).
template <typename KeyT, typename IdxT, int NB>
__device__ void radix_pass_nb(const KeyT* kin, const IdxT* iin, KeyT* kout, IdxT* iout, int n,
                              int shift, int* hist, int* sc) {
  constexpr int NBIN = 1 << NB;
  constexpr unsigned MASK = (unsigned)NBIN - 1u;
  const int W = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = (((n + W - 1) / W) + 31) & ~31;
  const int beg = wid * seg, end = min(n, beg + seg);
  for (int i = threadIdx.x; i < W * NBIN; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  int* my = hist + wid * NBIN;
  for (int base = beg; base < end; base += 32) {
    int i = base + lane;
    if (i < end) atomicAdd(&my[(unsigned)(kin[i] >> shift) & MASK], 1);  // warp-private
  }
  __syncthreads();
  for (int b = threadIdx.x; b < NBIN; b += blockDim.x) {
    int tot = 0;
    for (int w = 0; w < W; ++w) tot += hist[w * NBIN + b];
    sc[b] = tot;
  }
  __syncthreads();
  if (wid == 0) {
    constexpr int PER = (NBIN + 31) / 32;  // digits per lane
    int v[PER], s = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = lane * PER + i;
      v[i] = b < NBIN ? sc[b] : 0;
      s += v[i];
    }
    int run = warp_incl_scan(s) - s;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = lane * PER + i;
      if (b < NBIN) sc[b] = run;
      run += v[i];
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < NBIN; b += blockDim.x) {
    int run = sc[b];
    for (int w = 0; w < W; ++w) {
      const int c = hist[w * NBIN + b];
      hist[w * NBIN + b] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int base = beg; base < end; base += 32) {
    int i = base + lane;
    const unsigned dg = (i < end) ? ((unsigned)(kin[i] >> shift) & MASK) : 0u;
    const unsigned peers = warp_match_nb<NB>(dg, i < end);
    int pos = 0;
    if (i < end) pos = my[dg] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (i < end && lane == __ffs(peers) - 1) my[dg] += __popc(peers);
    __syncwarp();
    if (i < end) {
      kout[pos] = kin[i];
      iout[pos] = iin[i];
    }
  }
  __syncthreads();
}

template <typename KeyT, typename IdxT>
__device__ int radix_sort_narrow(KeyT* kA, IdxT* iA, KeyT* kB, IdxT* iB, int n, KeyT kor,
                                 KeyT kand, int nbits, int* hist, int* sc) {
  int cur = 0;
  if (n <= 1) return 0;
  const KeyT diff = kor ^ kand;
  int lo = 0;
  while (true) {
    while (lo < nbits && ((diff >> lo) & 1) == 0) ++lo;
    if (lo >= nbits) break;
    int w = min(8, nbits - lo);
    while (w > 1 && ((diff >> (lo + w - 1)) & 1) == 0) --w;
    KeyT* ki = cur ? kB : kA;
    IdxT* ii = cur ? iB : iA;
    KeyT* ko = cur ? kA : kB;
    IdxT* io = cur ? iA : iB;
    switch (w) {
      case 1: radix_pass_nb<KeyT, IdxT, 1>(ki, ii, ko, io, n, lo, hist, sc); break;
      case 2: radix_pass_nb<KeyT, IdxT, 2>(ki, ii, ko, io, n, lo, hist, sc); break;
      case 3: radix_pass_nb<KeyT, IdxT, 3>(ki, ii, ko, io, n, lo, hist, sc); break;
      case 4: radix_pass_nb<KeyT, IdxT, 4>(ki, ii, ko, io, n, lo, hist, sc); break;
      case 5: radix_pass_nb<KeyT, IdxT, 5>(ki, ii, ko, io, n, lo, hist, sc); break;
      case 6: radix_pass_nb<KeyT, IdxT, 6>(ki, ii, ko, io, n, lo, hist, sc); break;
      case 7: radix_pass_nb<KeyT, IdxT, 7>(ki, ii, ko, io, n, lo, hist, sc); break;
      default: radix_pass_nb<KeyT, IdxT, 8>(ki, ii, ko, io, n, lo, hist, sc); break;
    }
    cur ^= 1;
    lo += w;
  }
  return cur;
}

template <typename T>
__device__ __forceinline__ T block_reduce_or(T v, T* s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(FULL, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) s[wid] = v;
  __syncthreads();
  T r = 0;
  for (int w = 0; w < nw; ++w) r |= s[w];
  __syncthreads();
  return r;
}
template <typename T>
__device__ __forceinline__ T block_reduce_and(T v, T* s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v &= __shfl_xor_sync(FULL, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) s[wid] = v;
  __syncthreads();
  T r = ~(T)0;
  for (int w = 0; w < nw; ++w) r &= s[w];
  __syncthreads();
  return r;
}

// OR and AND of every thread's key bits in one pass (redux.sync per warp, one
// barrier to combine; s holds 64 words).
__device__ __forceinline__ void block_reduce_or_and(uint32_t& o, uint32_t& a, uint32_t* s) {
  o = __reduce_or_sync(FULL, o);
  a = __reduce_and_sync(FULL, a);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) {
    s[wid] = o;
    s[32 + wid] = a;
  }
  __syncthreads();
  uint32_t ro = 0, ra = ~0u;
  for (int w = 0; w < nw; ++w) {
    ro |= s[w];
    ra &= s[32 + w];
  }
  __syncthreads();
  o = ro;
  a = ra;
}

}  // namespace rails
