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
