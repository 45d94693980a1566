// k_sched.cu -- the generic atomic-flow LPT entry rails_lpt_assign ("small
// application-layer messages") on sm_100a.  The hot-path schedule of
// (unit, node) message matrices is the fused kernel of k_node.cu.
//
// One CTA per flow set: stable radix sort of the weights descending (key ~w, index
// order among equal weights = the tie-break of R#4), then warp 0 runs Alg. 2 step 3
// with a 64-bit butterfly argmin over (load, rail): lowest-index rail on
// ties (R#5), offset = LoadState before the add (R#19).
#include <climits>

#include "common.cuh"
#include "radix.cuh"

namespace rails {

constexpr int SORT_THREADS = 512;

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
