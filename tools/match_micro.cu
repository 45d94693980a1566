// Micro-benchmark (not part of the library): cost per 32-lane group of finding the
// lanes with an equal key -- match.any.sync vs the per-bit ballot multi-split
// (warp_match_bits in common.cuh) for 9- and 8-bit keys -- at full occupancy.
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mm tools/match_micro.cu && /tmp/mm
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned match_bits(unsigned key, int bits) {
  unsigned peers = 0xffffffffu;
  for (int b = 0; b < bits; ++b) {
    const unsigned m = (key >> b) & 1u ? 0xffffffffu : 0u;
    const unsigned bal = __ballot_sync(0xffffffffu, (key >> b) & 1u);
    peers &= ~(bal ^ m);
  }
  return peers;
}

template <int MODE>
__global__ void k(int iters, int bits, unsigned* out) {
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    const unsigned key = (x >> 7) & ((1u << bits) - 1);
    unsigned p;
    if (MODE == 0) p = __match_any_sync(0xffffffffu, key);
    else p = match_bits(key, bits);
    acc += __popc(p & ((1u << (threadIdx.x & 31)) - 1));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out;
  const int blocks = sms * 4, threads = 512, iters = 4096;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bits : {8, 9}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<blocks, threads>>>(iters, bits, out);
        else k<1><<<blocks, threads>>>(iters, bits, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double groups = (double)blocks * threads / 32 * iters;
        if (rep == 2)
          printf("{\"bits\": %d, \"mode\": \"%s\", \"ms\": %.3f, \"groups_per_sm_per_cycle\": %.4f}\n",
                 bits, mode == 0 ? "match.any" : "ballot_bits", ms,
                 groups / sms / (ms * 1e-3 * 1.965e9));
      }
    }
  }
  return cudaGetLastError() != cudaSuccess;
}
