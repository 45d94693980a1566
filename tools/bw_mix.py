#!/usr/bin/env python
"""Achievable HBM bandwidth for the pack's access mix, without the pack's logic.

Plain streaming kernels (built here with torch.utils.cpp_extension, sm_100a) over
8 KiB rows, one warp per row, 16-byte vectors, grid = SMs x 1..128 CTAs (best kept):
  copy_1r1w   read a row, write it once (same layout)            -- 1:1 copy
  dup_1r2w    read a row, write it to two separate buffers       -- the pack's 1:2 mix
  dup_1r2w_x  as dup_1r2w, destinations permuted by a row hash   -- scattered rows
Reports GB/s of (read + written) bytes, CUDA events, L2-exceeding buffers.  Context
for the pack's roofline fraction, not a bench line.
"""
import json
import os
import sys

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
#include <cuda_runtime.h>
#include <c10/cuda/CUDAStream.h>

template <int MODE>
__global__ void __launch_bounds__(256) k_mix(const uint4* __restrict__ x, uint4* __restrict__ a,
                                             uint4* __restrict__ b, long long rows) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * 8;
  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += nw) {
    uint4 v[16];
    const uint4* s = x + r * 512;
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __ldcs(s + i * 32 + lane);
    long long ra = r, rb = r;
    if (MODE == 2) {  // scattered destinations: a multiplicative permutation of rows
      ra = (r * 40503LL) % rows;
      rb = (r * 69069LL + 1) % rows;
    }
    uint4* da = a + ra * 512;
#pragma unroll
    for (int i = 0; i < 16; ++i) __stcs(da + i * 32 + lane, v[i]);
    if (MODE >= 1) {
      uint4* db = b + rb * 512;
#pragma unroll
      for (int i = 0; i < 16; ++i) __stcs(db + i * 32 + lane, v[i]);
    }
  }
}

void run(torch::Tensor x, torch::Tensor a, torch::Tensor b, int64_t mode, int64_t grid) {
  const long long rows = x.numel() / 8192;
  auto st = c10::cuda::getCurrentCUDAStream();
  auto X = (const uint4*)x.data_ptr(); auto A = (uint4*)a.data_ptr(); auto B = (uint4*)b.data_ptr();
  if (mode == 0) k_mix<0><<<grid, 256, 0, st>>>(X, A, B, rows);
  else if (mode == 1) k_mix<1><<<grid, 256, 0, st>>>(X, A, B, rows);
  else k_mix<2><<<grid, 256, 0, st>>>(X, A, B, rows);
}
"""
CPP = "void run(torch::Tensor x, torch::Tensor a, torch::Tensor b, int64_t mode, int64_t grid);"


def main():
    mod = load_inline("bw_mix", CPP, cuda_sources=SRC, functions=["run"],
                      extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                      build_directory=None, verbose=False)
    dev = "cuda:0"
    n = 4 << 30  # 4 GiB of source rows (>> L2)
    x = torch.empty(n, dtype=torch.uint8, device=dev).random_(0, 255)
    a = torch.empty(n, dtype=torch.uint8, device=dev)
    b = torch.empty(n, dtype=torch.uint8, device=dev)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "MEASURED_PEAKS.json")
    peak = json.load(open(peaks))["hbm_gbs"] if os.path.exists(peaks) else None
    res = {"device": torch.cuda.get_device_name(0), "peak_gbs": peak, "bytes_src": n}
    for name, mode, mult in (("copy_1r1w", 0, 2), ("dup_1r2w", 1, 3), ("dup_1r2w_x", 2, 3)):
        best = None
        for per_sm in (1, 2, 4, 8, 16, 32, 64, 128):
            g = sms * per_sm
            for _ in range(2):
                mod.run(x, a, b, mode, g)
            torch.cuda.synchronize()
            ts = []
            for _ in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                mod.run(x, a, b, mode, g)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[len(ts) // 2]
            gbs = mult * n / (ms / 1e3) / 1e9
            print(name, per_sm, round(gbs), file=sys.stderr)
            if best is None or gbs > best["gbs"]:
                best = {"ctas_per_sm": per_sm, "median_ms": ms, "gbs": gbs,
                        "frac": gbs / peak if peak else None}
        res[name] = best
        print(name, best, file=sys.stderr)
    s = json.dumps(res, indent=1)
    print(s)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(s)


if __name__ == "__main__":
    main()
