// k_hist.cu -- a1: per-node send histogram + stable in-bucket rank (sm_100a).
//
// D^(1) row block of one source GPU (Alg. 1 "Select input slices for local
// experts according to Gate and E"): counts[g][h] = #(t,s) routed to global
// GPU h; msg_bytes = counts * RB for remote h (R#2); row_rank = position of (t,s)
// among the earlier slots of GPU g with the same h (R#18), which the pack needs.
//
// Batched default (>= 16 segments per SM): k_hist_w1a, one warp per (unit, node,
// source GPU), one shared count per bin, atomicAdd + read-back ranking (below), 16
// groups of ids per batch with the next batch's loads in flight, the instance -> GPU
// table in shared memory when it fits 16 KiB.  Few segments (C3: 512): k_hist_rank
// below, W warps per segment.
// k_hist_rank: one CTA per (unit, node, source GPU).  The T*k routing entries are
// split into W contiguous warp segments.  Pass 1: each warp counts its segment
// into its private shared-memory sub-histogram (shared atomics that only ever
// collide within the warp; counts are order-free).  Scan: per bin, an exclusive prefix across warps
// turns the sub-histograms into the warp's starting rank; the column total is the
// count.  Pass 2 re-walks the segment (L1/L2-resident) in 32-entry groups; the
// lanes with the same destination are found by the tag trick of k_hist_w1 (ranks
// < 2^24; with 16 warps per segment: C3 36.9 -> 28.7 us) or, for larger ranks, a
// ballot-per-bit multi-split (warp_match_bits), and rank = warp base + running count +
// peers below in the group: deterministic and identical to the sequential definition.  HBM traffic per CTA: read 4*T*k B of
// routing, write 4*T*k B of ranks + 12*G B of counts/bytes.
#include <cstdlib>

#include "common.cuh"

namespace rails {

constexpr int HR_MAX_WARPS = 16;

template <int UNR, bool TAG, bool STASH>
__global__ void __launch_bounds__(HR_MAX_WARPS * 32, 4)  // 4 x 16 warps per SM: one wave for C3
    k_hist_rank(const int32_t* __restrict__ topk, const int32_t* __restrict__ lut, int n_inst,
                int M, int N, int ngs, int d0, int nd, int T, int k, long long RB, int hbits,
                int32_t* __restrict__ counts, int64_t* __restrict__ msg,
                int32_t* __restrict__ rank, int* err) {
  extern __shared__ __align__(16) int32_t cnt[];  // [W][G], then (STASH) u16 h per entry
  pdl_trigger();  // the schedule kernel may be scheduled on the SMs this grid leaves free
  const int W = blockDim.x >> 5;
  const int G = M * N;
  const unsigned cta = blockIdx.x;  // ((u*nd) + dl)*ngs + gl  (32-bit index math)
  const unsigned ul = cta / (unsigned)ngs;
  const int d = d0 + (int)(ul % (unsigned)nd);
  const long long ne = (long long)T * k;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;

  {  // zero the sub-histograms, 16 bytes per store
    int4* c4 = reinterpret_cast<int4*>(cnt);
    const int n4 = (W * G) >> 2;
    for (int i = threadIdx.x; i < n4; i += blockDim.x) c4[i] = make_int4(0, 0, 0, 0);
    for (int i = (n4 << 2) + threadIdx.x; i < W * G; i += blockDim.x) cnt[i] = 0;
  }
  __syncthreads();

  // 32-bit indices inside the segment (T*k < 2^31: ranks are int32)
  const int nei = (int)ne;
  const int seg = (((nei + W - 1) / W) + 31) & ~31;
  const int beg = wid * seg;
  const int end = min(nei, beg + seg);
  int32_t* my = cnt + wid * G;
  bool bad = false;
  // this lane's id stream: one 64-bit base per warp segment, 32-bit offsets after it
  const int32_t* __restrict__ src = topk + (size_t)cta * (size_t)ne + beg + lane;

  // ids of one batch -> destination GPUs (-1 = invalid or past the end); all
  // loads of a batch, then all LUT lookups, are in flight together.  Full batches
  // need no bounds test (immediate offsets off one address).
  auto fetch = [&](int off, int (&hv)[UNR]) {
    if (beg + off + 32 * UNR <= end) {
#pragma unroll
      for (int j = 0; j < UNR; ++j) hv[j] = __ldg(src + off + j * 32);
    } else {
#pragma unroll
      for (int j = 0; j < UNR; ++j)
        hv[j] = (beg + off + j * 32 + lane < end) ? __ldg(src + off + j * 32) : -1;
    }
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      int h = ((unsigned)hv[j] < (unsigned)n_inst) ? __ldg(lut + hv[j]) : -1;
      hv[j] = ((unsigned)h < (unsigned)G) ? h : -1;
    }
  };

  // ---- pass 1: per-warp sub-histogram (STASH: each entry's destination kept in
  // shared memory as u16 for pass 2, instead of re-reading the id and the table)
  uint16_t* stash = reinterpret_cast<uint16_t*>(cnt + W * G) + beg + lane;
  for (int off = 0; beg + off < end; off += 32 * UNR) {
    int hv[UNR];
    fetch(off, hv);
    const bool full = beg + off + 32 * UNR <= end;  // warp-uniform: no per-entry bounds test
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const bool in = full || beg + off + j * 32 + lane < end;
      bad |= hv[j] < 0 && in;
      if (hv[j] >= 0) atomicAdd(&my[hv[j]], 1);  // private to this warp: order-free count
      if (STASH && in) stash[off + j * 32] = (uint16_t)hv[j];
    }
  }
  if (bad) flag_error(err, ERR_RANGE);
  __syncthreads();

  // ---- scan across warps per bin; totals are the counts
  for (int h = threadIdx.x; h < G; h += W * 32) {
    int run = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      int c = cnt[w * G + h];
      cnt[w * G + h] = run;
      run += c;
    }
    counts[(size_t)cta * G + h] = run;
    msg[(size_t)cta * G + h] = ((unsigned)(h - d * N) < (unsigned)N) ? 0LL : (long long)run * RB;
  }
  if (rank == nullptr) return;
  __syncthreads();

  // ---- pass 2: stable ranks
  int32_t* __restrict__ dst = rank + (size_t)cta * (size_t)ne + beg + lane;
  const unsigned lt = lanemask_lt();
  for (int off = 0; beg + off < end; off += 32 * UNR) {
    int hv[UNR];
    const bool full = beg + off + 32 * UNR <= end;
    if (STASH) {
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int v = (full || beg + off + j * 32 + lane < end) ? stash[off + j * 32] : 0xffff;
        hv[j] = v == 0xffff ? -1 : v;  // invalid entries were stashed as 0xffff
      }
    } else {
      fetch(off, hv);
    }
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const bool in = full || beg + off + j * 32 + lane < end;
      const int h = hv[j];
      const bool valid = h >= 0;
      if constexpr (TAG) {
        // equal destinations by the tag trick of k_hist_w1 below (ranks < 2^24):
        // tag byte write, one word read, a loop over the (rare) losers
        if (valid) ((uint8_t*)(my + h))[3] = (uint8_t)lane;
        __syncwarp();
        const uint32_t word = valid ? (uint32_t)my[h] : 0u;
        const int t = (int)(word >> 24);
        const int c = (int)(word & 0xffffffu);
        const bool loser = valid && t != lane;
        unsigned peers = (1u << lane) | (loser ? (1u << t) : 0u);
        unsigned lm = __ballot_sync(FULL, loser);
        while (lm) {
          const int b = __ffs(lm) - 1;
          lm &= lm - 1;
          if (__shfl_sync(FULL, h, b) == h) peers |= 1u << b;
        }
        const unsigned below = peers & lt;
        if (valid && below == 0) my[h] = (int32_t)((c + __popc(peers)) & 0xffffff);
        __syncwarp();
        if (in) dst[off + j * 32] = valid ? c + __popc(below) : -1;
      } else {
        const unsigned peers = warp_match_bits((unsigned)h, hbits, valid);
        int r = -1;
        if (valid) r = my[h] + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) my[h] += __popc(peers);
        __syncwarp();
        if (in) dst[off + j * 32] = r;
      }
    }
  }
}



// ---------------------------------------------------------------- warp-per-segment variant
// Default for batched launches (T*k <= 65535, >= 16 segments per SM).  One warp
// owns one (unit, node, source GPU): it walks the T*k routing entries once, in
// order, 32 at a time, with a private running count per bin in shared memory, so
// rank = running count + equal destinations among lower lanes and no cross-warp
// scan or second pass is needed.  16 groups of 32 ids per batch with the next
// batch's loads in flight; the instance -> GPU table staged in shared memory when it
// fits 16 KiB (its random lookups cost ~3.5 shared wavefronts per 32 ids instead of
// an L1 gather; ncu: the L1 data pipe is the kernel's saturated unit).  Ranks are
// stored as they are produced (coalesced 128 B per group); counts and bytes are
// written once at the end.
constexpr int HW_WARPS = 4;

// Atomic ranking: two shared accesses per 32 ids (a tag-trick variant needed three;
// ncu showed the L1 data pipe, shared + global wavefronts, saturated at 93.6%).
// Every lane does old = atomicAdd(&bin[h], 1) and then reads now = bin[h]; d = now - old
// is 1 for a lane with no equal key in the group, and among p lanes with the same key
// (hardware order) the d values are 1..p, so exactly one has d = 1.  Lanes with no
// collision take rank = old.  Otherwise: loop over the d >= 2 lanes (shfl of their keys)
// gives each member its d >= 2 peers (p - 1 of them), a second loop over the colliding
// d = 1 lanes adds the last one; c = now - p and the stable rank is c + #peers below.
// The count in shared memory is already c + p: no count store.
template <int UNR, bool RANK, bool SLUT>
__global__ void __launch_bounds__(HW_WARPS * 32, 8)
    k_hist_w1a(const int32_t* __restrict__ topk, const int32_t* __restrict__ lut, int n_inst,
               int M, int N, int ngs, int d0, int nd, int T, int k, long long RB,
               long long nsegs, int32_t* __restrict__ counts, int64_t* __restrict__ msg,
               int32_t* __restrict__ rank, int* err) {
  extern __shared__ __align__(16) uint32_t sw1[];
  pdl_trigger();
  const int G = M * N;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long sg = (long long)blockIdx.x * HW_WARPS + wid;
  uint32_t* const bin = sw1 + wid * (G + 1);  // bin G: sink for invalid ids
  int32_t* const ls = (int32_t*)(sw1 + (size_t)HW_WARPS * (G + 1));  // SLUT only
  if constexpr (SLUT) {
    for (int i = threadIdx.x; i < n_inst; i += HW_WARPS * 32) ls[i] = __ldg(lut + i);
    __syncthreads();
  }
  if (sg >= nsegs) return;
  const long long ul = sg / ngs;
  const int d = d0 + (int)(ul % nd);
  const int ne = T * k;
  const int32_t* __restrict__ src = topk + sg * (long long)ne + lane;
  int32_t* __restrict__ dst = RANK ? rank + sg * (long long)ne + lane : nullptr;
  for (int i = lane; i <= G; i += 32) bin[i] = 0;
  const unsigned lt = lanemask_lt();
  bool bad = false;
  __syncwarp();
  int nx[UNR];
#pragma unroll
  for (int j = 0; j < UNR; ++j) nx[j] = (j * 32 + lane < ne) ? __ldg(src + j * 32) : -1;
  for (int base = 0; base < ne; base += 32 * UNR) {
    int hv[UNR];
    const int nb = base + 32 * UNR;
#pragma unroll
    for (int j = 0; j < UNR; ++j) hv[j] = nx[j];
#pragma unroll
    for (int j = 0; j < UNR; ++j) nx[j] = (nb + j * 32 + lane < ne) ? __ldg(src + nb + j * 32) : -1;
#pragma unroll
    for (int j = 0; j < UNR; ++j)
      hv[j] = ((unsigned)hv[j] < (unsigned)n_inst) ? (SLUT ? ls[hv[j]] : __ldg(lut + hv[j]))
                                                    : -1;
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const bool in = base + j * 32 + lane < ne;
      const bool valid = (unsigned)hv[j] < (unsigned)G;
      const int h = valid ? hv[j] : G;
      bad |= in && !valid;
      const uint32_t old = atomicAdd(&bin[h], 1u);
      __syncwarp();
      const uint32_t now = bin[h];
      __syncwarp();  // the next group's atomics come after every lane's read
      const uint32_t dd = now - old;
      uint32_t r = old;
      unsigned lm = __ballot_sync(FULL, dd >= 2);
      if (lm) {
        unsigned mine = 0;  // my key's d >= 2 members
        for (unsigned m = lm; m; m &= m - 1) {
          const int b = __ffs(m) - 1;
          if (__shfl_sync(FULL, h, b) == h) mine |= 1u << b;
        }
        // colliding d = 1 lanes: one per colliding key
        unsigned l1 = __ballot_sync(FULL, dd == 1 && mine != 0);
        unsigned peers = mine;
        for (; l1; l1 &= l1 - 1) {
          const int b = __ffs(l1) - 1;
          if (__shfl_sync(FULL, h, b) == h) peers |= 1u << b;
        }
        if (mine) r = now - (uint32_t)(__popc(mine) + 1) + (uint32_t)__popc(peers & lt);
      }
      if (RANK && in) dst[base + j * 32] = valid ? (int32_t)r : -1;
    }
  }
  if (__any_sync(FULL, bad) && lane == 0) flag_error(err, ERR_RANGE);
  for (int h = lane; h < G; h += 32) {
    const int c = (int)bin[h];
    counts[sg * G + h] = c;
    msg[sg * G + h] = ((unsigned)(h - d * N) < (unsigned)N) ? 0LL : (long long)c * RB;
  }
}

template <bool TAG, bool STASH>
static cudaError_t launch_rank(const LaunchCtx& c, long long grid, int W, int M, int N, int ngs,
                               int d0, int nd, int T, int k, const int32_t* topk,
                               const int32_t* lut, int n_inst, long long RB, int hbits,
                               int32_t* counts, int64_t* msg, int32_t* rank) {
  const int seg = (int)(((T * k + W - 1) / W + 31) & ~31);  // entries per warp, padded
  const size_t smem = (size_t)W * M * N * sizeof(int32_t) +
                      (STASH ? (size_t)W * seg * sizeof(uint16_t) : 0);
  auto kern = k_hist_rank<8, TAG, STASH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, W * 32, smem, c.stream>>>(topk, lut, n_inst, M, N, ngs, d0, nd, T, k,
                                                    RB, hbits, counts, msg, rank, c.err);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_histogram(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int ngs,
                             int T, int k, const int32_t* topk, const int32_t* lut, int n_inst,
                             long long row_bytes, int32_t* counts, int64_t* msg,
                             int32_t* rank) {
  const long long grid = (long long)U * nd * ngs;
  const long long G = (long long)M * N;
  const long long ne = (long long)T * k;
  // warp-per-segment when there are enough segments to fill the GPU (>= 16 warps
  // per SM); otherwise the multi-warp-per-segment kernel keeps latency down
  if (G <= 12288 && ne <= 65535 && grid >= (long long)c.num_sms * 16) {
    size_t smem = (size_t)HW_WARPS * (G + 1) * 4;
    const bool slut = (size_t)n_inst * 4 <= 16384;
    if (slut) smem += (size_t)n_inst * 4;
    auto kern = slut ? (rank ? k_hist_w1a<16, true, true> : k_hist_w1a<16, false, true>)
                     : (rank ? k_hist_w1a<16, true, false> : k_hist_w1a<16, false, false>);
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)((grid + HW_WARPS - 1) / HW_WARPS), HW_WARPS * 32, smem, c.stream>>>(
        topk, lut, n_inst, M, N, ngs, d0, nd, T, k, row_bytes, grid, counts, msg, rank, c.err);
    count_launch(1);
    return cudaGetLastError();
  }
  // Warps per CTA: as many private sub-histograms as fit in 64 KiB (>= 1), 16 when
  // the segments alone cannot fill the SMs' warp slots with 8 (C3: 36.9 -> 28.7 us)
  int W = 1;
  if (grid * 16 <= (long long)c.num_sms * 64 && G * 16 * 4 <= 65536) W = 16;
  else if (G * 8 * 4 <= 65536) W = 8;
  else if (G * 4 * 4 <= 65536) W = 4;
  else if (G * 2 * 4 <= 98304) W = 2;
  // ranks below 2^24: the tag trick; else the per-bit ballot match on the bin index
  int hbits = 0;
  while ((1LL << hbits) < G) ++hbits;
  // pass 2 reads the destinations pass 1 stashed (u16) when they fit next to the
  // sub-histograms without costing the 4 CTAs per SM (C3: 32 + 16 KiB)
  const long long stash_bytes = (long long)W * ((((ne + W - 1) / W) + 31) & ~31LL) * 2;
  const bool stash = rank != nullptr && G < 65535 &&
                     (long long)W * G * 4 + stash_bytes <= 56 * 1024;
  if (ne < (1LL << 24) && stash)
    return launch_rank<true, true>(c, grid, W, M, N, ngs, d0, nd, T, k, topk, lut, n_inst,
                                   row_bytes, hbits, counts, msg, rank);
  if (ne < (1LL << 24))
    return launch_rank<true, false>(c, grid, W, M, N, ngs, d0, nd, T, k, topk, lut, n_inst,
                                    row_bytes, hbits, counts, msg, rank);
  return launch_rank<false, false>(c, grid, W, M, N, ngs, d0, nd, T, k, topk, lut, n_inst,
                                   row_bytes, hbits, counts, msg, rank);
}

}  // namespace rails
