// k_hist.cu -- a1: per-node send histogram + stable in-bucket rank (sm_100a).
//
// D^(1) row block of one source GPU (Alg. 1 "Select input slices for local
// experts according to Gate and E"): counts[g][h] = #(t,s) routed to global
// GPU h; msg_bytes = counts * RB for remote h (R#2); row_rank = position of (t,s)
// among the earlier slots of GPU g with the same h (R#18), which the pack needs.
//
// Batched default (>= 16 segments per SM): k_hist_w1a, one warp per (unit, node,
// source GPU), one shared count per bin, atomicAdd + read-back ranking (below);
// k_hist_w1 (RAILS_HIST_ATOM=0) packs (count | tag) per bin and resolves ties inside a
// 32-entry group by a tag write / read-back and a loser-ballot loop.  Both: 16
// groups of ids per batch with the next batch's loads in flight, the instance -> GPU
// table in shared memory when it fits 16 KiB.  Few segments
// (C3: 512): k_hist_rank below, W warps per segment.
// k_hist_rank: one CTA per (unit, node, source GPU).  The T*k routing entries are
// split into W contiguous warp segments.  Pass 1: each warp counts its segment
// into its private shared-memory sub-histogram (shared atomics that only ever
// collide within the warp; counts are order-free).  Scan: per bin, an exclusive prefix across warps
// turns the sub-histograms into the warp's starting rank; the column total is the
// count.  Pass 2 re-walks the segment (L1/L2-resident) in 32-entry groups; the
// lanes with the same destination are found by the tag trick of k_hist_w1 (ranks
// < 2^24; with 16 warps per segment: C3 36.9 -> 28.7 us) or a ballot-per-bit multi-split
// (warp_match_nb, RAILS_HIST_MATCH=1), and rank = warp base + running count +
// peers below in the group: deterministic and identical to the sequential definition.  HBM traffic per CTA: read 4*T*k B of
// routing, write 4*T*k B of ranks + 12*G B of counts/bytes.
#include <cstdlib>

#include "common.cuh"

namespace rails {

template <int W, int UNR, int HB>
__global__ void __launch_bounds__(W * 32)
    k_hist_rank(const int32_t* __restrict__ topk, const int32_t* __restrict__ lut, int n_inst,
                int M, int N, int ngs, int d0, int nd, int T, int k, long long RB,
                int32_t* __restrict__ counts, int64_t* __restrict__ msg,
                int32_t* __restrict__ rank, int* err) {
  extern __shared__ int32_t cnt[];  // [W][G]
  const int G = M * N;
  const long long cta = blockIdx.x;  // ((u*nd) + dl)*ngs + gl
  const long long ul = cta / ngs;
  const int d = d0 + (int)(ul % nd);
  const long long ne = (long long)T * k;
  const int32_t* __restrict__ src = topk + cta * ne;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < W * G; i += W * 32) cnt[i] = 0;
  __syncthreads();

  // 32-bit indices inside the segment (T*k < 2^31: ranks are int32)
  const int nei = (int)ne;
  const int seg = (((nei + W - 1) / W) + 31) & ~31;
  const int beg = wid * seg;
  const int end = min(nei, beg + seg);
  int32_t* my = cnt + wid * G;
  bool bad = false;

  // ids of one batch -> destination GPUs (-1 = invalid or past the end); all
  // loads of a batch, then all LUT lookups, are in flight together
  auto fetch = [&](int base, int (&hv)[UNR]) {
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const int e = base + j * 32 + lane;
      hv[j] = (e < end) ? __ldg(src + e) : -1;
    }
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      int h = ((unsigned)hv[j] < (unsigned)n_inst) ? __ldg(lut + hv[j]) : -1;
      hv[j] = ((unsigned)h < (unsigned)G) ? h : -1;
    }
  };

  // ---- pass 1: per-warp sub-histogram
  for (int base = beg; base < end; base += 32 * UNR) {
    int hv[UNR];
    fetch(base, hv);
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      bad |= hv[j] < 0 && base + j * 32 + lane < end;
      if (hv[j] >= 0) atomicAdd(&my[hv[j]], 1);  // private to this warp: order-free count
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
    counts[cta * G + h] = run;
    msg[cta * G + h] = ((unsigned)(h - d * N) < (unsigned)N) ? 0LL : (long long)run * RB;
  }
  if (rank == nullptr) return;
  __syncthreads();

  // ---- pass 2: stable ranks
  int32_t* __restrict__ dst = rank + cta * ne;
  const unsigned lt = lanemask_lt();
  for (int base = beg; base < end; base += 32 * UNR) {
    int hv[UNR];
    fetch(base, hv);
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const int e = base + j * 32 + lane;
      const int h = hv[j];
      const bool valid = h >= 0;
      if constexpr (HB == 0) {
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
        if (e < end) dst[e] = valid ? c + __popc(below) : -1;
      } else {
        const unsigned peers = warp_match_nb<HB>((unsigned)h, valid);
        int r = -1;
        if (valid) r = my[h] + __popc(peers & lt);
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) my[h] += __popc(peers);
        __syncwarp();
        if (e < end) dst[e] = r;
      }
    }
  }
}



// ---------------------------------------------------------------- warp-per-segment variant
// Default for batched launches (T*k <= 65535, >= 16 segments per SM).  One warp
// owns one (unit, node, source GPU): it walks
// the T*k routing entries once, in order, 32 at a time, with a private running
// count per bin in shared memory, so rank = running count + equal destinations
// among lower lanes and no cross-warp scan or second pass is needed.  Each bin is
// one 32-bit shared word (running count | tag byte).  Equal destinations inside a
// group: every lane writes its lane id into the tag byte of its bin; one 32-bit
// read then returns both the surviving tag and the count; a lane that reads
// another id (a "loser") knows the winner's lane, and the winner learns its
// losers by a warp-uniform loop over the (rarely non-empty) loser ballot.  Three
// shared accesses per 32 entries (tag store, word load, leader's count store).
// Ranks are stored as they are produced (coalesced 128 B per group); counts and
// bytes are written once at the end.
constexpr int HW_WARPS = 4;

__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ASYNC: the routing ids stream through a per-warp double buffer in shared memory
// filled by cp.async two batches ahead (no registers held for the prefetch, more
// bytes in flight per SM); needs T*k % 4 == 0 for 16-byte copies.
// SLUT: the instance -> GPU table is staged in shared memory once per CTA; its random
// lookups then cost ~3.5 shared wavefronts per 32 ids instead of an L1 gather (ncu:
// the L1 data pipe, shared + global wavefronts, is the kernel's saturated unit)
template <int UNR, bool RANK, bool ASYNC = false, bool SLUT = false>
__global__ void __launch_bounds__(HW_WARPS * 32, SLUT ? 8 : 1)
    k_hist_w1(const int32_t* __restrict__ topk, const int32_t* __restrict__ lut, int n_inst,
              int M, int N, int ngs, int d0, int nd, int T, int k, long long RB,
              long long nsegs, int32_t* __restrict__ counts, int64_t* __restrict__ msg,
              int32_t* __restrict__ rank, int* err) {
  // one 32-bit word per bin: bits 0..23 running count, bits 24..31 tag (lane id)
  extern __shared__ __align__(16) uint32_t sw1[];
  const int G = M * N;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long sg = (long long)blockIdx.x * HW_WARPS + wid;  // ((u*nd)+dl)*ngs + gl
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
  // routing ids of the next batch are loaded while this batch is ranked (software
  // pipelining: the HBM latency of the stream overlaps the shared-memory work)
  int nx[ASYNC ? 1 : UNR];
  int32_t* stage = nullptr;
  const int32_t* __restrict__ seg_src = topk + sg * (long long)ne;
  auto issue = [&](int b, int buf) {  // batch starting at id b into stage[buf]
#pragma unroll
    for (int q = 0; q < UNR / 4; ++q) {
      const int i0 = b + (lane + 32 * q) * 4;
      if (i0 < ne) {
        const int nbytes = (ne - i0 >= 4 ? 4 : ne - i0) * 4;
        cp_async16(stage + buf * (UNR * 32) + (lane + 32 * q) * 4, seg_src + i0, nbytes);
      }
    }
    cp_async_commit();
  };
  if constexpr (ASYNC) {
    stage = (int32_t*)(sw1 + (((size_t)HW_WARPS * (G + 1) + 3) & ~(size_t)3)) +
            (size_t)wid * 2 * UNR * 32;
    issue(0, 0);
    issue(32 * UNR, 1);
  } else {
#pragma unroll
    for (int j = 0; j < UNR; ++j) nx[j] = (j * 32 + lane < ne) ? __ldg(src + j * 32) : -1;
  }
  int bi = 0;
  for (int base = 0; base < ne; base += 32 * UNR, ++bi) {
    int hv[UNR];
    const int nb = base + 32 * UNR;
    if constexpr (ASYNC) {
      cp_async_wait<1>();  // this batch has landed (the next may still be in flight)
      __syncwarp();
#pragma unroll
      for (int j = 0; j < UNR; ++j)
        hv[j] = (base + j * 32 + lane < ne) ? stage[(bi & 1) * (UNR * 32) + j * 32 + lane] : -1;
      __syncwarp();
      if (nb + 32 * UNR < ne) issue(nb + 32 * UNR, bi & 1);
      else cp_async_commit();  // empty group keeps the wait count aligned
    } else {
#pragma unroll
      for (int j = 0; j < UNR; ++j) hv[j] = nx[j];
#pragma unroll
      for (int j = 0; j < UNR; ++j)
        nx[j] = (nb + j * 32 + lane < ne) ? __ldg(src + nb + j * 32) : -1;
    }
#pragma unroll
    for (int j = 0; j < UNR; ++j)  // all LUT lookups of the batch in flight together
      hv[j] = ((unsigned)hv[j] < (unsigned)n_inst) ? (SLUT ? ls[hv[j]] : __ldg(lut + hv[j]))
                                                    : -1;
#pragma unroll
    for (int j = 0; j < UNR; ++j) {
      const bool in = base + j * 32 + lane < ne;
      // invalid ids (and the tail's idle lanes) all go to the sink bin G, so every
      // lane runs the same branch-free sequence
      const bool valid = (unsigned)hv[j] < (unsigned)G;
      const int h = valid ? hv[j] : G;
      bad |= in && !valid;
      // 1. tag write: for equal keys one lane's id survives
      ((uint8_t*)(bin + h))[3] = (uint8_t)lane;
      __syncwarp();
      // 2. one read gives the surviving tag and the running count
      const uint32_t word = bin[h];
      const int t = (int)(word >> 24);
      const int c = (int)(word & 0xffffffu);
      const bool loser = t != lane;
      // 3. peers: a loser knows the winner (its tag); every lane scans the losers
      // (a 5-bit ballot match on the surviving tag instead measured slower)
      unsigned peers = (1u << lane) | (loser ? (1u << t) : 0u);
      unsigned lm = __ballot_sync(FULL, loser);
      while (lm) {
        const int b = __ffs(lm) - 1;
        lm &= lm - 1;
        if (__shfl_sync(FULL, h, b) == h) peers |= 1u << b;
      }
      if (RANK && in) dst[base + j * 32] = valid ? c + __popc(peers & lt) : -1;
      // 4. the lowest lane of each key advances the count
      if ((peers & lt) == 0) bin[h] = (uint32_t)((c + __popc(peers)) & 0xffffffu);
      __syncwarp();
    }
  }
  if (__any_sync(FULL, bad) && lane == 0) flag_error(err, ERR_RANGE);
  for (int h = lane; h < G; h += 32) {
    const int c = (int)(bin[h] & 0xffffffu);
    counts[sg * G + h] = c;
    msg[sg * G + h] = ((unsigned)(h - d * N) < (unsigned)N) ? 0LL : (long long)c * RB;  // h / N == d
  }
}

// Atomic ranking (default; RAILS_HIST_ATOM=0 selects k_hist_w1 above): two shared
// accesses per 32 ids instead of three -- ncu shows the L1 data pipe (shared + global
// wavefronts) as the saturated unit of k_hist_w1 (93.6%).
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

template <int W, int HB>
static cudaError_t launch_wh(const LaunchCtx& c, long long grid, int M, int N, int ngs, int d0,
                             int nd,
                             int T, int k, const int32_t* topk, const int32_t* lut, int n_inst,
                             long long RB, int32_t* counts, int64_t* msg, int32_t* rank) {
  size_t smem = (size_t)W * M * N * sizeof(int32_t);
  auto kern = k_hist_rank<W, 8, HB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, W * 32, smem, c.stream>>>(topk, lut, n_inst, M, N, ngs, d0, nd, T, k,
                                                    RB, counts, msg, rank, c.err);
  count_launch(1);
  return cudaGetLastError();
}

// key width (bits of the largest bin index) as a template parameter
template <int W>
static cudaError_t launch_w(const LaunchCtx& c, long long grid, int M, int N, int ngs, int d0,
                            int nd,
                            int T, int k, const int32_t* topk, const int32_t* lut, int n_inst,
                            long long RB, int32_t* counts, int64_t* msg, int32_t* rank) {
  int hb = 0;
  while ((1LL << hb) < (long long)M * N) ++hb;
  // ranks below 2^24: the tag path (HB = 0) unless RAILS_HIST_MATCH=1 asks for the
  // per-bit ballot match
  const char* mv = getenv("RAILS_HIST_MATCH");
  if ((long long)T * k < (1LL << 24) && !(mv && mv[0] == '1')) hb = 0;
  switch (hb) {
#define RAILS_HB0                                                                          \
  case 0:                                                                                   \
    return launch_wh<W, 0>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, RB, counts, msg, \
                           rank);
#define RAILS_HB(B)                                                                         \
  case B:                                                                                   \
    return launch_wh<W, B>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, RB, counts, msg, \
                           rank);
    RAILS_HB0 RAILS_HB(1) RAILS_HB(2) RAILS_HB(3) RAILS_HB(4) RAILS_HB(5) RAILS_HB(6) RAILS_HB(7)
    RAILS_HB(8) RAILS_HB(9) RAILS_HB(10) RAILS_HB(11) RAILS_HB(12) RAILS_HB(13) RAILS_HB(14)
    RAILS_HB(15) RAILS_HB(16)
#undef RAILS_HB
#undef RAILS_HB0
    default:
      return cudaErrorInvalidValue;
  }
}

cudaError_t launch_histogram(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int ngs,
                             int T, int k, const int32_t* topk, const int32_t* lut, int n_inst,
                             long long row_bytes, int32_t* counts, int64_t* msg,
                             int32_t* rank) {
  const long long grid = (long long)U * nd * ngs;
  const long long G = (long long)M * N;
  const char* hv = getenv("RAILS_HIST_IMPL");
  const long long ne = (long long)T * k;
  // warp-per-segment when there are enough segments to fill the GPU (>= 16 warps
  // per SM); otherwise the multi-warp-per-segment kernels keep latency down
  const bool many = grid >= (long long)c.num_sms * 16;
  if (!(hv && (hv[0] == '1' || hv[0] == '2')) && G <= 12288 && ne <= 65535 &&
      (many || (hv && hv[0] == '3'))) {
    size_t smem = (size_t)HW_WARPS * (G + 1) * 4;
    // 16 groups of 32 routing ids per batch (measured best on C4: 8 -> 16 took the
    // batch from 0.610 to 0.573 ms); RAILS_HIST_UNR=8|32 overrides.
    // RAILS_HIST_ASYNC=1: ids through cp.async shared-memory stages (needs T*k % 4
    // == 0) -- measured slower (0.637 ms: 32 KiB per CTA costs occupancy), kept as
    // an alternative.
    const char* uv = getenv("RAILS_HIST_UNR");
    const int unr = uv ? atoi(uv) : 16;
    const char* av = getenv("RAILS_HIST_ASYNC");
    const bool async_ok = ne % 4 == 0 && av && av[0] == '1';
    // LUT in shared memory when it is small (RAILS_HIST_SLUT=0 keeps the L1 gather)
    const char* slv = getenv("RAILS_HIST_SLUT");
    const bool slut = (size_t)n_inst * 4 <= 16384 && !(slv && slv[0] == '0');
    auto kern = unr == 32 ? (rank ? k_hist_w1<32, true> : k_hist_w1<32, false>)
              : unr == 8  ? (rank ? k_hist_w1<8, true> : k_hist_w1<8, false>)
              : slut      ? (rank ? k_hist_w1<16, true, false, true> : k_hist_w1<16, false, false, true>)
                          : (rank ? k_hist_w1<16, true> : k_hist_w1<16, false>);
    if (slut && !async_ok && unr == 16) smem += (size_t)n_inst * 4;
    // atomic-add ranking by default (C4 0.545 -> 0.481 ms); RAILS_HIST_ATOM=0 keeps the
    // tag-trick kernel
    const char* atv = getenv("RAILS_HIST_ATOM");
    if (!(atv && atv[0] == '0') && unr == 16 && !async_ok)
      kern = slut ? (rank ? k_hist_w1a<16, true, true> : k_hist_w1a<16, false, true>)
                  : (rank ? k_hist_w1a<16, true, false> : k_hist_w1a<16, false, false>);
    if (async_ok) {
      kern = rank ? k_hist_w1<16, true, true> : k_hist_w1<16, false, true>;
      smem = (((size_t)HW_WARPS * (G + 1) + 3) & ~(size_t)3) * 4 +
             (size_t)HW_WARPS * 2 * 16 * 32 * 4;
    }
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)((grid + HW_WARPS - 1) / HW_WARPS), HW_WARPS * 32, smem, c.stream>>>(
        topk, lut, n_inst, M, N, ngs, d0, nd, T, k, row_bytes, grid, counts, msg, rank, c.err);
    count_launch(1);
    return cudaGetLastError();
  }
  // Warps per CTA: as many private sub-histograms as fit in 64 KiB (>= 1); 16 when
  // the segments alone cannot fill the SMs' warp slots with 8 (RAILS_HIST_W=8|16|32
  // overrides).
  const char* wv = getenv("RAILS_HIST_W");
  const int wo = wv ? atoi(wv) : 0;
  if (wo == 32 && G * 32 * 4 <= 65536)
    return launch_w<32>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, row_bytes, counts,
                        msg, rank);
  if ((wo == 16 || (wo == 0 && grid * 16 <= (long long)c.num_sms * 64)) && G * 16 * 4 <= 65536)
    return launch_w<16>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, row_bytes, counts,
                        msg, rank);
  if (G * 8 * 4 <= 65536)
    return launch_w<8>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, row_bytes, counts, msg,
                       rank);
  if (G * 4 * 4 <= 65536)
    return launch_w<4>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, row_bytes, counts, msg,
                       rank);
  if (G * 2 * 4 <= 98304)
    return launch_w<2>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, row_bytes, counts, msg,
                       rank);
  return launch_w<1>(c, grid, M, N, ngs, d0, nd, T, k, topk, lut, n_inst, row_bytes, counts, msg,
                     rank);
}

}  // namespace rails
