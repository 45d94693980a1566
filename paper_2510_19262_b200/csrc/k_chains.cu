// k_chains.cu -- the schedule (a2-a4) of MANY (unit, node) segments at once: C2's
// 16 000 iterations, a C4 iteration's 4 096 (node, layer) units (sm_100a).
//
// Same method and outputs as the fused per-node kernel (k_node.cu, whose header
// states the chunking, sort and closed form), split into kernels that each run at
// their own best occupancy, which wins once the segments oversubscribe the GPU:
//   k_chunk_sort  1 CTA per segment: full_base scan + remainder compaction (a2), then
//                 the stable LSD radix sort of the remainder keys C-1-size (a3, R#4);
//                 writes the sorted sizes and the inverse permutation;
//   k_lpt_wstage  1 WARP per segment (4 per CTA), N = 8, C < 2^23: the sorted-register
//                 LPT network of lpt.cuh with the size list staged through shared
//                 memory one batch ahead (a4);  k_lpt_chain: any N / C, lane j holds
//                 rail j's load, argmin by redux.sync (or a 64-bit butterfly);
//   k_qp_rank     the QP map (Alg. 2 step 4, R#34) when asked;
//   k_expand      results (sorted order) -> per-message rem_rail / rem_off, four
//                 messages per thread with their gathers in flight together.
#include "common.cuh"
#include "lpt.cuh"
#include "radix.cuh"

namespace rails {

constexpr int SORT_THREADS = 256;
constexpr int CS_NARROW_MINB = 8;  // 128-thread sorts (N*G <= 2048): 64 registers, 8 CTAs per SM

template <typename KeyT, typename IdxT, bool SMEM, int MAXT = SORT_THREADS, int MINB = 3>
__global__ void __launch_bounds__(MAXT, MINB)
    k_chunk_sort(const int64_t* __restrict__ msg, long long NG, int N, int d0, int nd,
                 long long C, int cshift, int nbits, int64_t* __restrict__ full_base,
                 int32_t* __restrict__ ws_inv, int64_t* __restrict__ n_full_out,
                 int32_t* __restrict__ n_rem_out, uint32_t* __restrict__ ws_w,
                 uint8_t* __restrict__ ws_scratch, int use_smem,
                 int* err) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ long long scan_scratch[33];
  __shared__ int hist[(SORT_THREADS / 32) * 256];
  __shared__ int sc[256];
  __shared__ uint32_t red32[64];

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

  // Pass over the messages in tiles of blockDim.x * IPT, each thread owning IPT
  // consecutive messages: its loads are all in flight at once and one block scan
  // per tile gives the running (full chunks, remainders) prefix.
  constexpr int IPT = 8;
  long long carry_full = 0;
  int carry_rem = 0;
  KeyT kor = 0, kand = (KeyT)~(KeyT)0;
  int64_t* __restrict__ fbg = full_base + seg * NG;
  const bool vec = aligned32(mg) && aligned32(fbg);  // 256-bit accesses (ld8/st8_s64)
  bool bad_range = false, bad_ovf = false;  // flagged once after the pass
  // later tiles' messages requested into L2 now (their loads then wait on L2, not
  // DRAM, behind each tile's block scan)
  for (long long t0 = (long long)blockDim.x * IPT; t0 < NG; t0 += (long long)blockDim.x * IPT) {
    const long long m0 = t0 + (long long)threadIdx.x * IPT;
    if (m0 < NG) asm volatile("prefetch.global.L2 [%0];" ::"l"(mg + m0));
  }
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
    // destination GPU h = m mod G of the first item, then stepped (one division
    // per thread and tile instead of one per message)
    int h = (int)((unsigned long long)m0 % (unsigned long long)G);
    const int lo = d * N, hi = d * N + N;  // the source node's own GPUs (R#2)
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      // negative bytes, or bytes to a GPU of the source node (R#2), are invalid
      const bool inval = B[j] < 0 || (B[j] != 0 && h >= lo && h < hi);
      bad_range |= inval;
      if (inval) B[j] = 0;
      if (++h >= G) h -= G;
      nfv[j] = cd.div(B[j]);
      bad_ovf |= nfv[j] >= (1LL << 40);
      snf += nfv[j];
      srem += (B[j] - nfv[j] * C) > 0;
    }
    long long tot;
    const long long ex = block_excl_scan((snf << 16) | srem, scan_scratch, &tot);
    long long fb = carry_full + (ex >> 16);
    int pos = carry_rem + (int)(ex & 0xffff);
    long long fbv[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const long long m = m0 + j;
      if (m >= NG) break;
      const long long nf = nfv[j];
      const long long rem = B[j] - nf * C;
      fbv[j] = fb;
      if (!whole) fbg[m] = fb;
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
    if (whole) st8_s64(fbg + m0, fbv);
    carry_full += tot >> 16;
    carry_rem += (int)(tot & 0xffff);
  }
  if (bad_range) flag_error(err, ERR_RANGE);
  if (bad_ovf) flag_error(err, ERR_OVERFLOW);
  {
    uint32_t o = kor, an = kand;
    block_reduce_or_and(o, an, red32);
    kor = (KeyT)o;
    kand = (KeyT)an;
  }
  if (threadIdx.x == 0) {
    n_full_out[seg] = carry_full;
    n_rem_out[seg] = carry_rem;
  }
  __syncthreads();
  const int n = carry_rem;
  const int which =
      radix_sort_narrow<KeyT, IdxT>(kA, iA, kB, iB, n, kor, kand, nbits, hist, sc);
  const KeyT* ks = which ? kB : kA;
  const IdxT* is = which ? iB : iA;
  // inverse permutation in the free index buffer, then written out coalesced
  // (message m -> sorted position of its remainder, -1 if none)
  IdxT* inv = which ? iA : iB;
  constexpr IdxT NONE = (IdxT)~(IdxT)0;
  for (long long m = threadIdx.x; m < NG; m += blockDim.x) inv[m] = NONE;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ws_w[seg * NG + i] = (uint32_t)(C - 1 - (long long)ks[i]);
    inv[is[i]] = (IdxT)i;
  }
  __syncthreads();
  for (long long m = threadIdx.x; m < NG; m += blockDim.x)
    ws_inv[seg * NG + m] = inv[m] == NONE ? -1 : (int32_t)inv[m];
}

// ---------------------------------------------------------------- a4 chains
constexpr int CHAIN_WARPS = 4;

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

// Few long chains or many: one chain per warp.  All 32 lanes stream the sorted
// remainder list through a double-buffered shared-memory stage filled by cp.async
// (512 sizes per batch, one batch ahead, no staging registers: 62 registers), and all
// run the same (warp-uniform) register state.  A run of
// >= 32 equal sizes -- routing traffic has only C / row_bytes distinct remainder
// sizes -- is assigned by single network steps until the cyclic condition holds,
// then written by the whole warp (lpt_run_cyclic); other items go eight at a time
// through lpt_group8_v with lane 0 storing.
constexpr int WS_WARPS = 4;
constexpr int WS_BATCH = 512;

template <int NT>
__global__ void __launch_bounds__(WS_WARPS * 32, 7)  // <= 72 registers: C4 (1024 CTAs) fits one wave
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
  // batch b (WS_BATCH sizes) -> sW[wid][buf] by cp.async (zero-filled past nr): the
  // next batch lands in shared memory while this one is assigned, with no registers
  auto issue = [&](int b, int buf) {
#pragma unroll
    for (int p = 0; p < PL; ++p) {
      const int i = b + p * 32 + lane;
      const bool in = i < nr;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&sW[wid][buf][p * 32 + lane]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst),
                   "l"(in ? gw + i : gw), "r"(in ? 4 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0, 0);
  int cur = 0;
  for (int b0 = 0; b0 < nr; b0 += WS_BATCH) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (b0 + WS_BATCH < nr) issue(b0 + WS_BATCH, cur ^ 1);
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
          e += __popc(__ballot_sync(0xffffffffu, j >= i && j < cnt && w_[j] == w));
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

// QP map (Alg. 2 step 4, R#34) of every segment: one CTA each (lpt.cuh).
__global__ void __launch_bounds__(256)
    k_qp_rank(int N, int Q, long long NG, const int64_t* __restrict__ n_full,
              const int32_t* __restrict__ n_rem, const uint64_t* __restrict__ ws_res,
              uint32_t* __restrict__ ws_qp) {
  const long long seg = blockIdx.x;
  qp_rank_block(N, Q, n_full[seg], n_rem[seg], ws_res + seg * NG, ws_qp + seg * NG);
}

// Expand the sorted-order chain results into per-message rem_rail / rem_off: message
// m has a remainder iff ws_inv[m] >= 0 (its sorted position).  Four consecutive
// messages per thread, their dependent gathers in flight together (one per thread
// measured latency-bound: two dependent loads per message).  Segments beyond
// gridDim.y are looped.
__global__ void __launch_bounds__(256)
    k_expand(long long NG, long long nseg, const int32_t* __restrict__ ws_inv,
             const uint64_t* __restrict__ ws_res, int8_t* __restrict__ rem_rail,
             int64_t* __restrict__ rem_off, const uint32_t* __restrict__ ws_qp,
             int32_t* __restrict__ rem_qp) {
  const long long m0 = ((long long)blockIdx.x * 256 + threadIdx.x) * 4;
  if (m0 >= NG) return;
  for (long long seg = blockIdx.y; seg < nseg; seg += gridDim.y) {
    const long long b = seg * NG;
    int p[4];
    uint64_t v[4];
    uint32_t qv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = m0 + i < NG ? ws_inv[b + m0 + i] : -1;
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = p[i] >= 0 ? ws_res[b + p[i]] : 0ull;
    if (rem_qp) {
#pragma unroll
      for (int i = 0; i < 4; ++i) qv[i] = p[i] >= 0 ? ws_qp[b + p[i]] : 0u;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (m0 + i >= NG) break;
      rem_rail[b + m0 + i] = p[i] >= 0 ? (int8_t)(v[i] >> 56) : (int8_t)-1;
      rem_off[b + m0 + i] = p[i] >= 0 ? (long long)(v[i] & (uint64_t)OFF_MASK) : 0;
      if (rem_qp) rem_qp[b + m0 + i] = p[i] >= 0 ? (int32_t)qv[i] : -1;
    }
  }
}

// workspace (within rails_schedule_workspace's buffer, after the fused kernel's
// accumulators): res u64 | qp u32 | sizes u32 | inverse permutation i32 | sort spill
cudaError_t launch_chains(const LaunchCtx& c, int U, int nd, int d0, int M, int N, long long C,
                          const int64_t* msg, const rails_sched_t& s, uint64_t* ws_res,
                          uint32_t* ws_qp, uint32_t* ws_w, int32_t* ws_inv, uint8_t* scratch,
                          int32_t* rem_qp, int qps_per_rail, int cshift, int nbits,
                          bool defer_expand) {
  const long long nseg = (long long)U * nd;
  const long long NG = (long long)N * M * N;
  cudaError_t e;
  const bool k16 = C <= 65536;
  const size_t smem = (size_t)NG * (2 * (k16 ? 2 : 4) + 2 * sizeof(uint16_t));
  if (NG <= 16384 && smem <= 200 * 1024) {
    // 16-bit keys when C <= 65536 and 16-bit indices: several CTAs per SM
    const int thr = NG <= 2048 ? 128 : SORT_THREADS;
    auto kern = thr == 128
                    ? (k16 ? k_chunk_sort<uint16_t, uint16_t, true, 128, CS_NARROW_MINB>
                           : k_chunk_sort<uint32_t, uint16_t, true, 128, CS_NARROW_MINB>)
                    : (k16 ? k_chunk_sort<uint16_t, uint16_t, true>
                           : k_chunk_sort<uint32_t, uint16_t, true>);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)nseg, thr, smem, c.stream>>>(msg, NG, N, d0, nd, C, cshift, nbits,
                                                  s.full_base, ws_inv, s.n_full, s.n_rem, ws_w,
                                                  nullptr, 1, c.err);
  } else {
    k_chunk_sort<uint32_t, uint32_t, false><<<(unsigned)nseg, SORT_THREADS, 0, c.stream>>>(
        msg, NG, N, d0, nd, C, cshift, nbits, s.full_base, ws_inv, s.n_full, s.n_rem, ws_w,
        scratch, 0, c.err);
  }
  count_launch(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (N == 8 && C < (1LL << 23)) {
    k_lpt_wstage<8><<<(unsigned)((nseg + WS_WARPS - 1) / WS_WARPS), WS_WARPS * 32, 0, c.stream>>>(
        nseg, C, NG, s.n_full, s.n_rem, ws_w, ws_res, s.send_load);
  } else {
    k_lpt_chain<<<(unsigned)((nseg + CHAIN_WARPS - 1) / CHAIN_WARPS), CHAIN_WARPS * 32, 0,
                  c.stream>>>(nseg, N, C, NG, s.n_full, s.n_rem, ws_w, ws_res, s.send_load, c.err);
  }
  count_launch(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (rem_qp) {
    k_qp_rank<<<(unsigned)nseg, 256, 0, c.stream>>>(N, qps_per_rail, NG, s.n_full, s.n_rem,
                                                    ws_res, ws_qp);
    count_launch(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (defer_expand && !rem_qp) return cudaSuccess;  // the evaluation expands (k_eval.cu)
  const long long gy = nseg < 65535 ? nseg : 65535;
  k_expand<<<dim3((unsigned)((NG / 4 + 256) / 256), (unsigned)gy), 256, 0, c.stream>>>(
      NG, nseg, ws_inv, ws_res, s.rem_rail, s.rem_off, rem_qp ? ws_qp : nullptr, rem_qp);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace rails
