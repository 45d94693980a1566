// k_pack.cu -- a7: scatter token rows into rail-ordered send buffers (sm_100a).
//
// Message (g,h) of node d is the concatenation, in ascending (t,s), of the RB-byte
// rows x[g][t] of every remote slot routed to GPU h (R#18, R#20); the copy of rank
// rho occupies message bytes [rho*RB, (rho+1)*RB).  Chunk c of the message lands at
// rail_base[rail(c)] + off(c) (R#19) where, from the compact LPT schedule, full
// chunk c (c < floor(B/C)) has node-global index i = full_base + c -> rail i mod N,
// offset floor(i/N)*C, and the remainder chunk has (rem_rail, rem_off).
//
// The pack is input-driven and HBM-bound: every source row is read from HBM once
// (16-byte streaming loads, all of a warp's loads in flight before its first store)
// and each remote copy is written with 16-byte streaming stores, 512 contiguous
// bytes per warp instruction, split only at chunk boundaries (all offsets are
// multiples of 16 because RB and C are).  Persistent grid: one warp per row, rows
// strided over (SM count x resident warps).  Slot metadata (routing -> LUT ->
// message tables -> rail base) is computed by lanes 0..k-1 while the row's payload
// loads are in flight, then broadcast by shuffle.
//   MULTI = false: C >= RB, a row copy spans at most two chunks.
//   MULTI = true : C <  RB, the chunk of every 16-byte vector is computed.
#include <cstdlib>

#include "common.cuh"

namespace rails {

constexpr int PACK_THREADS = 256;

struct SlotMeta {
  long long dst0;   // output byte address of row byte 0
  long long dst1;   // output byte address of the start of chunk c0+1 (MULTI=false)
  long long p0;     // message byte of row byte 0 (rho * RB)
  long long fb;     // full_base of the message
  long long nfull;  // floor(B / C)
  long long ro;     // rem_off
  int b0;           // row bytes that fall in chunk c0
  int rr;           // rem_rail
  int ok;           // remote and valid
};

__device__ __forceinline__ long long chunk_addr(long long c, long long fb, long long nfull,
                                                int rr, long long ro, int N, long long C,
                                                const int64_t* __restrict__ rbase) {
  if (c < nfull) {
    const long long i = fb + c;
    const long long q = i / N;
    return rbase[i - q * N] + q * C;
  }
  return rr >= 0 ? rbase[rr] + ro : -(1LL << 62);
}

template <int VPL, bool MULTI, int CS = 0>
__global__ void __launch_bounds__(PACK_THREADS)
    k_pack(int U, int nd, int d0, int M, int N, int T, int k, long long C, int cshift,
           const uint4* __restrict__ x, const int32_t* __restrict__ topk,
           const int32_t* __restrict__ lut, int n_inst, const int32_t* __restrict__ rank,
           const int64_t* __restrict__ msg, long long RB, const int64_t* __restrict__ full_base,
           const int8_t* __restrict__ rem_rail, const int64_t* __restrict__ rem_off,
           const int64_t* __restrict__ rail_base, uint8_t* __restrict__ out, long long out_cap,
           int* err) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (PACK_THREADS / 32);
  const long long rows = (long long)U * nd * N * T;
  const long long G = (long long)M * N;
  const int nvec = (int)(RB >> 4);
  const ChunkDiv cd{C, cshift};

  for (long long row = (long long)blockIdx.x * (PACK_THREADS / 32) + (threadIdx.x >> 5);
       row < rows; row += nwarps) {
    const long long ug = row / T;  // (u*nd + dl)*N + g
    const long long ul = ug / N;
    const int d = d0 + (int)(ul % nd);
    const uint4* __restrict__ src = x + row * nvec;
    const int64_t* __restrict__ rbase = rail_base + ul * N;

    // 1. payload loads of the first window (all in flight)
    uint4 v[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int vi = i * 32 + lane;
      if (vi < nvec) v[i] = (CS & 2) ? __ldcs(src + vi) : ld_stream(src + vi);
    }

    // 2. slot metadata on lanes 0..k-1
    SlotMeta sm{0, 0, 0, 0, 0, 0, 0, -1, 0};
    if (lane < k) {
      const long long e = row * k + lane;
      const int inst = __ldg(topk + e);
      int h = (inst >= 0 && inst < n_inst) ? __ldg(lut + inst) : -1;
      if (h < 0 || h >= G) {
        flag_error(err, ERR_RANGE);
        h = -1;
      }
      if (h >= 0 && h / N != d) {
        const long long mi = ug * G + h;
        const long long B = msg[mi];
        const int rk = rank[e];
        sm.p0 = (long long)rk * RB;
        if (rk < 0 || sm.p0 + RB > B) {
          flag_error(err, ERR_RANGE);
        } else {
          sm.fb = full_base[mi];
          sm.nfull = cd.div(B);
          sm.rr = rem_rail[mi];
          sm.ro = rem_off[mi];
          const long long c0 = cd.div(sm.p0);
          sm.dst0 = chunk_addr(c0, sm.fb, sm.nfull, sm.rr, sm.ro, N, C, rbase) + (sm.p0 - c0 * C);
          const long long b0 = (c0 + 1) * C - sm.p0;
          sm.b0 = (int)(b0 < RB ? b0 : RB);
          if (!MULTI && sm.b0 < RB)
            sm.dst1 = chunk_addr(c0 + 1, sm.fb, sm.nfull, sm.rr, sm.ro, N, C, rbase);
          sm.ok = 1;
        }
      }
    }

    // 3. stores, window by window
    for (int w0 = 0; w0 < nvec; w0 += VPL * 32) {
      if (w0 > 0) {
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int vi = w0 + i * 32 + lane;
          if (vi < nvec) v[i] = (CS & 2) ? __ldcs(src + vi) : ld_stream(src + vi);
        }
      }
      for (int s = 0; s < k; ++s) {
        if (!__shfl_sync(FULL, sm.ok, s)) continue;
        const long long D0 = __shfl_sync(FULL, sm.dst0, s);
        const int B0 = __shfl_sync(FULL, sm.b0, s);
        if (!MULTI) {
          const long long D1 = __shfl_sync(FULL, sm.dst1, s);
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            const int vi = w0 + i * 32 + lane;
            if (vi < nvec) {
              const long long o = (long long)vi << 4;
              const long long a = (o < B0) ? D0 + o : D1 + (o - B0);
              if (a >= 0 && a + 16 <= out_cap) {
                if (CS & 1)
                  st_cs((uint4*)(out + a), v[i]);
                else
                  st_stream((uint4*)(out + a), v[i]);
              } else {
                flag_error(err, ERR_NOSPC);
              }
            }
          }
        } else {
          const long long P0 = __shfl_sync(FULL, sm.p0, s);
          const long long FB = __shfl_sync(FULL, sm.fb, s);
          const long long NF = __shfl_sync(FULL, sm.nfull, s);
          const long long RO = __shfl_sync(FULL, sm.ro, s);
          const int RR = __shfl_sync(FULL, sm.rr, s);
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            const int vi = w0 + i * 32 + lane;
            if (vi < nvec) {
              const long long o = (long long)vi << 4;
              long long a;
              if (o < B0) {
                a = D0 + o;
              } else {
                const long long p = P0 + o;
                const long long c = cd.div(p);
                a = chunk_addr(c, FB, NF, RR, RO, N, C, rbase) + (p - c * C);
              }
              if (a >= 0 && a + 16 <= out_cap)
                st_stream((uint4*)(out + a), v[i]);
              else
                flag_error(err, ERR_NOSPC);
            }
          }
        }
      }
    }
  }
}

template <int VPL, bool MULTI>
static cudaError_t launch_v(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T, int k,
                            long long C, int cshift, const void* x, const int32_t* topk,
                            const int32_t* lut, int n_inst, const int32_t* rank,
                            const int64_t* msg, long long RB, const rails_sched_t& s,
                            const int64_t* rail_base, void* out, long long out_cap) {
  // RAILS_PACK_ST: bit 0 = .cs (evict-first) stores, bit 1 = .cs payload loads
  const char* st = getenv("RAILS_PACK_ST");
  const int cs = st ? atoi(st) : 0;
  auto kern = cs == 1 ? k_pack<VPL, MULTI, 1> : cs == 2 ? k_pack<VPL, MULTI, 2>
            : cs == 3 ? k_pack<VPL, MULTI, 3> : k_pack<VPL, MULTI, 0>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PACK_THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long rows = (long long)U * nd * N * T;
  const long long need = (rows + PACK_THREADS / 32 - 1) / (PACK_THREADS / 32);
  // waves of CTAs, ~8 rows per warp (wave_grid); RAILS_PACK_CTAS sets CTAs per SM
  long long grid;
  const char* pv = getenv("RAILS_PACK_CTAS");
  if (pv && atoi(pv) >= 1) {
    grid = (long long)c.num_sms * atoi(pv);
    if (grid > need) grid = need;
  } else {
    grid = wave_grid(c.num_sms, per_sm, need, "RAILS_PACK_RPW");
  }
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, PACK_THREADS, 0, c.stream>>>(
      U, nd, d0, M, N, T, k, C, cshift, (const uint4*)x, topk, lut, n_inst, rank, msg, RB,
      s.full_base, s.rem_rail, s.rem_off, rail_base, (uint8_t*)out, out_cap, c.err);
  count_launch(1);
  return cudaGetLastError();
}

template <bool MULTI>
static cudaError_t launch_m(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T, int k,
                            long long C, int cshift, const void* x, const int32_t* topk,
                            const int32_t* lut, int n_inst, const int32_t* rank,
                            const int64_t* msg, long long RB, const rails_sched_t& s,
                            const int64_t* rail_base, void* out, long long out_cap) {
  const long long nvec = RB >> 4;
  long long vpl = (nvec + 31) / 32;
  // tuning knob: RAILS_PACK_VPL caps the 16-byte vectors held per lane (the row is
  // then copied in windows; fewer registers, more resident warps)
  if (const char* ev = getenv("RAILS_PACK_VPL")) {
    const long long cap = atoll(ev);
    if (cap >= 1 && cap < vpl) vpl = cap;
  }
#define RAILS_PACK_CASE(V)                                                                  \
  if (vpl <= V)                                                                             \
    return launch_v<V, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank, \
                              msg, RB, s, rail_base, out, out_cap);
  RAILS_PACK_CASE(1)
  RAILS_PACK_CASE(2)
  RAILS_PACK_CASE(4)
  RAILS_PACK_CASE(8)
#undef RAILS_PACK_CASE
  // rows longer than 8 KiB are copied in 8 KiB windows: 16 vectors per lane keep
  // enough warps resident (C4's 12 KiB rows: 90% of the copy peak vs 87% with the
  // whole row in 24 registers-worth of vectors)
  return launch_v<16, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank,
                             msg, RB, s, rail_base, out, out_cap);
}

// ---------------------------------------------------------------- TMA-staged variant
// Same contract as k_pack.  Each warp is an independent bulk-copy pipeline with S
// shared-memory row stages: lane 0 issues cp.async.bulk global->shared row loads
// D rows ahead (completion on a per-stage mbarrier with expect_tx), then, for the
// current row, one cp.async.bulk shared->global store per piece (a piece = the part
// of a remote copy inside one chunk; 1-2 pieces when C >= RB), committed as one
// bulk group.  A stage is reloaded only after cp.async.bulk.wait_group.read shows
// its previous stores have read it.  No payload byte passes through registers.
// Slot metadata for row j+D is computed by lanes 0..k-1 into shared memory when
// the row's load is issued, so its latency is hidden behind D rows of copies.
constexpr int TMA_WARPS = 4;
constexpr int TMA_MAXK = 8;

struct TmaMeta {
  long long dst0, dst1, p0, fb, nfull, ro;
  int b0, rr, ok, pad;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int S, int D, bool MULTI>
__global__ void __launch_bounds__(TMA_WARPS * 32)
    k_pack_tma(int U, int nd, int d0, int M, int N, int T, int k, long long C, int cshift,
               const uint8_t* __restrict__ x, const int32_t* __restrict__ topk,
               const int32_t* __restrict__ lut, int n_inst, const int32_t* __restrict__ rank,
               const int64_t* __restrict__ msg, long long RB,
               const int64_t* __restrict__ full_base, const int8_t* __restrict__ rem_rail,
               const int64_t* __restrict__ rem_off, const int64_t* __restrict__ rail_base,
               uint8_t* __restrict__ out, long long out_cap, int* err) {
  static_assert(D >= 1 && D < S, "prefetch distance");
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t bars[TMA_WARPS][S];
  __shared__ TmaMeta meta[TMA_WARPS][S][TMA_MAXK];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * TMA_WARPS;
  const long long rows = (long long)U * nd * N * T;
  const long long G = (long long)M * N;
  const ChunkDiv cd{C, cshift};
  uint8_t* buf = sbuf + (size_t)wid * S * RB;
  uint64_t* bar = bars[wid];
  const long long row0 = (long long)blockIdx.x * TMA_WARPS + wid;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // metadata of row `row` into meta[wid][st][lane] (lanes < k)
  auto make_meta = [&](long long row, int st) {
    if (lane >= k) return;
    TmaMeta m{0, 0, 0, 0, 0, 0, 0, -1, 0, 0};
    const long long ug = row / T;
    const long long ul = ug / N;
    const int d = d0 + (int)(ul % nd);
    const int64_t* __restrict__ rbase = rail_base + ul * N;
    const long long e = row * k + lane;
    const int inst = __ldg(topk + e);
    int h = (inst >= 0 && inst < n_inst) ? __ldg(lut + inst) : -1;
    if (h < 0 || h >= G) {
      flag_error(err, ERR_RANGE);
      h = -1;
    }
    if (h >= 0 && h / N != d) {
      const long long mi = ug * G + h;
      const long long B = msg[mi];
      const int rk = rank[e];
      m.p0 = (long long)rk * RB;
      if (rk < 0 || m.p0 + RB > B) {
        flag_error(err, ERR_RANGE);
      } else {
        m.fb = full_base[mi];
        m.nfull = cd.div(B);
        m.rr = rem_rail[mi];
        m.ro = rem_off[mi];
        const long long c0 = cd.div(m.p0);
        m.dst0 = chunk_addr(c0, m.fb, m.nfull, m.rr, m.ro, N, C, rbase) + (m.p0 - c0 * C);
        const long long b0 = (c0 + 1) * C - m.p0;
        m.b0 = (int)(b0 < RB ? b0 : RB);
        if (!MULTI && m.b0 < RB)
          m.dst1 = chunk_addr(c0 + 1, m.fb, m.nfull, m.rr, m.ro, N, C, rbase);
        m.ok = 1;
      }
    }
    meta[wid][st][lane] = m;
  };

  // prologue: loads of rows 0..D-1 of this warp
  for (int j = 0; j < D; ++j) {
    const long long row = row0 + (long long)j * nwarps;
    if (row >= rows) break;
    make_meta(row, j);
    if (lane == 0) {
      mbar_expect_tx(&bar[j], (uint32_t)RB);
      bulk_load(buf + (size_t)j * RB, x + row * RB, (uint32_t)RB, &bar[j]);
    }
  }
  long long j = 0;
  for (long long row = row0; row < rows; row += nwarps, ++j) {
    // issue row j + D
    const long long rn = row + (long long)D * nwarps;
    const int stn = (int)((j + D) % S);
    if (rn < rows) {
      make_meta(rn, stn);
      if (lane == 0) {
        bulk_wait_read<S - D - 1>();  // stage stn's previous stores have read it
        mbar_expect_tx(&bar[stn], (uint32_t)RB);
        bulk_load(buf + (size_t)stn * RB, x + rn * RB, (uint32_t)RB, &bar[stn]);
      }
    }
    __syncwarp();
    const int st = (int)(j % S);
    if (lane == 0) {
      mbar_wait(&bar[st], (uint32_t)((j / S) & 1));
      const uint8_t* src = buf + (size_t)st * RB;
      const long long ul = (row / T) / N;
      const int64_t* __restrict__ rbase = rail_base + ul * N;
      for (int s = 0; s < k; ++s) {
        const TmaMeta& m = meta[wid][st][s];
        if (!m.ok) continue;
        long long a = m.dst0;
        long long len = m.b0;
        if (a >= 0 && a + len <= out_cap)
          bulk_store(out + a, src, (uint32_t)len);
        else
          flag_error(err, ERR_NOSPC);
        long long p = m.b0;
        while (p < RB) {
          long long c, base;
          if (!MULTI) {
            base = m.dst1;
            len = RB - p;
          } else {
            const long long q = m.p0 + p;
            c = cd.div(q);
            base = chunk_addr(c, m.fb, m.nfull, m.rr, m.ro, N, C, rbase) + (q - c * C);
            len = min(C - (q - c * C), RB - p);
          }
          if (base >= 0 && base + len <= out_cap)
            bulk_store(out + base, src + p, (uint32_t)len);
          else
            flag_error(err, ERR_NOSPC);
          p += len;
        }
      }
      bulk_commit();
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait_all();
}

// ---------------------------------------------------------------- TMA pipeline v2
// C >= RB only (a row copy spans at most two chunks).  As k_pack_tma, but the
// slot metadata -- a chain of dependent loads (routing -> LUT -> message tables
// -> rail base) -- is computed for 32 rows at once, one row per lane, into a
// per-warp shared table, so its latency is paid once per 32 rows instead of once
// per row on the issuing path.  W warps per CTA, S row stages per warp, loads D
// rows ahead.
constexpr int TMA2_MAXK = 4;
struct TmaMeta2 {
  long long dst0, dst1;  // output address of row byte 0 / of chunk c0+1
  int b0, ok;            // row bytes in chunk c0; remote and valid
};

template <int S, int D, int W>
__global__ void __launch_bounds__(W * 32)
    k_pack_tma2(int U, int nd, int d0, int M, int N, int T, int k, long long C, int cshift,
                const uint8_t* __restrict__ x, const int32_t* __restrict__ topk,
                const int32_t* __restrict__ lut, int n_inst, const int32_t* __restrict__ rank,
                const int64_t* __restrict__ msg, long long RB,
                const int64_t* __restrict__ full_base, const int8_t* __restrict__ rem_rail,
                const int64_t* __restrict__ rem_off, const int64_t* __restrict__ rail_base,
                uint8_t* __restrict__ out, long long out_cap, int* err) {
  static_assert(D >= 1 && D < S, "prefetch distance");
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ __align__(8) uint64_t bars[W][S];
  __shared__ TmaMeta2 meta[W][32][TMA2_MAXK];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long nwarps = (long long)gridDim.x * W;
  const long long rows = (long long)U * nd * N * T;
  const long long G = (long long)M * N;
  const ChunkDiv cd{C, cshift};
  uint8_t* buf = sbuf + (size_t)wid * S * RB;
  uint64_t* bar = bars[wid];
  const long long row0 = (long long)blockIdx.x * W + wid;
  if (lane == 0) {
    for (int q = 0; q < S; ++q) mbar_init(&bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // metadata of this warp's rows j0 .. j0+31 (lane l: row j0 + l)
  auto make_meta32 = [&](long long j0) {
    const long long row = row0 + (j0 + lane) * nwarps;
    for (int sl = 0; sl < k; ++sl) {
      TmaMeta2 m{0, 0, 0, 0};
      if (row < rows) {
        const long long ug = row / T;
        const long long ul = ug / N;
        const int d = d0 + (int)(ul % nd);
        const int64_t* __restrict__ rbase = rail_base + ul * N;
        const long long e = row * k + sl;
        const int inst = __ldg(topk + e);
        int h = (inst >= 0 && inst < n_inst) ? __ldg(lut + inst) : -1;
        if (h < 0 || h >= G) {
          flag_error(err, ERR_RANGE);
          h = -1;
        }
        if (h >= 0 && h / N != d) {
          const long long mi = ug * G + h;
          const long long B = msg[mi];
          const int rk = rank[e];
          const long long p0 = (long long)rk * RB;
          if (rk < 0 || p0 + RB > B) {
            flag_error(err, ERR_RANGE);
          } else {
            const long long fb = full_base[mi], nfull = cd.div(B);
            const int rr = rem_rail[mi];
            const long long ro = rem_off[mi];
            const long long c0 = cd.div(p0);
            m.dst0 = chunk_addr(c0, fb, nfull, rr, ro, N, C, rbase) + (p0 - c0 * C);
            const long long b0 = (c0 + 1) * C - p0;
            m.b0 = (int)(b0 < RB ? b0 : RB);
            if (m.b0 < RB) m.dst1 = chunk_addr(c0 + 1, fb, nfull, rr, ro, N, C, rbase);
            m.ok = 1;
          }
        }
      }
      meta[wid][lane][sl] = m;
    }
  };
  // prologue: loads of rows 0..D-1 of this warp
  if (lane == 0) {
    for (int j = 0; j < D; ++j) {
      const long long row = row0 + (long long)j * nwarps;
      if (row >= rows) break;
      mbar_expect_tx(&bar[j], (uint32_t)RB);
      bulk_load(buf + (size_t)j * RB, x + row * RB, (uint32_t)RB, &bar[j]);
    }
  }
  long long j = 0;
  for (long long row = row0; row < rows; row += nwarps, ++j) {
    if ((j & 31) == 0) {
      __syncwarp();
      make_meta32(j);
      __syncwarp();
    }
    if (lane == 0) {
      const long long rn = row + (long long)D * nwarps;
      const int stn = (int)((j + D) % S);
      if (rn < rows) {
        bulk_wait_read<S - D - 1>();  // stage stn's previous stores have read it
        mbar_expect_tx(&bar[stn], (uint32_t)RB);
        bulk_load(buf + (size_t)stn * RB, x + rn * RB, (uint32_t)RB, &bar[stn]);
      }
      const int st = (int)(j % S);
      mbar_wait(&bar[st], (uint32_t)((j / S) & 1));
      const uint8_t* src = buf + (size_t)st * RB;
      for (int sl = 0; sl < k; ++sl) {
        const TmaMeta2 m = meta[wid][j & 31][sl];
        if (!m.ok) continue;
        if (m.dst0 >= 0 && m.dst0 + m.b0 <= out_cap)
          bulk_store(out + m.dst0, src, (uint32_t)m.b0);
        else
          flag_error(err, ERR_NOSPC);
        if (m.b0 < RB) {
          if (m.dst1 >= 0 && m.dst1 + (RB - m.b0) <= out_cap)
            bulk_store(out + m.dst1, src + m.b0, (uint32_t)(RB - m.b0));
          else
            flag_error(err, ERR_NOSPC);
        }
      }
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
}

template <int S, int D, int W>
static cudaError_t launch_tma2(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T,
                               int k, long long C, int cshift, const void* x,
                               const int32_t* topk, const int32_t* lut, int n_inst,
                               const int32_t* rank, const int64_t* msg, long long RB,
                               const rails_sched_t& s, const int64_t* rail_base, void* out,
                               long long out_cap) {
  auto kern = k_pack_tma2<S, D, W>;
  const size_t smem = (size_t)W * S * RB;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  if (const char* pv = getenv("RAILS_PACK_CTAS")) {  // CTAs per SM (more than resident: waves)
    const int v = atoi(pv);
    if (v >= 1) per_sm = v;
  }
  const long long rows = (long long)U * nd * N * T;
  long long grid = (long long)c.num_sms * per_sm;
  const long long need = (rows + W - 1) / W;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, W * 32, smem, c.stream>>>(
      U, nd, d0, M, N, T, k, C, cshift, (const uint8_t*)x, topk, lut, n_inst, rank, msg, RB,
      s.full_base, s.rem_rail, s.rem_off, rail_base, (uint8_t*)out, out_cap, c.err);
  count_launch(1);
  return cudaGetLastError();
}

template <int S, int D, bool MULTI>
static cudaError_t launch_tma_sd(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T,
                                 int k, long long C, int cshift, const void* x,
                                 const int32_t* topk, const int32_t* lut, int n_inst,
                                 const int32_t* rank, const int64_t* msg, long long RB,
                                 const rails_sched_t& s, const int64_t* rail_base, void* out,
                                 long long out_cap) {
  auto kern = k_pack_tma<S, D, MULTI>;
  const size_t smem = (size_t)TMA_WARPS * S * RB;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TMA_WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  if (const char* pv = getenv("RAILS_PACK_CTAS")) {  // CTAs per SM (more than resident: waves)
    const int v = atoi(pv);
    if (v >= 1) per_sm = v;
  }
  const long long rows = (long long)U * nd * N * T;
  long long grid = (long long)c.num_sms * per_sm;
  const long long need = (rows + TMA_WARPS - 1) / TMA_WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, TMA_WARPS * 32, smem, c.stream>>>(
      U, nd, d0, M, N, T, k, C, cshift, (const uint8_t*)x, topk, lut, n_inst, rank, msg, RB,
      s.full_base, s.rem_rail, s.rem_off, rail_base, (uint8_t*)out, out_cap, c.err);
  count_launch(1);
  return cudaGetLastError();
}

template <bool MULTI>
static cudaError_t launch_tma(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T,
                              int k, long long C, int cshift, const void* x, const int32_t* topk,
                              const int32_t* lut, int n_inst, const int32_t* rank,
                              const int64_t* msg, long long RB, const rails_sched_t& s,
                              const int64_t* rail_base, void* out, long long out_cap) {
  // stages per warp from a ~200 KiB shared-memory budget (4 warps per CTA)
  const long long budget = 200 * 1024;
  const long long S = budget / (TMA_WARPS * RB);
  if (S >= 8)
    return launch_tma_sd<8, 4, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst,
                                      rank, msg, RB, s, rail_base, out, out_cap);
  if (S >= 6)
    return launch_tma_sd<6, 3, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst,
                                      rank, msg, RB, s, rail_base, out, out_cap);
  if (S >= 4)
    return launch_tma_sd<4, 2, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst,
                                      rank, msg, RB, s, rail_base, out, out_cap);
  if (S >= 3)
    return launch_tma_sd<3, 1, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst,
                                      rank, msg, RB, s, rail_base, out, out_cap);
  return launch_tma_sd<2, 1, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst,
                                    rank, msg, RB, s, rail_base, out, out_cap);
}

cudaError_t launch_pack(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T, int k,
                        long long C, const void* x, const int32_t* topk, const int32_t* lut,
                        int n_inst, const int32_t* rank, const int64_t* msg, long long row_bytes,
                        const rails_sched_t& s, const int64_t* rail_base, void* out,
                        long long out_cap, int impl) {
  int cshift = -1;
  if ((C & (C - 1)) == 0) {
    cshift = 0;
    while ((1LL << cshift) < C) ++cshift;
  }
  // impl 3: TMA pipeline v2 (batched metadata), RAILS_PACK_TMA = "S,D,W" selects
  // the stage / distance / warps shape among the compiled ones
  if (impl == 3 && k <= TMA2_MAXK && C >= row_bytes && row_bytes <= 8 * 1024) {
    const char* sh = getenv("RAILS_PACK_TMA");
    const int v = sh ? atoi(sh) : 0;
#define RAILS_TMA2(SS, DD, WW)                                                               \
  if (v == SS * 100 + DD * 10 + WW || (v == 0 && SS == 4 && DD == 3 && WW == 6))            \
    return launch_tma2<SS, DD, WW>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, \
                                   rank, msg, row_bytes, s, rail_base, out, out_cap);
    if (row_bytes * 4 * 6 <= 200 * 1024) {
      RAILS_TMA2(4, 3, 6)
      RAILS_TMA2(3, 2, 8)
      RAILS_TMA2(6, 4, 4)
      RAILS_TMA2(4, 2, 6)
      RAILS_TMA2(2, 1, 8)
    }
#undef RAILS_TMA2
    return launch_tma2<2, 1, 4>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank,
                                msg, row_bytes, s, rail_base, out, out_cap);
  }
  // impl 2: TMA bulk-copy pipeline (rows up to 48 KiB, k <= 8); 1: LDG/STG registers
  if (impl == 2 && k <= TMA_MAXK && row_bytes <= 48 * 1024) {
    if (C >= row_bytes)
      return launch_tma<false>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank,
                               msg, row_bytes, s, rail_base, out, out_cap);
    return launch_tma<true>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank, msg,
                            row_bytes, s, rail_base, out, out_cap);
  }
  if (C >= row_bytes)
    return launch_m<false>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank, msg,
                           row_bytes, s, rail_base, out, out_cap);
  return launch_m<true>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank, msg,
                        row_bytes, s, rail_base, out, out_cap);
}

}  // namespace rails
