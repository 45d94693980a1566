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

template <int VPL, bool MULTI>
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
      if (vi < nvec) v[i] = ld_stream(src + vi);
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
          if (vi < nvec) v[i] = ld_stream(src + vi);
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
  auto kern = k_pack<VPL, MULTI>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PACK_THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long rows = (long long)U * nd * N * T;
  const long long need = (rows + PACK_THREADS / 32 - 1) / (PACK_THREADS / 32);
  // waves of CTAs, ~8 rows per warp (wave_grid)
  const long long grid = wave_grid(c.num_sms, per_sm, need, 8);
  kern<<<(unsigned)grid, PACK_THREADS, 0, c.stream>>>(
      U, nd, d0, M, N, T, k, C, cshift, (const uint4*)x, topk, lut, n_inst, rank, msg, RB,
      s.full_base, s.rem_rail, s.rem_off, rail_base, (uint8_t*)out, out_cap, c.err);
  count_launch(1);
  return cudaGetLastError();
}

// Vectors per lane: rows up to 2 KiB hold the whole row in 4 x 16 B per lane; longer
// rows are copied in 8 KiB windows of 16 vectors per lane (C4's 12 KiB rows: 90% of
// the copy peak vs 87% with the whole row in 24 registers-worth of vectors).
template <bool MULTI>
static cudaError_t launch_m(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T, int k,
                            long long C, int cshift, const void* x, const int32_t* topk,
                            const int32_t* lut, int n_inst, const int32_t* rank,
                            const int64_t* msg, long long RB, const rails_sched_t& s,
                            const int64_t* rail_base, void* out, long long out_cap) {
  if ((RB >> 4) <= 4 * 32)
    return launch_v<4, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank,
                              msg, RB, s, rail_base, out, out_cap);
  return launch_v<16, MULTI>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank,
                             msg, RB, s, rail_base, out, out_cap);
}

cudaError_t launch_pack(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T, int k,
                        long long C, const void* x, const int32_t* topk, const int32_t* lut,
                        int n_inst, const int32_t* rank, const int64_t* msg, long long row_bytes,
                        const rails_sched_t& s, const int64_t* rail_base, void* out,
                        long long out_cap) {
  int cshift = -1;
  if ((C & (C - 1)) == 0) {
    cshift = 0;
    while ((1LL << cshift) < C) ++cshift;
  }
  if (C >= row_bytes)
    return launch_m<false>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank, msg,
                           row_bytes, s, rail_base, out, out_cap);
  return launch_m<true>(c, U, nd, d0, M, N, T, k, C, cshift, x, topk, lut, n_inst, rank, msg,
                        row_bytes, s, rail_base, out, out_cap);
}

}  // namespace rails
