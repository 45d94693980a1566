// eval.cuh -- a5 helpers shared by the standalone evaluation (k_eval.cu) and the
// fused per-node kernel (k_node.cu): exact 128-bit -> double, split 64-bit shared
// accumulation, the per-unit finalize (T, T*, busbw; Thm 2 + Thm 3,
// R#8, R#10, R#40) and the rail-offset scan.
//
// Reduction record of one unit (RAILS_RED_SUM_LEN / RAILS_RED_MAX_LEN, rails.h):
//   red_sum: R[M][N], R_e[M][N], R_u[M][N], colsum[M], total, total_e
//   red_max: max S, max S_e, max row sum, max S_u
#pragma once

#include "common.cuh"

namespace rails {

struct RedLayout {
  long long MN, M;
  __host__ __device__ long long R() const { return 0; }
  __host__ __device__ long long Re() const { return MN; }
  __host__ __device__ long long Ru() const { return 2 * MN; }
  __host__ __device__ long long col() const { return 3 * MN; }
  __host__ __device__ long long tot() const { return 3 * MN + M; }
  __host__ __device__ long long len() const { return 3 * MN + M + 2; }
};
enum { RMAX_S = 0, RMAX_SE = 1, RMAX_ROW = 2, RMAX_SU = 3 };

__device__ __forceinline__ double u128_to_double(unsigned __int128 v) {
  const unsigned long long hi = (unsigned long long)(v >> 64), lo = (unsigned long long)v;
  if (hi == 0) return __ull2double_rn(lo);
  return __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
}

// MSE of one node's loads (Eq. 6; R#11): sum_j (N*L_j - sum L)^2 / N^3 exactly;
// nMSE = MSE / (sum L)^2, 0 when sum L = 0 (R#12).  Called by one full warp, lane j
// holding L_j (lanes >= N: any value).
__device__ __forceinline__ void warp_mse(long long s, int N, long long total, double* mse,
                                         double* nmse) {
  unsigned __int128 sq = 0;
  for (int j = 0; j < N; ++j) {
    const long long sj = __shfl_sync(FULL, s, j);
    const __int128 dv = (__int128)N * sj - (__int128)total;
    sq += (unsigned __int128)(dv * dv);
  }
  const double dN = (double)N;
  const double m = __ddiv_rn(u128_to_double(sq), __dmul_rn(__dmul_rn(dN, dN), dN));
  *mse = m;
  *nmse = total == 0 ? 0.0 : __ddiv_rn(m, __dmul_rn(__ll2double_rn(total), __ll2double_rn(total)));
}

__device__ __forceinline__ void divmod_n(long long a, int N, long long& q, int& r) {
  if (a >= 0 && a < (1LL << 32)) {
    const unsigned ua = (unsigned)a;
    const unsigned uq = ua / (unsigned)N;
    q = uq;
    r = (int)(ua - uq * (unsigned)N);
  } else {
    q = a / N;
    r = (int)(a - q * N);
  }
}

// 64-bit accumulation as two 32-bit shared atomics (the carry out of the low half
// goes to the high half); exact and order-independent.
__device__ __forceinline__ void add64_split(unsigned* lo, unsigned* hi, unsigned long long v) {
  const unsigned l = (unsigned)v, h = (unsigned)(v >> 32);
  const unsigned old = atomicAdd(lo, l);
  const unsigned carry = (old + l < old) ? 1u : 0u;
  if (h + carry) atomicAdd(hi, h + carry);
}

// 64-bit sums as two independent 32-bit shared reductions (no returned value, so the
// adds are fire-and-forget): low 20 bits and the rest.  Exact while a bin receives at
// most 4096 addends (low word < 2^32) and their sum stays below 2^52; the fused
// kernel's bins get at most N^2 <= 1024 messages of < 2^40 bytes each.
__device__ __forceinline__ void add_split20(unsigned* lo, unsigned* hi, unsigned long long v) {
  atomicAdd(lo, (unsigned)(v & 0xFFFFFull));
  if (v >> 20) atomicAdd(hi, (unsigned)(v >> 20));
}
__device__ __forceinline__ unsigned long long get_split20(unsigned lo, unsigned hi) {
  return ((unsigned long long)hi << 20) + lo;
}

// T, T*, busbw of unit u from the reduced maxima and totals (R#8, R#10, Thm 2/3;
// uniform policy R#41; busbw 0 without traffic, R#40).
__device__ __forceinline__ void finalize_unit(long long u, int N, double R2, long long mR,
                                              long long mRe, long long mRu, long long mc,
                                              const long long (&rm)[RAILS_RED_MAX_LEN],
                                              long long total, long long total_e,
                                              const rails_final_t& out) {
  const long long maxload = max(rm[RMAX_S], mR);
  const long long maxload_e = max(rm[RMAX_SE], mRe);
  const long long maxload_u = max(rm[RMAX_SU], mRu);
  const long long rowmax = rm[RMAX_ROW];
  const double T = __ddiv_rn(__ll2double_rn(maxload), R2);
  const double T_e = __ddiv_rn(__ll2double_rn(maxload_e), R2);
  const double T_u = __ddiv_rn(__ll2double_rn(maxload_u), R2);
  const long long lb = max(rowmax, mc);
  const double T_star = __ddiv_rn(__ll2double_rn(lb), __dmul_rn((double)N, R2));
  if (out.maxload) out.maxload[u] = maxload;
  if (out.maxload_e) out.maxload_e[u] = maxload_e;
  if (out.maxload_u) out.maxload_u[u] = maxload_u;
  if (out.total) out.total[u] = total;
  if (out.rowmax) out.rowmax[u] = rowmax;
  if (out.colmax) out.colmax[u] = mc;
  if (out.T) out.T[u] = T;
  if (out.T_e) out.T_e[u] = T_e;
  if (out.T_u) out.T_u[u] = T_u;
  if (out.T_star) out.T_star[u] = T_star;
  if (out.busbw) out.busbw[u] = total > 0 ? __ddiv_rn(__ll2double_rn(total), T) : 0.0;
  if (out.busbw_e) out.busbw_e[u] = total_e > 0 ? __ddiv_rn(__ll2double_rn(total_e), T_e) : 0.0;
  if (out.busbw_u) out.busbw_u[u] = total > 0 ? __ddiv_rn(__ll2double_rn(total), T_u) : 0.0;
}

// One CTA finalizes unit u from its fully reduced record (rs: red_sum of the unit,
// rm: red_max of the unit).  LOADCG: read through L2 only (the record was written by
// other CTAs of the same kernel).
template <bool LOADCG>
__device__ void block_finalize_unit(long long u, int M, int N, double R2, const int64_t* rs,
                                    const int64_t* rm, const rails_final_t& out) {
  __shared__ long long s4[4][32];
  const RedLayout L{(long long)M * N, M};
  auto ld = [](const int64_t* p) -> long long {
    return LOADCG ? (long long)__ldcg((const long long*)p) : (long long)*p;
  };
  long long mR = 0, mRe = 0, mRu = 0, mc = 0;
  for (long long i = threadIdx.x; i < L.MN; i += blockDim.x) {
    mR = max(mR, ld(rs + L.R() + i));
    mRe = max(mRe, ld(rs + L.Re() + i));
    mRu = max(mRu, ld(rs + L.Ru() + i));
  }
  for (long long i = threadIdx.x; i < M; i += blockDim.x) mc = max(mc, ld(rs + L.col() + i));
  mR = warp_max(mR);
  mRe = warp_max(mRe);
  mRu = warp_max(mRu);
  mc = warp_max(mc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s4[0][wid] = mR;
    s4[1][wid] = mRe;
    s4[2][wid] = mRu;
    s4[3][wid] = mc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mR = max(mR, s4[0][w]);
      mRe = max(mRe, s4[1][w]);
      mRu = max(mRu, s4[2][w]);
      mc = max(mc, s4[3][w]);
    }
    long long rmv[RAILS_RED_MAX_LEN];
#pragma unroll
    for (int i = 0; i < RAILS_RED_MAX_LEN; ++i) rmv[i] = ld(rm + i);
    finalize_unit(u, N, R2, mR, mRe, mRu, mc, rmv, ld(rs + L.tot()), ld(rs + L.tot() + 1), out);
  }
  __syncthreads();
}

// Exclusive prefix of send_load in (u, dl, j) order -> rail_base; total bytes
// (one CTA).
template <bool LOADCG>
__device__ void block_rail_offsets(long long n, const int64_t* send_load, int64_t* rail_base,
                                   int64_t* total) {
  __shared__ long long scratch[33];
  long long carry = 0;
  for (long long t0 = 0; t0 < n; t0 += blockDim.x) {
    const long long i = t0 + threadIdx.x;
    long long v = 0;
    if (i < n) v = LOADCG ? (long long)__ldcg((const long long*)send_load + i) : send_load[i];
    long long tot;
    const long long ex = block_excl_scan(v, scratch, &tot);
    if (i < n) rail_base[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

}  // namespace rails
