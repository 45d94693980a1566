// k_eval.cu -- a5: loads, completion time, T*, busbw, MSE, ECMP baseline (sm_100a).
//
// Load model (Eq. 4-5; rail pairing NIC(k,n) -> NIC(f,n), R#7):
// a chunk of node d on rail j bound for node f adds to S[d][j] and R[f][j].
// From the compact schedule, message (g,h) with n = floor(B/C) full chunks
// starting at node-global full index fb puts q*C on every rail plus C on the r
// rails fb mod N, fb+1 mod N, ... (q = n div N, r = n mod N), and its remainder on
// rem_rail.  So eval is O(messages * N), never O(chunks).
//
// k_eval_node2 (default): one CTA per (unit, node), destination nodes in tiles of
// 256/N; stage 1 stages each message's bytes, remainder, remainder rail and ECMP
// rail in shared memory (loads batched per thread), stage 2 runs one thread per
// (f, j) over the tile's N*N messages into f and adds the full chunks by the
// closed form above.  Then R[f][j] += R_d[f][j] (int64 atomics: order-independent,
// hence deterministic), S[d][j] = sum_f R_d[f][j] (register partials per rail),
// colsum[f] += sum_j R_d[f][j].  (k_eval_node, the first version, is kept behind
// RAILS_EVAL_IMPL=1.)  The ECMP
// baseline (R#13-R#14) hashes each whole message onto one rail.
// MSE (Eq. 6; Alg. 2 step 6; R#11) is the exact integer
// sum_j (N*S_j - sum S)^2 over N^3, converted once (R#25).
// k_eval_finalize: per unit, max over the reduced R, T = maxload/R2,
// T* = max(rowmax, colmax)/(N*R2) (Thm 2 + Thm 3), busbw = total/T (R#10).
#include <cstdlib>

#include "common.cuh"

namespace rails {

constexpr int EVAL_WARPS = 8;

__device__ __forceinline__ double u128_to_double(unsigned __int128 v) {
  const unsigned long long hi = (unsigned long long)(v >> 64), lo = (unsigned long long)v;
  if (hi == 0) return __ull2double_rn(lo);
  return __dadd_rn(__dmul_rn(__ull2double_rn(hi), 18446744073709551616.0), __ull2double_rn(lo));
}

__global__ void __launch_bounds__(EVAL_WARPS * 32)
    k_eval_node(int M, int N, int nd, int d0, long long C, int cshift, uint64_t seed,
                const int64_t* __restrict__ msg, const int64_t* __restrict__ full_base,
                const int8_t* __restrict__ rem_rail, int64_t* __restrict__ S,
                int64_t* __restrict__ S_e, double* __restrict__ mse,
                double* __restrict__ nmse, int64_t* __restrict__ red_sum,
                int64_t* __restrict__ red_max, long long rsl) {
  __shared__ long long sS[EVAL_WARPS][32], sSe[EVAL_WARPS][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long seg = blockIdx.x;
  const long long u = seg / nd;
  const int d = d0 + (int)(seg % nd);
  const long long G = (long long)M * N, NG = (long long)N * G;
  const ChunkDiv cd{C, cshift};
  const int64_t* __restrict__ mg = msg + seg * NG;
  const int64_t* __restrict__ fbp = full_base + seg * NG;
  const int8_t* __restrict__ rrp = rem_rail + seg * NG;
  unsigned long long* rs = (unsigned long long*)(red_sum + u * rsl);
  unsigned long long* R = rs;
  unsigned long long* Re = rs + M * (long long)N;
  unsigned long long* col = Re + M * (long long)N;
  unsigned long long* tot = col + M;

  long long Sj = 0, Sej = 0;
  const int NN = N * N;
  for (int f = wid; f < M; f += EVAL_WARPS) {
    if (f == d) continue;  // intra-node traffic never crosses the rails (R#2)
    long long Rf = 0, Ref = 0;
    for (int b0 = 0; b0 < NN; b0 += 32) {
      const int l = b0 + lane;
      long long B = 0, q = 0, rem = 0;
      int r = 0, st = 0, rr = -1, e = -1;
      if (l < NN) {
        const int g = l / N, m = l - (l / N) * N;
        const long long idx = (long long)g * G + (long long)f * N + m;
        B = mg[idx];
        if (B > 0) {
          const long long nf = cd.div(B);
          rem = B - nf * C;
          const long long fb = fbp[idx];
          q = nf / N;
          r = (int)(nf - q * N);
          st = (int)(fb % N);
          rr = (rem > 0) ? (int)rrp[idx] : -1;
          e = ecmp_rail(seed, (long long)d * N + g, (long long)f * N + m, N);
        } else {
          B = 0;
        }
      }
      const int cnt = min(32, NN - b0);
      for (int b = 0; b < cnt; ++b) {
        const long long Bb = __shfl_sync(FULL, B, b);
        if (Bb == 0) continue;
        const long long qb = __shfl_sync(FULL, q, b);
        const long long remb = __shfl_sync(FULL, rem, b);
        const int rb = __shfl_sync(FULL, r, b);
        const int stb = __shfl_sync(FULL, st, b);
        const int rrb = __shfl_sync(FULL, rr, b);
        const int eb = __shfl_sync(FULL, e, b);
        if (lane < N) {
          int dj = lane - stb;
          if (dj < 0) dj += N;
          Rf += qb * C + (dj < rb ? C : 0) + (lane == rrb ? remb : 0);
          if (lane == eb) Ref += Bb;
        }
      }
    }
    if (lane < N) {
      if (Rf) atomicAdd(R + (long long)f * N + lane, (unsigned long long)Rf);
      if (Ref) atomicAdd(Re + (long long)f * N + lane, (unsigned long long)Ref);
      Sj += Rf;
      Sej += Ref;
    }
    const long long cf = warp_sum(lane < N ? Rf : 0LL);
    if (lane == 0 && cf) atomicAdd(col + f, (unsigned long long)cf);
  }
  sS[wid][lane] = Sj;
  sSe[wid][lane] = Sej;
  __syncthreads();
  if (wid != 0) return;
  long long s = 0, se = 0;
#pragma unroll
  for (int w = 0; w < EVAL_WARPS; ++w) {
    s += sS[w][lane];
    se += sSe[w][lane];
  }
  if (lane >= N) s = se = 0;
  if (lane < N) {
    S[seg * N + lane] = s;
    S_e[seg * N + lane] = se;
  }
  const long long total = warp_sum(s), total_e = warp_sum(se);
  const long long mx = warp_max(s), mxe = warp_max(se);
  unsigned __int128 sq = 0;
  for (int j = 0; j < N; ++j) {
    const long long sj = __shfl_sync(FULL, s, j);
    const __int128 dv = (__int128)N * sj - (__int128)total;
    sq += (unsigned __int128)(dv * dv);
  }
  if (lane == 0) {
    const double dN = (double)N;
    const double m = __ddiv_rn(u128_to_double(sq), __dmul_rn(__dmul_rn(dN, dN), dN));
    mse[seg] = m;
    nmse[seg] =
        total == 0 ? 0.0
                   : __ddiv_rn(m, __dmul_rn(__ll2double_rn(total), __ll2double_rn(total)));
    if (total) atomicAdd(tot, (unsigned long long)total);
    if (total_e) atomicAdd(tot + 1, (unsigned long long)total_e);
    atomicMax((long long*)red_max + u * RAILS_RED_MAX_LEN + 0, mx);
    atomicMax((long long*)red_max + u * RAILS_RED_MAX_LEN + 1, mxe);
    atomicMax((long long*)red_max + u * RAILS_RED_MAX_LEN + 2, total);
  }
}


// ---------------------------------------------------------------- tiled eval (v2)
// Same outputs as k_eval_node.  The node's messages are processed in tiles of FT
// destination nodes.  Stage 1 (thread per message): B, remainder, its rail and the
// ECMP rail go to shared memory, plus, per (g, f), the node-global full-chunk
// index where the block of messages (g, f*N .. f*N+N-1) starts, as (q, r) = divmod
// by N.  Messages of fixed g and f are contiguous in (g,h) order, so their full
// chunks form ONE index range [a, b); rail j receives cnt(b) - cnt(a) of them with
// cnt(x) = floor(x/N) + (j < x mod N).  Stage 2 (thread per (f, j)): R_d[f][j] =
// C * sum_g (cnt(b) - cnt(a)) + sum of remainders on j, R_e likewise from the ECMP
// rails; then R[f][j] += R_d[f][j] (one global atomic), S_j, S_e_j and colsum[f]
// accumulate in shared memory.
constexpr int EV2_THREADS = 256;

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

template <int NT>  // NT = N when it is a power of two <= 32 (divisions by shifts), else 0
__global__ void __launch_bounds__(EV2_THREADS)
    k_eval_node2(int M, int N_rt, int nd, int d0, long long C, int cshift, uint64_t seed, int FT,
                 const int64_t* __restrict__ msg, const int64_t* __restrict__ full_base,
                 const int8_t* __restrict__ rem_rail, const int64_t* __restrict__ n_full,
                 int64_t* __restrict__ S, int64_t* __restrict__ S_e, double* __restrict__ mse,
                 double* __restrict__ nmse, int64_t* __restrict__ red_sum,
                 int64_t* __restrict__ red_max, long long rsl) {
  extern __shared__ __align__(16) uint8_t ev_smem[];
  __shared__ unsigned long long sS[32], sSe[32];
  const int N = NT ? NT : N_rt;
  const long long seg = blockIdx.x;
  const long long u = seg / nd;
  const int d = d0 + (int)(seg % nd);
  const long long G = (long long)M * N, NG = (long long)N * G;
  const ChunkDiv cd{C, cshift};
  const int64_t* __restrict__ mg = msg + seg * NG;
  const int64_t* __restrict__ fbp = full_base + seg * NG;
  const int8_t* __restrict__ rrp = rem_rail + seg * NG;
  const long long nfull_node = n_full[seg];
  unsigned long long* rs = (unsigned long long*)(red_sum + u * rsl);
  unsigned long long* R = rs;
  unsigned long long* Re = rs + M * (long long)N;
  unsigned long long* col = Re + M * (long long)N;
  unsigned long long* tot = col + M;

  long long* sQ = (long long*)ev_smem;                 // [N][FT+1]
  int* sR = (int*)(sQ + N * (FT + 1));                 // [N][FT+1]
  __shared__ unsigned long long sCol[64];
  // per (fl, j) of the tile: remainder bytes into NIC (f, j) and ECMP bytes, as
  // 64-bit sums split into 32-bit halves (32-bit shared atomics are native)
  __shared__ unsigned aRlo[EV2_THREADS], aRhi[EV2_THREADS], aElo[EV2_THREADS],
      aEhi[EV2_THREADS];

  if (threadIdx.x < 32) {
    sS[threadIdx.x] = 0;
    sSe[threadIdx.x] = 0;
  }
  const bool pow2 = NT != 0;
  unsigned long long accS = 0, accSe = 0;
  __shared__ unsigned long long sAcc[2][EV2_THREADS];
  for (int f0 = 0; f0 < M; f0 += FT) {
    const int ft = min(FT, M - f0);
    __syncthreads();
    if (threadIdx.x < 64) sCol[threadIdx.x] = 0;
    aRlo[threadIdx.x] = aRhi[threadIdx.x] = aElo[threadIdx.x] = aEhi[threadIdx.x] = 0u;
    __syncthreads();
    // stage 1: per-message fields, t = g * (ft*N) + rest with h = f0*N + rest; a
    // thread takes one `rest` for every g, all N loads in flight before any use
    // (small tiles: threads beyond the tile's width split the g range)
    const int tn = ft * N;
    const int gsp = tn >= EV2_THREADS ? 1 : EV2_THREADS / tn;
    for (int r0 = 0; r0 < tn; r0 += EV2_THREADS) {
      const int rest = r0 + (gsp > 1 ? threadIdx.x % tn : threadIdx.x);
      const int gq = gsp > 1 ? threadIdx.x / tn : 0;
      if (rest >= tn || gq >= gsp) continue;
      const long long h = (long long)f0 * N + rest;
      constexpr int GB = NT ? (NT < 4 ? NT : 4) : 1;  // loads in flight per batch
      for (int g0 = gq; g0 < N; g0 += GB * gsp) {
        long long Bv[GB];
        int8_t Rv[GB];
#pragma unroll
        for (int q = 0; q < GB; ++q) {
          const int g = g0 + q * gsp;
          Bv[q] = 0;
          Rv[q] = -1;
          if (g < N) {
            const long long idx = (long long)g * G + h;
            Bv[q] = mg[idx];
            Rv[q] = rrp[idx];
          }
        }
#pragma unroll
        for (int q = 0; q < GB; ++q) {
          const int g = g0 + q * gsp;
          if (g >= N) break;
          const long long B = Bv[q];
          if (B > 0 && (int)(h / N) != d) {
            const int fb = (rest / N) * N;  // (fl, 0) of this message's destination
            const long long nf = cd.div(B);
            const long long rem = B - nf * C;
            if (rem && Rv[q] >= 0 && Rv[q] < N)
              add64_split(&aRlo[fb + Rv[q]], &aRhi[fb + Rv[q]], (unsigned long long)rem);
            const int e = ecmp_rail(seed, (long long)d * N + g, h, N);
            add64_split(&aElo[fb + e], &aEhi[fb + e], (unsigned long long)B);
          }
        }
      }
    }
    // block boundaries: full index at message (g, (f0+fl)*N), fl = 0..ft
    for (int t = threadIdx.x; t < N * (ft + 1); t += EV2_THREADS) {
      const int g = t / (ft + 1), fl = t - g * (ft + 1);
      const long long p = (long long)g * G + (long long)(f0 + fl) * N;
      const long long a = (p < NG) ? fbp[p] : nfull_node;
      long long q;
      int r;
      divmod_n(a, N, q, r);
      sQ[g * (FT + 1) + fl] = q;
      sR[g * (FT + 1) + fl] = r;
    }
    __syncthreads();
    // stage 2: thread per (fl, j).  N a power of two: j = t mod N is the same for a
    // thread in every tile, so S / S_e accumulate in registers and the column sum
    // of fl is a shuffle reduction over its N consecutive lanes (64-bit shared
    // atomics are CAS loops on this GPU); other N use shared atomics.
    for (int t0 = 0; t0 < ft * N; t0 += EV2_THREADS) {
      const int t = t0 + threadIdx.x;
      const bool act = t < ft * N;
      const int fl = t / N, j = t - (t / N) * N;
      const int f = f0 + fl;
      long long full = 0, Rv = 0, Rev = 0;
      if (act && f != d) {
        for (int g = 0; g < N; ++g) {
          const long long qa = sQ[g * (FT + 1) + fl], qb = sQ[g * (FT + 1) + fl + 1];
          const int ra = sR[g * (FT + 1) + fl], rb = sR[g * (FT + 1) + fl + 1];
          full += (qb - qa) + (j < rb ? 1 : 0) - (j < ra ? 1 : 0);
        }
        Rv = full * C + (long long)(((unsigned long long)aRhi[t] << 32) | aRlo[t]);
        Rev = (long long)(((unsigned long long)aEhi[t] << 32) | aElo[t]);
      }
      if (Rv) atomicAdd(R + (long long)f * N + j, (unsigned long long)Rv);
      if (Rev) atomicAdd(Re + (long long)f * N + j, (unsigned long long)Rev);
      if (pow2) {
        accS += (unsigned long long)Rv;
        accSe += (unsigned long long)Rev;
        unsigned long long v = (unsigned long long)Rv;
        for (int o = 1; o < N; o <<= 1) v += __shfl_xor_sync(FULL, v, o);
        if (act && j == 0) sCol[fl] = v;
      } else {
        if (Rv) {
          atomicAdd(&sS[j], (unsigned long long)Rv);
          atomicAdd(&sCol[fl], (unsigned long long)Rv);
        }
        if (Rev) atomicAdd(&sSe[j], (unsigned long long)Rev);
      }
    }
    __syncthreads();
    for (int fl = threadIdx.x; fl < ft; fl += EV2_THREADS)
      if (sCol[fl]) atomicAdd(col + f0 + fl, sCol[fl]);
  }
  if (pow2) {  // per-rail totals of the register partials (thread t holds rail t mod N)
    sAcc[0][threadIdx.x] = accS;
    sAcc[1][threadIdx.x] = accSe;
    __syncthreads();
    if (threadIdx.x < N) {
      unsigned long long a = 0, b = 0;
      for (int t = threadIdx.x; t < EV2_THREADS; t += N) {
        a += sAcc[0][t];
        b += sAcc[1][t];
      }
      sS[threadIdx.x] = a;
      sSe[threadIdx.x] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  long long s = lane < N ? (long long)sS[lane] : 0, se = lane < N ? (long long)sSe[lane] : 0;
  if (lane < N) {
    S[seg * N + lane] = s;
    S_e[seg * N + lane] = se;
  }
  const long long total = warp_sum(s), total_e = warp_sum(se);
  const long long mx = warp_max(s), mxe = warp_max(se);
  unsigned __int128 sq = 0;
  for (int j = 0; j < N; ++j) {
    const long long sj = __shfl_sync(FULL, s, j);
    const __int128 dv = (__int128)N * sj - (__int128)total;
    sq += (unsigned __int128)(dv * dv);
  }
  if (lane == 0) {
    const double dN = (double)N;
    const double m = __ddiv_rn(u128_to_double(sq), __dmul_rn(__dmul_rn(dN, dN), dN));
    mse[seg] = m;
    nmse[seg] =
        total == 0 ? 0.0
                   : __ddiv_rn(m, __dmul_rn(__ll2double_rn(total), __ll2double_rn(total)));
    if (total) atomicAdd(tot, (unsigned long long)total);
    if (total_e) atomicAdd(tot + 1, (unsigned long long)total_e);
    atomicMax((long long*)red_max + u * RAILS_RED_MAX_LEN + 0, mx);
    atomicMax((long long*)red_max + u * RAILS_RED_MAX_LEN + 1, mxe);
    atomicMax((long long*)red_max + u * RAILS_RED_MAX_LEN + 2, total);
  }
}

__device__ void finalize_unit(long long u, int N, double R2, long long mR, long long mRe,
                              long long mc, long long rm0, long long rm1, long long rm2,
                              long long total, long long total_e, const rails_final_t& out);

__global__ void __launch_bounds__(256)
    k_eval_finalize(int M, int N, double R2, long long rsl, const int64_t* __restrict__ red_sum,
                    const int64_t* __restrict__ red_max, rails_final_t out) {
  __shared__ long long s3[3][8];
  const long long u = blockIdx.x;
  const int64_t* rs = red_sum + u * rsl;
  const long long MN = (long long)M * N;
  long long mR = 0, mRe = 0, mc = 0;
  for (long long i = threadIdx.x; i < MN; i += blockDim.x) {
    mR = max(mR, (long long)rs[i]);
    mRe = max(mRe, (long long)rs[MN + i]);
  }
  for (long long i = threadIdx.x; i < M; i += blockDim.x) mc = max(mc, (long long)rs[2 * MN + i]);
  mR = warp_max(mR);
  mRe = warp_max(mRe);
  mc = warp_max(mc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s3[0][wid] = mR;
    s3[1][wid] = mRe;
    s3[2][wid] = mc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    mR = max(mR, s3[0][w]);
    mRe = max(mRe, s3[1][w]);
    mc = max(mc, s3[2][w]);
  }
  const int64_t* rm = red_max + u * RAILS_RED_MAX_LEN;
  finalize_unit(u, N, R2, mR, mRe, mc, rm[0], rm[1], rm[2], rs[2 * MN + M], rs[2 * MN + M + 1],
                out);
}

// T, T*, busbw of unit u from the reduced maxima and totals (R#8, R#10, Thm 2/3).
__device__ void finalize_unit(long long u, int N, double R2, long long mR, long long mRe,
                              long long mc, long long rm0, long long rm1, long long rm2,
                              long long total, long long total_e, const rails_final_t& out) {
  const long long maxload = max(rm0, mR);
  const long long maxload_e = max(rm1, mRe);
  const long long rowmax = rm2;
  const double T = __ddiv_rn(__ll2double_rn(maxload), R2);
  const double T_e = __ddiv_rn(__ll2double_rn(maxload_e), R2);
  const long long lb = max(rowmax, mc);
  const double T_star = __ddiv_rn(__ll2double_rn(lb), __dmul_rn((double)N, R2));
  if (out.maxload) out.maxload[u] = maxload;
  if (out.maxload_e) out.maxload_e[u] = maxload_e;
  if (out.total) out.total[u] = total;
  if (out.rowmax) out.rowmax[u] = rowmax;
  if (out.colmax) out.colmax[u] = mc;
  if (out.T) out.T[u] = T;
  if (out.T_e) out.T_e[u] = T_e;
  if (out.T_star) out.T_star[u] = T_star;
  if (out.busbw) out.busbw[u] = total > 0 ? __ddiv_rn(__ll2double_rn(total), T) : 0.0;
  if (out.busbw_e) out.busbw_e[u] = total_e > 0 ? __ddiv_rn(__ll2double_rn(total_e), T_e) : 0.0;
}

// ---------------------------------------------------------------- a6 + finalize, peers
struct PeerBufs {
  uint8_t* p[RAILS_PEER_MAX];
};

__host__ __device__ static inline size_t al256e(size_t x) { return (x + 255) & ~(size_t)255; }

// [flags: U x world u32][slots: 2 (call parity) x world x U x rec int64]
size_t peer_buffer_bytes(int U, int world, long long rsl) {
  const long long rec = rsl + RAILS_RED_MAX_LEN;
  return al256e((size_t)U * world * 4) + 2 * (size_t)world * U * rec * 8;
}

// One CTA per unit: push this rank's partials to every rank, release a flag per
// (unit, rank), acquire every rank's flag, reduce the world's partials (in rank
// order, so every rank computes identical sums) and finalize the unit.  Slots are
// double-buffered by call parity and flags are waited on as ">= gen": a fast rank
// may push call gen+1 (other half) and bump its flag while a slow rank is still
// reading call gen, and it cannot get two calls ahead (call gen+1 waits for the
// slow rank's gen+1 flag).
__global__ void __launch_bounds__(256)
    k_finalize_peer(int M, int N, double R2, long long rsl, int U, int64_t* __restrict__ red_sum,
                    int64_t* __restrict__ red_max, PeerBufs pb, int rank, int world,
                    uint32_t gen, rails_final_t out, int* err) {
  __shared__ long long s3[3][8];
  __shared__ long long stot[2];
  const long long u = blockIdx.x;
  const long long rec = rsl + RAILS_RED_MAX_LEN;
  const size_t slots_off = al256e((size_t)U * world * 4) +
                           (size_t)(gen & 1u) * world * U * rec * 8;
  int64_t* rs = red_sum + u * rsl;
  int64_t* rmx = red_max + u * RAILS_RED_MAX_LEN;
  // 1. push (remote stores over NVLink for p != rank)
  for (int p = 0; p < world; ++p) {
    int64_t* dst = (int64_t*)(pb.p[p] + slots_off) + ((long long)rank * U + u) * rec;
    for (long long i = threadIdx.x; i < rec; i += blockDim.x)
      dst[i] = i < rsl ? rs[i] : rmx[i - rsl];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p)
      st_release_sys((uint32_t*)pb.p[p] + u * world + rank, gen);
  }
  // 2. wait for every rank's partials of this unit
  if (threadIdx.x < world)
    wait_flag_ge((const uint32_t*)pb.p[rank] + u * world + threadIdx.x, gen, err);
  __syncthreads();
  // 3. reduce in rank order (volatile loads: the data came from other GPUs)
  const volatile int64_t* slots = (const volatile int64_t*)(pb.p[rank] + slots_off);
  const long long MN = (long long)M * N;
  long long mR = 0, mRe = 0, mc = 0;
  for (long long i = threadIdx.x; i < rsl; i += blockDim.x) {
    long long v = 0;
    for (int p = 0; p < world; ++p) v += slots[((long long)p * U + u) * rec + i];
    rs[i] = v;
    if (i < MN) mR = max(mR, v);
    else if (i < 2 * MN) mRe = max(mRe, v);
    else if (i < 2 * MN + M) mc = max(mc, v);
    else stot[i - 2 * MN - M] = v;
  }
  if (threadIdx.x < RAILS_RED_MAX_LEN) {
    long long v = 0;
    for (int p = 0; p < world; ++p)
      v = max(v, (long long)slots[((long long)p * U + u) * rec + rsl + threadIdx.x]);
    rmx[threadIdx.x] = v;
  }
  mR = warp_max(mR);
  mRe = warp_max(mRe);
  mc = warp_max(mc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    s3[0][wid] = mR;
    s3[1][wid] = mRe;
    s3[2][wid] = mc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    mR = max(mR, s3[0][w]);
    mRe = max(mRe, s3[1][w]);
    mc = max(mc, s3[2][w]);
  }
  finalize_unit(u, N, R2, mR, mRe, mc, rmx[0], rmx[1], rmx[2], stot[0], stot[1], out);
}

cudaError_t launch_finalize_peer(const LaunchCtx& c, int U, int M, int N, double R2,
                                 int64_t* red_sum, int64_t* red_max, const rails_peer_t& peer,
                                 const rails_final_t& f) {
  PeerBufs pb;
  for (int p = 0; p < RAILS_PEER_MAX; ++p) pb.p[p] = (uint8_t*)(p < peer.world ? peer.buf[p] : nullptr);
  k_finalize_peer<<<(unsigned)U, 256, 0, c.stream>>>(M, N, R2, RAILS_RED_SUM_LEN(M, N), U, red_sum,
                                                     red_max, pb, peer.rank, peer.world, peer.gen,
                                                     f, c.err);
  count_launch(1);
  return cudaGetLastError();
}

// Exclusive prefix of send_load in (u, dl, j) order -> rail_base; total bytes.
__global__ void __launch_bounds__(1024)
    k_rail_offsets(long long n, const int64_t* __restrict__ send_load,
                   int64_t* __restrict__ rail_base, int64_t* __restrict__ total) {
  __shared__ long long scratch[33];
  long long carry = 0;
  for (long long t0 = 0; t0 < n; t0 += blockDim.x) {
    const long long i = t0 + threadIdx.x;
    const long long v = i < n ? send_load[i] : 0;
    long long tot;
    const long long ex = block_excl_scan(v, scratch, &tot);
    if (i < n) rail_base[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

static int pow2_shift(long long C) {
  if (C <= 0 || (C & (C - 1))) return -1;
  int s = 0;
  while ((1LL << s) < C) ++s;
  return s;
}

cudaError_t launch_eval(const LaunchCtx& c, int U, int nd, int d0, int M, int N, long long C,
                        uint64_t seed, const int64_t* msg, const rails_sched_t& s,
                        const rails_eval_t& e) {
  const long long rsl = RAILS_RED_SUM_LEN(M, N);
  cudaError_t err =
      cudaMemsetAsync(e.red_sum, 0, (size_t)U * rsl * sizeof(int64_t), c.stream);
  if (err != cudaSuccess) return err;
  err = cudaMemsetAsync(e.red_max, 0, (size_t)U * RAILS_RED_MAX_LEN * sizeof(int64_t), c.stream);
  if (err != cudaSuccess) return err;
  const char* ev = getenv("RAILS_EVAL_IMPL");
  if (ev && ev[0] == '1') {
    k_eval_node<<<(unsigned)((long long)U * nd), EVAL_WARPS * 32, 0, c.stream>>>(
        M, N, nd, d0, C, pow2_shift(C), seed, msg, s.full_base, s.rem_rail, e.S, e.S_e, e.mse,
        e.nmse, e.red_sum, e.red_max, rsl);
  } else {
    const int FT = (EV2_THREADS / N) < 64 ? (EV2_THREADS / N) : 64;
    const size_t smem = 16 + (size_t)N * (FT + 1) * (8 + 4);
    void (*kern)(int, int, int, int, long long, int, uint64_t, int, const int64_t*,
                 const int64_t*, const int8_t*, const int64_t*, int64_t*, int64_t*, double*,
                 double*, int64_t*, int64_t*, long long) =
        N == 2 ? k_eval_node2<2> : N == 4 ? k_eval_node2<4> : N == 8 ? k_eval_node2<8>
        : N == 16 ? k_eval_node2<16> : N == 32 ? k_eval_node2<32> : k_eval_node2<0>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    kern<<<(unsigned)((long long)U * nd), EV2_THREADS, smem, c.stream>>>(
        M, N, nd, d0, C, pow2_shift(C), seed, FT, msg, s.full_base, s.rem_rail, s.n_full, e.S,
        e.S_e, e.mse, e.nmse, e.red_sum, e.red_max, rsl);
  }
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const LaunchCtx& c, int U, int M, int N, double R2,
                            const int64_t* red_sum, const int64_t* red_max,
                            const rails_final_t& f) {
  k_eval_finalize<<<(unsigned)U, 256, 0, c.stream>>>(M, N, R2, RAILS_RED_SUM_LEN(M, N), red_sum,
                                                     red_max, f);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_rail_offsets(const LaunchCtx& c, long long n, const int64_t* send_load,
                                int64_t* rail_base, int64_t* total) {
  k_rail_offsets<<<1, 1024, 0, c.stream>>>(n, send_load, rail_base, total);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace rails
