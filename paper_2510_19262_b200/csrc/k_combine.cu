// k_combine.cu -- NEXT f1: the combine all-to-all (Alg. 1 step 4).
//
// Expert outputs return from expert GPU h = f*N+m to the token's GPU a = d*N+g.
// The combine round is a second all-to-all with its own LoadState:
//   k_transpose    D_c[f][m][a] = D_d[a][f*N+m]                        (R#28)
//   k_recv_offsets in_off[b][a] = first row of dispatch message a in the
//                  expert-output buffer y of GPU b (messages in ascending a)  (R#29)
//   (then rails_lpt_schedule / rails_eval on D_c, unchanged)
//   k_pack_combine combine message (m, a) = rows in_off[m][a] .. of y_m, cut into
//                  the combine schedule's chunks -> rail buffers of node f   (R#30)
//   k_unpack_combine on GPU (d,g): out[t] = sum_s w[t][s] * row(t,s) in fp32, s in
//                  order, each product and sum rounded (no FMA); row(t,s) is
//                  gathered from node f's combine rail buffers at the chunk holding
//                  message byte rho*RB (rho = dispatch rank), or from y directly
//                  when the expert sits on node d (intra-node, never railed) (R#31)
#include "common.cuh"

namespace rails {

// ---------------------------------------------------------------- transpose
__global__ void __launch_bounds__(1024)
    k_transpose(long long G, const int64_t* __restrict__ src, int64_t* __restrict__ dst) {
  __shared__ long long tile[32][33];
  const long long u = blockIdx.z;
  const long long a0 = (long long)blockIdx.y * 32, b0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t* s = src + u * G * G;
  int64_t* o = dst + u * G * G;
  if (a0 + ty < G && b0 + tx < G) tile[ty][tx] = s[(a0 + ty) * G + b0 + tx];
  __syncthreads();
  if (b0 + ty < G && a0 + tx < G) o[(b0 + ty) * G + a0 + tx] = tile[tx][ty];
}

// ---------------------------------------------------------------- receive offsets
// counts [U][G(a)][G(b)] int32 (dispatch, all nodes) -> in_off [U][G(b)][G(a)] int64
// exclusive prefix over a of counts[a][b]; rows_in [U][G(b)] = column total.
__global__ void __launch_bounds__(256)
    k_recv_offsets(long long G, const int32_t* __restrict__ counts, int64_t* __restrict__ in_off,
                   int64_t* __restrict__ rows_in) {
  __shared__ long long scratch[33];
  const long long ub = blockIdx.x;  // u*G + b
  const long long u = ub / G, b = ub - u * G;
  const int32_t* c = counts + u * G * G + b;
  int64_t* o = in_off + ub * G;
  long long carry = 0;
  for (long long t0 = 0; t0 < G; t0 += blockDim.x) {
    const long long a = t0 + threadIdx.x;
    const long long v = a < G ? (long long)c[a * G] : 0;
    long long tot;
    const long long ex = block_excl_scan(v, scratch, &tot);
    if (a < G) o[a] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) rows_in[ub] = carry;
}

// ---------------------------------------------------------------- shared address logic
struct CSched {
  const int64_t* full_base;
  const int8_t* rem_rail;
  const int64_t* rem_off;
};

// byte address (in `out`) of message byte p of message mi whose node block has rail
// bases rbase[0..N): full chunk -> rail (fb+c) mod N, else the remainder.
__device__ __forceinline__ long long msg_byte_addr(long long p, long long mi, long long nfull,
                                                   const CSched& s, int N, long long C,
                                                   const ChunkDiv& cd,
                                                   const int64_t* __restrict__ rbase) {
  const long long c = cd.div(p);
  const long long in_c = p - c * C;
  if (c < nfull) {
    const long long i = s.full_base[mi] + c;
    const long long q = i / N;
    return rbase[i - q * N] + q * C + in_c;
  }
  const int rr = s.rem_rail[mi];
  return rr >= 0 ? rbase[rr] + s.rem_off[mi] + in_c : -(1LL << 62);
}

// ---------------------------------------------------------------- combine pack
constexpr int CP_THREADS = 256;

template <int VPL>
__global__ void __launch_bounds__(CP_THREADS)
    k_pack_combine(int U, int nd, int d0, int M, int N, long long Rcap, long long C, int cshift,
                   const uint4* __restrict__ y, const int64_t* __restrict__ in_off,
                   const int64_t* __restrict__ rows_in, const int64_t* __restrict__ msgc,
                   CSched s, const int64_t* __restrict__ rail_base, uint8_t* __restrict__ out,
                   long long out_cap, long long RB, int* err) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (CP_THREADS / 32);
  const long long G = (long long)M * N;
  const long long rows = (long long)U * nd * N * Rcap;
  const int nvec = (int)(RB >> 4);
  const ChunkDiv cd{C, cshift};
  for (long long row = (long long)blockIdx.x * (CP_THREADS / 32) + (threadIdx.x >> 5);
       row < rows; row += nwarps) {
    const long long um = row / Rcap;  // (u*nd + dl)*N + m  (sender GPU f*N+m)
    const long long r = row - um * Rcap;
    const long long ul = um / N;
    const int m = (int)(um - ul * N);
    const long long u = ul / nd;
    const int f = d0 + (int)(ul - u * nd);
    const long long b = (long long)f * N + m;
    if (r >= rows_in[u * G + b]) continue;
    // the row's first window of payload loads is in flight while the message and
    // chunk lookups (a binary search, then the schedule) run
    const uint4* src = y + row * nvec;
    uint4 v[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int vi = i * 32 + lane;
      if (vi < nvec) v[i] = ld_stream(src + vi);
    }
    // message a: largest a with in_off[a] <= r (empty messages share offsets)
    const int64_t* io = in_off + (u * G + b) * G;
    long long lo = 0, hi = G - 1;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (io[mid] <= r) lo = mid; else hi = mid - 1;
    }
    const long long a = lo;
    if (a / N == f) continue;  // intra-node: never railed (R#2)
    const long long mi = um * G + a;
    const long long B = msgc[mi];
    const long long p0 = (r - io[a]) * RB;
    if (p0 + RB > B) {
      flag_error(err, ERR_RANGE);
      continue;
    }
    const long long nfull = cd.div(B);
    const int64_t* rbase = rail_base + ul * N;
    // C >= RB: the row lies in at most two chunks (bytes [0, b0) and [b0, RB))
    const long long c0 = cd.div(p0);
    const long long b0 = min((c0 + 1) * C - p0, RB);
    const long long dst0 = msg_byte_addr(p0, mi, nfull, s, N, C, cd, rbase);
    const long long dst1 = (C >= RB && b0 < RB)
                               ? msg_byte_addr(p0 + b0, mi, nfull, s, N, C, cd, rbase)
                               : 0;
    for (int w0 = 0; w0 < nvec; w0 += VPL * 32) {
      if (w0 > 0) {
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int vi = w0 + i * 32 + lane;
          if (vi < nvec) v[i] = ld_stream(src + vi);
        }
      }
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int vi = w0 + i * 32 + lane;
        if (vi < nvec) {
          const long long o = (long long)vi << 4;
          long long addr;
          if (o < b0) addr = dst0 < 0 ? -1 : dst0 + o;
          else if (C >= RB) addr = dst1 < 0 ? -1 : dst1 + (o - b0);
          else addr = msg_byte_addr(p0 + o, mi, nfull, s, N, C, cd, rbase);
          if (addr >= 0 && addr + 16 <= out_cap)
            st_stream((uint4*)(out + addr), v[i]);
          else
            flag_error(err, ERR_NOSPC);
        }
      }
    }
  }
}

// ---------------------------------------------------------------- unpack + combine
constexpr int UP_THREADS = 256;
constexpr int UP_VW = 4;  // 16-byte vectors per lane per window (32 fp32 accumulators)

__device__ __forceinline__ void bf16x8_fma(float* acc, const uint4& v, float w) {
  const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(q[i] << 16);
    const float hi = __uint_as_float(q[i] & 0xffff0000u);
    acc[2 * i] = __fadd_rn(acc[2 * i], __fmul_rn(w, lo));
    acc[2 * i + 1] = __fadd_rn(acc[2 * i + 1], __fmul_rn(w, hi));
  }
}

// KS = k known at compile time (1 or 2): the window issues every slot's loads
// before the first multiply-add (the slots' rows are independent gathers), with
// the per-slot metadata broadcast once per token.  KS = 0: any k, slot by slot.
// The fp32 sum is formed in slot order either way (R#31).
template <int KS>
__global__ void __launch_bounds__(UP_THREADS)
    k_unpack_combine(int U, int nd, int d0, int M, int N, int T, int k, long long C, int cshift,
                     const int32_t* __restrict__ topk, const int32_t* __restrict__ lut,
                     int n_inst, const int32_t* __restrict__ rank, const float* __restrict__ wts,
                     const uint4* __restrict__ y, long long Rcap,
                     const int64_t* __restrict__ in_off, const int64_t* __restrict__ msgc,
                     CSched s, const int64_t* __restrict__ rail_base_c,
                     const uint8_t* __restrict__ comb_out, float* __restrict__ out, long long RB,
                     int* err) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (UP_THREADS / 32);
  const long long G = (long long)M * N;
  const long long tokens = (long long)U * nd * N * T;
  const int nvec = (int)(RB >> 4);
  const ChunkDiv cd{C, cshift};
  for (long long tok = (long long)blockIdx.x * (UP_THREADS / 32) + (threadIdx.x >> 5);
       tok < tokens; tok += nwarps) {
    const long long ug = tok / T;  // (u*nd + dl)*N + g
    const long long ul = ug / N;
    const int g = (int)(ug - ul * N);
    const long long u = ul / nd;
    const int d = d0 + (int)(ul - u * nd);
    const long long a = (long long)d * N + g;
    // slot metadata on lanes < k: source of row bytes [0, RB)
    long long srcA = -1, srcB = -1, mi = 0, p0 = 0, nfull = 0;
    int bsplit = 0, intra = 0, ok = 0;
    long long fblk = 0;
    float w = 0.f;
    if (lane < k) {
      const long long e = tok * k + lane;
      const int inst = __ldg(topk + e);
      const int h = (inst >= 0 && inst < n_inst) ? __ldg(lut + inst) : -1;
      const int rk = rank[e];
      w = wts[e];
      if (h < 0 || h >= G || rk < 0) {
        flag_error(err, ERR_RANGE);
      } else {
        const int f = h / N, m = h - (h / N) * N;
        if (f == d) {
          // expert on this node: its output row is in y of GPU (d, m)
          const long long um = (u * nd + (d - d0)) * N + m;
          srcA = (um * Rcap + in_off[(u * G + h) * G + a] + rk) * RB;
          intra = 1;
          ok = 1;
        } else {
          fblk = u * M + f;
          mi = (fblk * N + m) * G + a;
          const long long B = msgc[mi];
          p0 = (long long)rk * RB;
          if (p0 + RB > B) {
            flag_error(err, ERR_RANGE);
          } else {
            nfull = cd.div(B);
            const int64_t* rb = rail_base_c + fblk * N;
            srcA = msg_byte_addr(p0, mi, nfull, s, N, C, cd, rb);
            const long long c0 = cd.div(p0);
            const long long b0 = (c0 + 1) * C - p0;
            bsplit = (int)(b0 < RB ? b0 : RB);
            if (bsplit < RB) srcB = msg_byte_addr(p0 + bsplit, mi, nfull, s, N, C, cd, rb);
            ok = 1;
          }
        }
      }
    }
    float* dst = out + tok * (RB >> 1);
    if constexpr (KS > 0) {
      constexpr int VW = KS == 1 ? 4 : 2;
      int okv[KS], inv_[KS], bsv[KS];
      float wsv[KS];
      long long Av[KS], Bv[KS], P0v[KS], MIv[KS], NFv[KS], FBv[KS];
#pragma unroll
      for (int sl = 0; sl < KS; ++sl) {
        okv[sl] = __shfl_sync(FULL, ok, sl);
        wsv[sl] = __shfl_sync(FULL, w, sl);
        inv_[sl] = __shfl_sync(FULL, intra, sl);
        Av[sl] = __shfl_sync(FULL, srcA, sl);
        Bv[sl] = __shfl_sync(FULL, srcB, sl);
        bsv[sl] = __shfl_sync(FULL, bsplit, sl);
        P0v[sl] = __shfl_sync(FULL, p0, sl);
        MIv[sl] = __shfl_sync(FULL, mi, sl);
        NFv[sl] = __shfl_sync(FULL, nfull, sl);
        FBv[sl] = __shfl_sync(FULL, fblk, sl);
      }
      for (int w0 = 0; w0 < nvec; w0 += VW * 32) {
        uint4 v[KS][VW];
#pragma unroll
        for (int sl = 0; sl < KS; ++sl) {
#pragma unroll
          for (int i = 0; i < VW; ++i) {
            const int vi = w0 + i * 32 + lane;
            v[sl][i] = make_uint4(0, 0, 0, 0);
            if (okv[sl] && vi < nvec) {
              const long long o = (long long)vi << 4;
              if (inv_[sl]) {
                v[sl][i] = ld_stream((const uint4*)((const uint8_t*)y + Av[sl] + o));
              } else {
                long long addr;
                if (o < bsv[sl]) addr = Av[sl] + o;
                else if (C >= RB) addr = Bv[sl] + (o - bsv[sl]);
                else addr = msg_byte_addr(P0v[sl] + o, MIv[sl], NFv[sl], s, N, C, cd,
                                          rail_base_c + FBv[sl] * N);
                v[sl][i] = ld_stream((const uint4*)(comb_out + addr));
              }
            }
          }
        }
        float acc[VW * 8];
#pragma unroll
        for (int q = 0; q < VW * 8; ++q) acc[q] = 0.f;
#pragma unroll
        for (int sl = 0; sl < KS; ++sl) {
          if (!okv[sl]) continue;
#pragma unroll
          for (int i = 0; i < VW; ++i) bf16x8_fma(acc + 8 * i, v[sl][i], wsv[sl]);
        }
#pragma unroll
        for (int i = 0; i < VW; ++i) {
          const int vi = w0 + i * 32 + lane;
          if (vi < nvec) {
            float4* p = (float4*)(dst + (long long)vi * 8);
            st_cs((uint4*)p, make_uint4(__float_as_uint(acc[8 * i]), __float_as_uint(acc[8 * i + 1]),
                                        __float_as_uint(acc[8 * i + 2]),
                                        __float_as_uint(acc[8 * i + 3])));
            st_cs((uint4*)p + 1,
                  make_uint4(__float_as_uint(acc[8 * i + 4]), __float_as_uint(acc[8 * i + 5]),
                             __float_as_uint(acc[8 * i + 6]), __float_as_uint(acc[8 * i + 7])));
          }
        }
      }
      continue;
    }
    for (int w0 = 0; w0 < nvec; w0 += UP_VW * 32) {
      float acc[UP_VW * 8];
#pragma unroll
      for (int i = 0; i < UP_VW * 8; ++i) acc[i] = 0.f;
      for (int sl = 0; sl < k; ++sl) {
        if (!__shfl_sync(FULL, ok, sl)) continue;
        const float ws = __shfl_sync(FULL, w, sl);
        const int in = __shfl_sync(FULL, intra, sl);
        const long long A = __shfl_sync(FULL, srcA, sl);
        const long long Bs = __shfl_sync(FULL, srcB, sl);
        const int bs = __shfl_sync(FULL, bsplit, sl);
        const long long P0 = __shfl_sync(FULL, p0, sl);
        const long long MI = __shfl_sync(FULL, mi, sl);
        const long long NF = __shfl_sync(FULL, nfull, sl);
        const long long FB = __shfl_sync(FULL, fblk, sl);
#pragma unroll
        for (int i = 0; i < UP_VW; ++i) {
          const int vi = w0 + i * 32 + lane;
          if (vi < nvec) {
            const long long o = (long long)vi << 4;
            uint4 v;
            if (in) {
              v = ld_stream((const uint4*)((const uint8_t*)y + A + o));
            } else {
              long long addr;
              if (o < bs) addr = A + o;
              else if (C >= RB) addr = Bs + (o - bs);
              else addr = msg_byte_addr(P0 + o, MI, NF, s, N, C, cd, rail_base_c + FB * N);
              v = ld_stream((const uint4*)(comb_out + addr));
            }
            bf16x8_fma(acc + 8 * i, v, ws);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < UP_VW; ++i) {
        const int vi = w0 + i * 32 + lane;
        if (vi < nvec) {
          float4* p = (float4*)(dst + (long long)vi * 8);
          p[0] = make_float4(acc[8 * i], acc[8 * i + 1], acc[8 * i + 2], acc[8 * i + 3]);
          p[1] = make_float4(acc[8 * i + 4], acc[8 * i + 5], acc[8 * i + 6], acc[8 * i + 7]);
        }
      }
    }
  }
}

static int cshift_of(long long C) {
  if (C <= 0 || (C & (C - 1))) return -1;
  int s = 0;
  while ((1LL << s) < C) ++s;
  return s;
}

cudaError_t launch_transpose(const LaunchCtx& c, int U, long long G, const int64_t* src,
                             int64_t* dst) {
  dim3 grid((unsigned)((G + 31) / 32), (unsigned)((G + 31) / 32), (unsigned)U);
  k_transpose<<<grid, dim3(32, 32), 0, c.stream>>>(G, src, dst);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_recv_offsets(const LaunchCtx& c, int U, long long G, const int32_t* counts,
                                int64_t* in_off, int64_t* rows_in) {
  k_recv_offsets<<<(unsigned)(U * G), 256, 0, c.stream>>>(G, counts, in_off, rows_in);
  count_launch(1);
  return cudaGetLastError();
}

template <int VPL>
static cudaError_t launch_pc(const LaunchCtx& c, int U, int nd, int d0, int M, int N,
                             long long Rcap, long long C, const void* y, const int64_t* in_off,
                             const int64_t* rows_in, const int64_t* msgc, const rails_sched_t& s,
                             const int64_t* rail_base, void* out, long long out_cap,
                             long long RB) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pack_combine<VPL>,
                                                                CP_THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long rows = (long long)U * nd * N * Rcap;
  const long long need = (rows + CP_THREADS / 32 - 1) / (CP_THREADS / 32);
  // persistent grid by default: waves of CTAs measured equal here (RAILS_COMBINE_RPW=8)
  const long long grid = wave_grid(c.num_sms, per_sm, need, 0);
  CSched cs{s.full_base, s.rem_rail, s.rem_off};
  k_pack_combine<VPL><<<(unsigned)grid, CP_THREADS, 0, c.stream>>>(
      U, nd, d0, M, N, Rcap, C, cshift_of(C), (const uint4*)y, in_off, rows_in, msgc, cs,
      rail_base, (uint8_t*)out, out_cap, RB, c.err);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_pack_combine(const LaunchCtx& c, int U, int nd, int d0, int M, int N,
                                long long Rcap, long long C, const void* y,
                                const int64_t* in_off, const int64_t* rows_in,
                                const int64_t* msgc, const rails_sched_t& s,
                                const int64_t* rail_base, void* out, long long out_cap,
                                long long RB) {
  const long long vpl = ((RB >> 4) + 31) / 32;
  if (vpl <= 4)
    return launch_pc<4>(c, U, nd, d0, M, N, Rcap, C, y, in_off, rows_in, msgc, s, rail_base, out,
                        out_cap, RB);
  return launch_pc<8>(c, U, nd, d0, M, N, Rcap, C, y, in_off, rows_in, msgc, s, rail_base, out,
                      out_cap, RB);
}

cudaError_t launch_unpack_combine(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int T,
                                  int k, long long C, const int32_t* topk, const int32_t* lut,
                                  int n_inst, const int32_t* rank, const float* w, const void* y,
                                  long long Rcap, const int64_t* in_off, const int64_t* msgc,
                                  const rails_sched_t& s, const int64_t* rail_base_c,
                                  const void* comb_out, float* out, long long RB) {
  int per_sm = 0;
  void (*kern)(int, int, int, int, int, int, int, long long, int, const int32_t*,
               const int32_t*, int, const int32_t*, const float*, const uint4*, long long,
               const int64_t*, const int64_t*, CSched, const int64_t*, const uint8_t*, float*,
               long long, int*) =
      k == 1 ? k_unpack_combine<1> : k == 2 ? k_unpack_combine<2> : k_unpack_combine<0>;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, UP_THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long toks = (long long)U * nd * N * T;
  const long long need = (toks + UP_THREADS / 32 - 1) / (UP_THREADS / 32);
  // persistent grid by default: waves of CTAs measured 2% slower here (RAILS_UNPACK_RPW=8)
  const long long grid = wave_grid(c.num_sms, per_sm, need, 0);
  CSched cs{s.full_base, s.rem_rail, s.rem_off};
  kern<<<(unsigned)grid, UP_THREADS, 0, c.stream>>>(
      U, nd, d0, M, N, T, k, C, cshift_of(C), topk, lut, n_inst, rank, w, (const uint4*)y, Rcap,
      in_off, msgc, cs, rail_base_c, (const uint8_t*)comb_out, out, RB, c.err);
  count_launch(1);
  return cudaGetLastError();
}

}  // namespace rails
