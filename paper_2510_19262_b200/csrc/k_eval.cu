// k_eval.cu -- a5 for a given schedule: loads, completion time, T*, busbw, MSE,
// ECMP and uniform baselines (sm_100a); a6 fused with the finalize over peer memory.
//
// Load model (Eq. 4-5; rail pairing NIC(k,n) -> NIC(f,n), R#7):
// a chunk of node d on rail j bound for node f adds to S[d][j] and R[f][j].
// From the compact schedule, message (g,h) with n = floor(B/C) full chunks
// starting at node-global full index fb puts q*C on every rail plus C on the r
// rails fb mod N, fb+1 mod N, ... (q = n div N, r = n mod N), and its remainder on
// rem_rail.  So eval is O(messages * N), never O(chunks).  The hot path evaluates
// inside the fused per-node kernel (k_node.cu); k_eval_node here serves
// rails_eval on any given schedule (e.g. the combine round) and the fallback for
// nodes too large for the fused kernel's shared memory.
//
// k_eval_node: one CTA per (unit, node), destination nodes in tiles of 256/N;
// stage 1 adds each message's remainder (on rem_rail), ECMP bytes (R#13-R#14)
// and uniform split (R#41: quotient per destination node, remainder histogram per
// (node, B mod N)) into per-(f, j) shared sums; stage 2 runs one thread per (f, j),
// adds the full chunks by the closed form above (messages of fixed g and f are
// contiguous in (g,h) order, so their full chunks form ONE index range [a, b); rail
// j receives cnt(b) - cnt(a), cnt(x) = floor(x/N) + (j < x mod N)), and adds
// R[f][j], R_e, R_u into the unit's red_sum (int64 atomics: order-free, hence
// deterministic).  MSE (Eq. 6; R#11) is the exact integer
// sum_j (N*S_j - sum S)^2 over N^3, converted once (R#25).
// k_eval_finalize: per unit, T = maxload/R2, T* = max(rowmax,
// colmax)/(N*R2) (Thm 2 + Thm 3), busbw = total/T (R#10, R#40), same for ECMP and
// uniform.
#include "common.cuh"
#include "eval.cuh"

namespace rails {

constexpr int EV2_THREADS = 256;

// NT = 8 (divisions by shifts) or 0 (runtime N).  MINB: CTAs per SM the registers
// are capped for -- 4 (64 registers) in general; 6 (40) when one tile holds every
// destination (M*N < 256, several source GPUs per thread: C2 757 -> 714 us, while
// C4's wide tiles lose 35 us at 6)
template <int NT, int MINB = 4>
__global__ void __launch_bounds__(EV2_THREADS, MINB)
    k_eval_node(int M, int N_rt, int nd, int d0, long long C, int cshift, uint64_t seed, int FT,
                const int64_t* __restrict__ msg, const int64_t* __restrict__ full_base,
                const int8_t* __restrict__ rem_rail, const int64_t* __restrict__ n_full,
                rails_eval_t ev, const int32_t* __restrict__ ex_inv,
                const uint64_t* __restrict__ ex_res, int8_t* __restrict__ ex_rail,
                int64_t* __restrict__ ex_off) {
  extern __shared__ __align__(16) uint8_t ev_smem[];
  __shared__ unsigned long long sS[32], sSe[32], sSu[32], sCol[EV2_THREADS];
  // per (fl, j) of the tile: remainder bytes into NIC (f, j), ECMP bytes; uniform:
  // remainder counts per (fl, B mod N) and quotient sums per fl.  64-bit sums as two
  // fire-and-forget 32-bit shared reductions (add_split20: a bin gets <= N^2 adds)
  __shared__ unsigned aRlo[EV2_THREADS], aRhi[EV2_THREADS], aElo[EV2_THREADS],
      aEhi[EV2_THREADS], cU[EV2_THREADS], aQlo[EV2_THREADS], aQhi[EV2_THREADS];
  const int N = NT ? NT : N_rt;
  const long long seg = blockIdx.x;
  const long long u = seg / nd;
  const int d = d0 + (int)(seg % nd);
  const long long G = (long long)M * N, NG = (long long)N * G;
  const ChunkDiv cd{C, cshift};
  const int64_t* __restrict__ mg = msg + seg * NG;
  const int64_t* __restrict__ fbp = full_base + seg * NG;
  const int8_t* __restrict__ rrp = rem_rail + seg * NG;
  // expand mode (ex_inv != nullptr): rem_rail / rem_off of every message come from the
  // chains' results through the inverse permutation and are written here
  const bool ex = ex_inv != nullptr;
  const int32_t* __restrict__ xinv = ex ? ex_inv + seg * NG : nullptr;
  const uint64_t* __restrict__ xres = ex ? ex_res + seg * NG : nullptr;
  int8_t* __restrict__ xrail = ex ? ex_rail + seg * NG : nullptr;
  int64_t* __restrict__ xoff = ex ? ex_off + seg * NG : nullptr;
  constexpr uint64_t XOFF_MASK = (1ull << 56) - 1;  // results: rail << 56 | offset
  const long long nfull_node = n_full[seg];
  const RedLayout RL{(long long)M * N, M};
  unsigned long long* rs = (unsigned long long*)(ev.red_sum + u * RL.len());

  long long* sQ = (long long*)ev_smem;  // [N][FT+1]
  int* sR = (int*)(sQ + N * (FT + 1));  // [N][FT+1]
  if (threadIdx.x < 32) sS[threadIdx.x] = sSe[threadIdx.x] = sSu[threadIdx.x] = 0;
  const bool jfix = (EV2_THREADS % N) == 0, wlanes = (32 % N) == 0;
  unsigned long long ps = 0, pe = 0, pu = 0;
  for (int f0 = 0; f0 < M; f0 += FT) {
    const int ft = min(FT, M - f0);
    __syncthreads();
    sCol[threadIdx.x] = 0;
    aRlo[threadIdx.x] = aRhi[threadIdx.x] = aElo[threadIdx.x] = aEhi[threadIdx.x] = 0u;
    cU[threadIdx.x] = aQlo[threadIdx.x] = aQhi[threadIdx.x] = 0u;
    // block boundaries of this tile: full index at message (g, (f0+fl)*N), fl = 0..ft
    // (N*(ft+1) <= 256 + N <= 2 per thread), loaded now so their latency overlaps
    // stage 1; converted into sQ / sR after it
    long long bnd[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t = threadIdx.x + q * EV2_THREADS;
      if (t < N * (ft + 1)) {
        const int g = t / (ft + 1), fl = t - g * (ft + 1);
        const long long p = (long long)g * G + (long long)(f0 + fl) * N;
        bnd[q] = (p < NG) ? fbp[p] : nfull_node;
      }
    }
    __syncthreads();
    // stage 1: t = g * (ft*N) + rest with h = f0*N + rest; a thread takes one
    // `rest` for every g (small tiles: threads beyond the tile's width split g)
    const int tn = ft * N;
    const int gsp = tn >= EV2_THREADS ? 1 : EV2_THREADS / tn;
    for (int r0 = 0; r0 < tn; r0 += EV2_THREADS) {
      const int rest = r0 + (gsp > 1 ? threadIdx.x % tn : threadIdx.x);
      const int gq = gsp > 1 ? threadIdx.x / tn : 0;
      if (rest >= tn || gq >= gsp) continue;
      const long long h = (long long)f0 * N + rest;
      const int fl = rest / N, fb = fl * N;  // (fl, 0) of this message's destination
      auto add_msg = [&](int g, long long B, int8_t rv) {
        if (B <= 0 || (int)(h / N) == d) return;
        const long long nf = cd.div(B);
        const long long rem = B - nf * C;
        if (rem && rv >= 0 && rv < N)
          add_split20(&aRlo[fb + rv], &aRhi[fb + rv], (unsigned long long)rem);
        const int e = ecmp_rail(seed, (long long)d * N + g, h, N);
        add_split20(&aElo[fb + e], &aEhi[fb + e], (unsigned long long)B);
        long long qb;
        int rb;
        divmod_n(B, N, qb, rb);
        if (qb) add_split20(&aQlo[fl], &aQhi[fl], (unsigned long long)qb);
        if (rb) atomicAdd(&cU[fb + rb], 1u);
      };
      // expand: message idx's remainder result (rail, offset), written out
      auto expand = [&](long long idx, int p, uint64_t v) -> int8_t {
        const int8_t r = p >= 0 ? (int8_t)(v >> 56) : (int8_t)-1;
        xrail[idx] = r;
        xoff[idx] = p >= 0 ? (long long)(v & XOFF_MASK) : 0;
        return r;
      };
      if (NT != 0 && gsp == 1) {
        // all N source GPUs' loads in flight at once (one DRAM latency per tile)
        long long Bv[NT ? NT : 1];
        int8_t rvv[NT ? NT : 1];
        if (ex) {
          int pv[NT ? NT : 1];
          uint64_t vv[NT ? NT : 1];
#pragma unroll
          for (int g = 0; g < NT; ++g) {
            Bv[g] = mg[(long long)g * G + h];
            pv[g] = xinv[(long long)g * G + h];
          }
#pragma unroll
          for (int g = 0; g < NT; ++g) vv[g] = pv[g] >= 0 ? xres[pv[g]] : 0ull;
#pragma unroll
          for (int g = 0; g < NT; ++g) rvv[g] = expand((long long)g * G + h, pv[g], vv[g]);
        } else {
#pragma unroll
          for (int g = 0; g < NT; ++g) {
            Bv[g] = mg[(long long)g * G + h];
            rvv[g] = rrp[(long long)g * G + h];
          }
        }
#pragma unroll
        for (int g = 0; g < NT; ++g) add_msg(g, Bv[g], rvv[g]);
      } else {
        for (int g = gq; g < N; g += gsp) {
          const long long idx = (long long)g * G + h;
          int8_t rv;
          if (ex) {
            const int p = xinv[idx];
            rv = expand(idx, p, p >= 0 ? xres[p] : 0ull);
          } else {
            rv = rrp[idx];
          }
          add_msg(g, mg[idx], rv);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t = threadIdx.x + q * EV2_THREADS;
      if (t < N * (ft + 1)) {
        const int g = t / (ft + 1), fl = t - g * (ft + 1);
        long long qq;
        int r;
        divmod_n(bnd[q], N, qq, r);
        sQ[g * (FT + 1) + fl] = qq;
        sR[g * (FT + 1) + fl] = r;
      }
    }
    __syncthreads();
    // stage 2: thread per (fl, j).  When N divides the block, j = t mod N is the
    // same for a thread in every tile, so S / S_e / S_u accumulate in registers;
    // when N divides 32 the column sum of fl is a shuffle reduction over its N
    // consecutive lanes (64-bit shared atomics are CAS loops on this GPU); other N
    // use shared atomics.
    for (int t0 = 0; t0 < ft * N; t0 += EV2_THREADS) {
      const int t = t0 + threadIdx.x;
      const int fl = t / N, j = t - (t / N) * N;
      const int f = f0 + fl;
      const bool act = t < ft * N && f != d;
      unsigned long long Rv = 0, Rev = 0, Ruv = 0;
      if (act) {
        long long full = 0;
        for (int g = 0; g < N; ++g) {
          const long long qa = sQ[g * (FT + 1) + fl], qb = sQ[g * (FT + 1) + fl + 1];
          const int ra = sR[g * (FT + 1) + fl], rb = sR[g * (FT + 1) + fl + 1];
          full += (qb - qa) + (j < rb ? 1 : 0) - (j < ra ? 1 : 0);
        }
        Rv = (unsigned long long)(full * C) + get_split20(aRlo[t], aRhi[t]);
        Rev = get_split20(aElo[t], aEhi[t]);
        Ruv = get_split20(aQlo[fl], aQhi[fl]);
        for (int r = j + 1; r < N; ++r) Ruv += cU[fl * N + r];
        if (Rv) atomicAdd(rs + RL.R() + (long long)f * N + j, Rv);
        if (Rev) atomicAdd(rs + RL.Re() + (long long)f * N + j, Rev);
        if (Ruv) atomicAdd(rs + RL.Ru() + (long long)f * N + j, Ruv);
      }
      if (jfix) {
        ps += Rv;
        pe += Rev;
        pu += Ruv;
      } else if (act) {
        if (Rv) atomicAdd(&sS[j], Rv);
        if (Rev) atomicAdd(&sSe[j], Rev);
        if (Ruv) atomicAdd(&sSu[j], Ruv);
      }
      if (wlanes) {
        unsigned long long v = Rv;
        for (int o = 1; o < N; o <<= 1) v += __shfl_xor_sync(FULL, v, o);
        if (act && j == 0 && v) atomicAdd(rs + RL.col() + f, v);
      } else if (act && Rv) {
        atomicAdd(&sCol[fl], Rv);
      }
    }
    __syncthreads();
    if (!wlanes)
      for (int fl = threadIdx.x; fl < ft; fl += EV2_THREADS)
        if (sCol[fl]) atomicAdd(rs + RL.col() + f0 + fl, sCol[fl]);
  }
  if (jfix) {  // per-rail totals of the register partials (thread t holds rail t mod N)
    __syncthreads();
    __shared__ unsigned long long part[3][EV2_THREADS];
    part[0][threadIdx.x] = ps;
    part[1][threadIdx.x] = pe;
    part[2][threadIdx.x] = pu;
    __syncthreads();
    if (threadIdx.x < N) {
      unsigned long long a = 0, b = 0, c2 = 0;
      for (int t = threadIdx.x; t < EV2_THREADS; t += N) {
        a += part[0][t];
        b += part[1][t];
        c2 += part[2][t];
      }
      sS[threadIdx.x] = a;
      sSe[threadIdx.x] = b;
      sSu[threadIdx.x] = c2;
    }
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const long long s = lane < N ? (long long)sS[lane] : 0, se = lane < N ? (long long)sSe[lane] : 0,
                  su = lane < N ? (long long)sSu[lane] : 0;
  if (lane < N) {
    ev.S[seg * N + lane] = s;
    ev.S_e[seg * N + lane] = se;
    ev.S_u[seg * N + lane] = su;
  }
  const long long total = warp_sum(s), total_e = warp_sum(se);
  const long long mx = warp_max(s), mxe = warp_max(se), mxu = warp_max(su);
  double mse, nmse;
  warp_mse(s, N, total, &mse, &nmse);
  if (lane == 0) {
    ev.mse[seg] = mse;
    ev.nmse[seg] = nmse;
    if (total) atomicAdd(rs + RL.tot(), (unsigned long long)total);
    if (total_e) atomicAdd(rs + RL.tot() + 1, (unsigned long long)total_e);
    long long* rm = (long long*)ev.red_max + u * RAILS_RED_MAX_LEN;
    atomicMax(rm + RMAX_S, mx);
    atomicMax(rm + RMAX_SE, mxe);
    atomicMax(rm + RMAX_ROW, total);
    atomicMax(rm + RMAX_SU, mxu);
  }
}

__global__ void __launch_bounds__(256)
    k_eval_finalize(int M, int N, double R2, const int64_t* __restrict__ red_sum,
                    const int64_t* __restrict__ red_max, rails_final_t out) {
  const long long u = blockIdx.x;
  block_finalize_unit<false>(u, M, N, R2, red_sum + u * RAILS_RED_SUM_LEN(M, N),
                             red_max + u * RAILS_RED_MAX_LEN, out);
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

// Per-rank pointers of the ranks a launch plays: one entry in the normal
// one-process-per-rank launch; `world` entries when one process drives every rank
// (rails_eval_finalize_peer_local: CTA (u, p) plays rank p).
struct PeerRanks {
  int64_t* red_sum[RAILS_PEER_MAX];
  int64_t* red_max[RAILS_PEER_MAX];
  rails_final_t out[RAILS_PEER_MAX];
};

// One CTA per (unit, played rank): push this rank's partials to every rank, release
// a flag per (unit, rank), acquire every rank's flag, reduce the world's partials (in
// rank order, so every rank computes identical sums) and finalize the unit.  Slots
// are double-buffered by call parity and flags are waited on as ">= gen": a fast
// rank may push call gen+1 (other half) and bump its flag while a slow rank is still
// reading call gen, and it cannot get two calls ahead (call gen+1 waits for the slow
// rank's gen+1 flag).
__global__ void __launch_bounds__(256)
    k_finalize_peer(int M, int N, double R2, long long rsl, int U, PeerRanks pr, PeerBufs pb,
                    int rank0, int world, uint32_t gen, int* err) {
  const long long u = blockIdx.x;
  const int rank = rank0 + (int)blockIdx.y;
  const long long rec = rsl + RAILS_RED_MAX_LEN;
  const size_t slots_off = al256e((size_t)U * world * 4) +
                           (size_t)(gen & 1u) * world * U * rec * 8;
  int64_t* rs = pr.red_sum[blockIdx.y] + u * rsl;
  int64_t* rmx = pr.red_max[blockIdx.y] + u * RAILS_RED_MAX_LEN;
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
  // 3. reduce in rank order (volatile loads: the data came from other GPUs), as an
  // all-reduce would leave it, then finalize the unit
  const volatile int64_t* slots = (const volatile int64_t*)(pb.p[rank] + slots_off);
  for (long long i = threadIdx.x; i < rsl; i += blockDim.x) {
    long long v = 0;
    for (int p = 0; p < world; ++p) v += slots[((long long)p * U + u) * rec + i];
    rs[i] = v;
  }
  if (threadIdx.x < RAILS_RED_MAX_LEN) {
    long long v = 0;
    for (int p = 0; p < world; ++p)
      v = max(v, (long long)slots[((long long)p * U + u) * rec + rsl + threadIdx.x]);
    rmx[threadIdx.x] = v;
  }
  __syncthreads();
  block_finalize_unit<false>(u, M, N, R2, rs, rmx, pr.out[blockIdx.y]);
}

// nplay = 1: this process is rank peer.rank (ordinary launch).  nplay = world: one
// process plays every rank (cooperative launch, so all CTAs are co-resident and the
// flag waits between them cannot deadlock).
cudaError_t launch_finalize_peer(const LaunchCtx& c, int U, int M, int N, double R2,
                                 int64_t* const* red_sum, int64_t* const* red_max,
                                 const rails_peer_t& peer, const rails_final_t* f, int nplay) {
  PeerBufs pb;
  for (int p = 0; p < RAILS_PEER_MAX; ++p) pb.p[p] = (uint8_t*)(p < peer.world ? peer.buf[p] : nullptr);
  PeerRanks pr{};
  for (int i = 0; i < nplay; ++i) {
    pr.red_sum[i] = red_sum[i];
    pr.red_max[i] = red_max[i];
    pr.out[i] = f[i];
  }
  int M_ = M, N_ = N, U_ = U, world = peer.world;
  int rank0 = nplay == 1 ? peer.rank : 0;
  uint32_t gen = peer.gen;
  double R2_ = R2;
  long long rsl = RAILS_RED_SUM_LEN(M, N);
  int* err = c.err;
  count_launch(1);
  if (nplay == 1) {
    k_finalize_peer<<<dim3((unsigned)U, 1), 256, 0, c.stream>>>(M, N, R2, rsl, U, pr, pb, rank0,
                                                                world, gen, err);
    return cudaGetLastError();
  }
  void* args[] = {&M_, &N_, &R2_, &rsl, &U_, &pr, &pb, &rank0, &world, &gen, &err};
  return cudaLaunchCooperativeKernel((const void*)k_finalize_peer, dim3((unsigned)U, nplay),
                                     dim3(256), args, 0, c.stream);
}

static int pow2_shift(long long C) {
  if (C <= 0 || (C & (C - 1))) return -1;
  int s = 0;
  while ((1LL << s) < C) ++s;
  return s;
}

__global__ void __launch_bounds__(1024)
    k_rail_offsets(long long n, const int64_t* __restrict__ send_load,
                   int64_t* __restrict__ rail_base, int64_t* __restrict__ total) {
  block_rail_offsets<false>(n, send_load, rail_base, total);
}

cudaError_t launch_eval(const LaunchCtx& c, int U, int nd, int d0, int M, int N, long long C,
                        uint64_t seed, const int64_t* msg, const rails_sched_t& s,
                        const rails_eval_t& e, const int32_t* ex_inv, const uint64_t* ex_res) {
  const long long rsl = RAILS_RED_SUM_LEN(M, N);
  cudaError_t err =
      cudaMemsetAsync(e.red_sum, 0, (size_t)U * rsl * sizeof(int64_t), c.stream);
  if (err != cudaSuccess) return err;
  err = cudaMemsetAsync(e.red_max, 0, (size_t)U * RAILS_RED_MAX_LEN * sizeof(int64_t), c.stream);
  if (err != cudaSuccess) return err;
  const int FT = (EV2_THREADS / N) < 64 ? (EV2_THREADS / N) : 64;
  const size_t smem = 16 + (size_t)N * (FT + 1) * (8 + 4);
  const bool narrow = (long long)M * N < EV2_THREADS;
  auto kern = N == 8 ? (narrow ? k_eval_node<8, 6> : k_eval_node<8>) : k_eval_node<0>;
  err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  kern<<<(unsigned)((long long)U * nd), EV2_THREADS, smem, c.stream>>>(
      M, N, nd, d0, C, pow2_shift(C), seed, FT, msg, s.full_base, s.rem_rail, s.n_full, e,
      ex_inv, ex_res, ex_inv ? s.rem_rail : nullptr, ex_inv ? s.rem_off : nullptr);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const LaunchCtx& c, int U, int M, int N, double R2,
                            const int64_t* red_sum, const int64_t* red_max,
                            const rails_final_t& f) {
  k_eval_finalize<<<(unsigned)U, 256, 0, c.stream>>>(M, N, R2, red_sum, red_max, f);
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
