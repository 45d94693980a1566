// k_owner.cu -- NEXT f2: rail-owner pack fused with the intra-node NVLink hop.
//
// One multi-GPU box is one RailS node: NIC j hangs off GPU j ("GPU (d,n) is
// connected to a dedicated NIC_{d,n}"), so rail j's send buffer must sit in GPU
// j's HBM, and traffic of GPU g sprayed onto rail j != g first crosses the
// intra-domain network (R1 > R2).  Here each GPU packs the
// rows of its own source GPUs and writes every chunk piece straight into the rail
// owner's buffer through peer (NVLink / NVSwitch) pointers -- the intra-node
// all-to-all happens inside the pack kernel, tile by tile, with no staging copy
// and no separate collective.  The node-wide LPT schedule (identical on every
// GPU) decides rail and offset exactly as in k_pack.
#include <cstdlib>

#include "common.cuh"

namespace rails {

constexpr int OWN_THREADS = 256;

struct RailPtrs {
  uint8_t* p[32];      // rail j buffer (peer-mapped), j < N
  long long cap[32];   // its capacity in bytes
};

struct OwnerLoc {
  int rail;
  long long off;  // byte offset inside the rail's buffer
};

__device__ __forceinline__ OwnerLoc chunk_loc(long long c, long long fb, long long nfull, int rr,
                                              long long ro, int N, long long C,
                                              const int64_t* __restrict__ rbase) {
  if (c < nfull) {
    const long long i = fb + c;
    const long long q = i / N;
    const int j = (int)(i - q * N);
    return {j, rbase[j] + q * C};
  }
  return {rr, rr >= 0 ? rbase[rr] + ro : -(1LL << 62)};
}

template <int VPL, bool MULTI>
__global__ void __launch_bounds__(OWN_THREADS)
    k_pack_owner(int U, int nd, int d0, int M, int N, int g0, int ng, int T, int k, long long C,
                 int cshift, const uint4* __restrict__ x, const int32_t* __restrict__ topk,
                 const int32_t* __restrict__ lut, int n_inst, const int32_t* __restrict__ rank,
                 const int64_t* __restrict__ msg, long long RB,
                 const int64_t* __restrict__ full_base, const int8_t* __restrict__ rem_rail,
                 const int64_t* __restrict__ rem_off, const int64_t* __restrict__ rail_base,
                 RailPtrs rp, int* err) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (OWN_THREADS / 32);
  const long long rows = (long long)U * nd * ng * T;
  const long long G = (long long)M * N;
  const int nvec = (int)(RB >> 4);
  const ChunkDiv cd{C, cshift};

  for (long long row = (long long)blockIdx.x * (OWN_THREADS / 32) + (threadIdx.x >> 5);
       row < rows; row += nwarps) {
    const long long ugl = row / T;  // (u*nd + dl)*ng + gl
    const long long ul = ugl / ng;
    const int g = g0 + (int)(ugl - ul * ng);
    const int d = d0 + (int)(ul % nd);
    const long long ug = ul * N + g;  // node-wide message row
    const uint4* __restrict__ src = x + row * nvec;
    const int64_t* __restrict__ rbase = rail_base + ul * N;

    uint4 v[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int vi = i * 32 + lane;
      if (vi < nvec) v[i] = ld_stream(src + vi);
    }

    // slot metadata on lanes 0..k-1: (rail, offset) of the first two pieces
    long long p0 = 0, fb = 0, nfull = 0, ro = 0, off0 = 0, off1 = 0;
    int b0 = 0, rr = -1, ok = 0, j0 = 0, j1 = 0;
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
        p0 = (long long)rk * RB;
        if (rk < 0 || p0 + RB > B) {
          flag_error(err, ERR_RANGE);
        } else {
          fb = full_base[mi];
          nfull = cd.div(B);
          rr = rem_rail[mi];
          ro = rem_off[mi];
          const long long c0 = cd.div(p0);
          const OwnerLoc l0 = chunk_loc(c0, fb, nfull, rr, ro, N, C, rbase);
          j0 = l0.rail;
          off0 = l0.off + (p0 - c0 * C);
          const long long bb = (c0 + 1) * C - p0;
          b0 = (int)(bb < RB ? bb : RB);
          if (!MULTI && b0 < RB) {
            const OwnerLoc l1 = chunk_loc(c0 + 1, fb, nfull, rr, ro, N, C, rbase);
            j1 = l1.rail;
            off1 = l1.off;
          }
          ok = (j0 >= 0 && j0 < N && j1 >= 0 && j1 < N);
          if (!ok) flag_error(err, ERR_RANGE);
        }
      }
    }

    for (int w0 = 0; w0 < nvec; w0 += VPL * 32) {
      if (w0 > 0) {
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int vi = w0 + i * 32 + lane;
          if (vi < nvec) v[i] = ld_stream(src + vi);
        }
      }
      for (int s = 0; s < k; ++s) {
        if (!__shfl_sync(FULL, ok, s)) continue;
        const int J0 = __shfl_sync(FULL, j0, s);
        const long long O0 = __shfl_sync(FULL, off0, s);
        const int B0 = __shfl_sync(FULL, b0, s);
        if (!MULTI) {
          const int J1 = __shfl_sync(FULL, j1, s);
          const long long O1 = __shfl_sync(FULL, off1, s);
          uint8_t* const P0 = rp.p[J0];
          uint8_t* const P1 = rp.p[J1];
          const long long cap0 = rp.cap[J0], cap1 = rp.cap[J1];
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            const int vi = w0 + i * 32 + lane;
            if (vi < nvec) {
              const long long o = (long long)vi << 4;
              const bool first = o < B0;
              const long long a = first ? O0 + o : O1 + (o - B0);
              const long long cap = first ? cap0 : cap1;
              if (a >= 0 && a + 16 <= cap)
                st_stream((uint4*)((first ? P0 : P1) + a), v[i]);
              else
                flag_error(err, ERR_NOSPC);
            }
          }
        } else {
          const long long P0v = __shfl_sync(FULL, p0, s);
          const long long FB = __shfl_sync(FULL, fb, s);
          const long long NF = __shfl_sync(FULL, nfull, s);
          const long long RO = __shfl_sync(FULL, ro, s);
          const int RR = __shfl_sync(FULL, rr, s);
#pragma unroll
          for (int i = 0; i < VPL; ++i) {
            const int vi = w0 + i * 32 + lane;
            if (vi < nvec) {
              const long long o = (long long)vi << 4;
              int j;
              long long a;
              if (o < B0) {
                j = J0;
                a = O0 + o;
              } else {
                const long long p = P0v + o;
                const long long c = cd.div(p);
                const OwnerLoc l = chunk_loc(c, FB, NF, RR, RO, N, C, rbase);
                j = l.rail;
                a = l.off + (p - c * C);
              }
              if (j >= 0 && j < N && a >= 0 && a + 16 <= rp.cap[j])
                st_stream((uint4*)(rp.p[j] + a), v[i]);
              else
                flag_error(err, ERR_NOSPC);
            }
          }
        }
      }
    }
  }
  // this thread's stores into peers' HBM are performed system-wide before it
  // exits, so a later rails_peer_barrier orders them for every rank
  __threadfence_system();
}

// Per-rail placement inside the owner buffers: rail_base[u][dl][j] = bytes of rail j
// from the (u', dl') blocks before (u, dl); rail_total[j] = rail j's buffer size.
__global__ void k_rail_offsets_owner(long long ublk, int N, const int64_t* __restrict__ send_load,
                                     int64_t* __restrict__ rail_base,
                                     int64_t* __restrict__ rail_total) {
  const int j = threadIdx.x;
  if (j >= N) return;
  long long run = 0;
  for (long long b = 0; b < ublk; ++b) {
    rail_base[b * N + j] = run;
    run += send_load[b * N + j];
  }
  rail_total[j] = run;
}

template <int VPL, bool MULTI>
static cudaError_t launch_ov(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int g0,
                             int ng, int T, int k, long long C, int cshift, const void* x,
                             const int32_t* topk, const int32_t* lut, int n_inst,
                             const int32_t* rank, const int64_t* msg, long long RB,
                             const rails_sched_t& s, const int64_t* rail_base,
                             const RailPtrs& rp) {
  auto kern = k_pack_owner<VPL, MULTI>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, OWN_THREADS, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long rows = (long long)U * nd * ng * T;
  const long long need = (rows + OWN_THREADS / 32 - 1) / (OWN_THREADS / 32);
  const long long grid = wave_grid(c.num_sms, per_sm, need, 8);
  kern<<<(unsigned)grid, OWN_THREADS, 0, c.stream>>>(
      U, nd, d0, M, N, g0, ng, T, k, C, cshift, (const uint4*)x, topk, lut, n_inst, rank, msg,
      RB, s.full_base, s.rem_rail, s.rem_off, rail_base, rp, c.err);
  count_launch(1);
  return cudaGetLastError();
}

template <bool MULTI>
static cudaError_t launch_om(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int g0,
                             int ng, int T, int k, long long C, int cshift, const void* x,
                             const int32_t* topk, const int32_t* lut, int n_inst,
                             const int32_t* rank, const int64_t* msg, long long RB,
                             const rails_sched_t& s, const int64_t* rail_base,
                             const RailPtrs& rp) {
  const long long vpl = ((RB >> 4) + 31) / 32;
#define RAILS_OWN_CASE(V)                                                                  \
  if (vpl <= V)                                                                            \
    return launch_ov<V, MULTI>(c, U, nd, d0, M, N, g0, ng, T, k, C, cshift, x, topk, lut,  \
                               n_inst, rank, msg, RB, s, rail_base, rp);
  RAILS_OWN_CASE(4)
#undef RAILS_OWN_CASE
  // rows over 8 KiB in 8 KiB windows, as k_pack (more resident warps)
  return launch_ov<16, MULTI>(c, U, nd, d0, M, N, g0, ng, T, k, C, cshift, x, topk, lut, n_inst,
                              rank, msg, RB, s, rail_base, rp);
}

cudaError_t launch_pack_owner(const LaunchCtx& c, int U, int nd, int d0, int M, int N, int g0,
                              int ng, int T, int k, long long C, const void* x,
                              const int32_t* topk, const int32_t* lut, int n_inst,
                              const int32_t* rank, const int64_t* msg, long long row_bytes,
                              const rails_sched_t& s, const int64_t* rail_base,
                              void* const* rail_ptr, const int64_t* rail_cap) {
  RailPtrs rp{};
  for (int j = 0; j < N; ++j) {
    rp.p[j] = (uint8_t*)rail_ptr[j];
    rp.cap[j] = rail_cap[j];
  }
  int cshift = -1;
  if ((C & (C - 1)) == 0) {
    cshift = 0;
    while ((1LL << cshift) < C) ++cshift;
  }
  if (C >= row_bytes)
    return launch_om<false>(c, U, nd, d0, M, N, g0, ng, T, k, C, cshift, x, topk, lut, n_inst,
                            rank, msg, row_bytes, s, rail_base, rp);
  return launch_om<true>(c, U, nd, d0, M, N, g0, ng, T, k, C, cshift, x, topk, lut, n_inst, rank,
                         msg, row_bytes, s, rail_base, rp);
}

cudaError_t launch_rail_offsets_owner(const LaunchCtx& c, long long ublk, int N,
                                      const int64_t* send_load, int64_t* rail_base,
                                      int64_t* rail_total) {
  k_rail_offsets_owner<<<1, 32, 0, c.stream>>>(ublk, N, send_load, rail_base, rail_total);
  count_launch(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- peer exchange
// Exchange buffer of a rail-owner rank (rails_owner_exchange_layout):
//   [barrier flags: RAILS_PEER_MAX x u32, 256 B][gather flags: U x world x u32,
//    256-aligned][msg_node: int64 [U][1][N][G]]
struct PeerBase {
  uint8_t* p[RAILS_PEER_MAX];
};

static inline size_t al256o(size_t x) { return (x + 255) & ~(size_t)255; }

void owner_exchange_layout(int U, int world, long long N, long long G, size_t* bytes,
                           size_t* gflag_off, size_t* msg_off) {
  *gflag_off = 256;
  *msg_off = 256 + al256o((size_t)U * world * 4);
  *bytes = *msg_off + (size_t)U * N * G * 8;
}

// One CTA per (unit, played rank p): rank p's message rows (source GPUs g0[p] ..
// g0[p]+ng-1) go into every rank's msg_node (NVLink stores), then a per-(unit,
// rank) flag; the CTA returns when every rank's rows of the unit have arrived at
// rank p.  One played rank in the one-process-per-rank launch; every rank in the
// cooperative single-process launch (rails_gather_rows_peer_local).
struct RowSrc {
  const int64_t* msg_loc[RAILS_PEER_MAX];
  int g0[RAILS_PEER_MAX];
};

__global__ void __launch_bounds__(256)
    k_gather_rows_peer(int U, int N, long long G, int ng, RowSrc rsrc, PeerBase pb, int rank0,
                       int world, uint32_t gen, size_t gflag_off, size_t msg_off, int* err) {
  const long long u = blockIdx.x;
  const int rank = rank0 + (int)blockIdx.y;
  const int g0 = rsrc.g0[blockIdx.y];
  const long long n = (long long)ng * G;  // int64 per unit and rank
  const int64_t* src = rsrc.msg_loc[blockIdx.y] + u * n;
  for (int p = 0; p < world; ++p) {
    int64_t* dst = (int64_t*)(pb.p[p] + msg_off) + (u * N + g0) * G;
    if (((uintptr_t)dst & 15) == 0 && ((uintptr_t)src & 15) == 0) {
      for (long long i = threadIdx.x; i < n / 2; i += blockDim.x)
        ((int4*)dst)[i] = ((const int4*)src)[i];
      if ((n & 1) && threadIdx.x == 0) dst[n - 1] = src[n - 1];
    } else {
      for (long long i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p)
      st_release_sys((uint32_t*)(pb.p[p] + gflag_off) + u * world + rank, gen);
  }
  if (threadIdx.x < world)
    wait_flag_ge((const uint32_t*)(pb.p[rank] + gflag_off) + u * world + threadIdx.x, gen, err);
  __syncthreads();
}

// Every rank's earlier stream work (its stores included) precedes every rank's
// later work: flag all ranks, wait for all ranks' flags (one warp per played rank).
__global__ void k_peer_barrier(PeerBase pb, int rank0, int world, uint32_t gen, int* err) {
  const int rank = rank0 + (int)blockIdx.y;
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p) st_release_sys((uint32_t*)pb.p[p] + rank, gen);
  }
  __syncwarp();
  if (threadIdx.x < world) wait_flag_ge((const uint32_t*)pb.p[rank] + threadIdx.x, gen, err);
  __syncwarp();
}

static PeerBase peer_base(const rails_peer_t& peer) {
  PeerBase pb;
  for (int p = 0; p < RAILS_PEER_MAX; ++p)
    pb.p[p] = (uint8_t*)(p < peer.world ? peer.buf[p] : nullptr);
  return pb;
}

cudaError_t launch_gather_rows_peer(const LaunchCtx& c, int U, int N, long long G, int ng,
                                    const int64_t* const* msg_loc, const int* g0,
                                    const rails_peer_t& peer, int nplay) {
  size_t bytes, gf, mo;
  owner_exchange_layout(U, peer.world, N, G, &bytes, &gf, &mo);
  RowSrc rs{};
  for (int i = 0; i < nplay; ++i) {
    rs.msg_loc[i] = msg_loc[i];
    rs.g0[i] = g0[i];
  }
  PeerBase pb = peer_base(peer);
  int U_ = U, N_ = N, ng_ = ng, world = peer.world, rank0 = nplay == 1 ? peer.rank : 0;
  long long G_ = G;
  uint32_t gen = peer.gen;
  int* err = c.err;
  count_launch(1);
  if (nplay == 1) {
    k_gather_rows_peer<<<dim3((unsigned)U, 1), 256, 0, c.stream>>>(U, N, G, ng, rs, pb, rank0,
                                                                   world, gen, gf, mo, err);
    return cudaGetLastError();
  }
  void* args[] = {&U_, &N_, &G_, &ng_, &rs, &pb, &rank0, &world, &gen, &gf, &mo, &err};
  return cudaLaunchCooperativeKernel((const void*)k_gather_rows_peer, dim3((unsigned)U, nplay),
                                     dim3(256), args, 0, c.stream);
}

cudaError_t launch_peer_barrier(const LaunchCtx& c, const rails_peer_t& peer, int nplay) {
  PeerBase pb = peer_base(peer);
  int rank0 = nplay == 1 ? peer.rank : 0, world = peer.world;
  uint32_t gen = peer.gen;
  int* err = c.err;
  count_launch(1);
  if (nplay == 1) {
    k_peer_barrier<<<dim3(1, 1), 32, 0, c.stream>>>(pb, rank0, world, gen, err);
    return cudaGetLastError();
  }
  void* args[] = {&pb, &rank0, &world, &gen, &err};
  return cudaLaunchCooperativeKernel((const void*)k_peer_barrier, dim3(1, nplay), dim3(32), args,
                                     0, c.stream);
}

}  // namespace rails
