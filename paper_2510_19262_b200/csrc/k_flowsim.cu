// k_flowsim.cu -- NEXT f4: batched fluid (flow-level) simulation of one all-to-all
// round per simulation, on the GPU (sm_100a).
//
// What is simulated (R#35-R#39; SPEC
// flowsim S:464-537): the Rail fabric's directed links (GPU<->NIC intra links,
// NIC<->leaf rail links, leaf<->spine links), the flows a policy makes of the
// round's messages (LPT chunks on rail paths; the continuous P* = 1/N split; ECMP
// and REPS whole messages on spine paths; MinRTT chunks on the least backlogged
// spine path), max-min fair rates by progressive filling, and completion events.
//
// B200 design: one CTA per simulation, so a batch of (unit, policy) simulations
// fills the SMs; every step of a simulation -- flow construction, MinRTT route
// choice, the link->subflow index, the whole event loop and the CCT statistics --
// runs on the device with no host round trip.  The event loop keeps link state in
// shared memory and updates it incrementally with integer weight sums and
// claim-based freezing (bitmaps), so a run is deterministic.  Floating point: IEEE
// binary64, no FMA contraction on the paths that feed discrete decisions
// (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn).
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "radix.cuh"

namespace rails {

constexpr int FS_THREADS = 1024;
constexpr int FS_MAXL = 4;  // links per subflow path
constexpr int FS_NSTATS = 10;

struct FsTopo {
  int M, N, S, L;
  long long G, Q;  // G = M*N GPUs, Q = M*N*G messages
  double R1, R2, Rs;
  long long C;
  uint64_t seed;
};

// ---------------------------------------------------------------- links (R#35)
__device__ __forceinline__ int l_gpu_up(const FsTopo& t, int k, int g, int n) {
  return (k * t.N + g) * t.N + n;
}
__device__ __forceinline__ int l_nic_up(const FsTopo& t, int k, int n) {
  return t.M * t.N * t.N + k * t.N + n;
}
__device__ __forceinline__ int l_leaf_spine(const FsTopo& t, int n, int j) {
  return t.M * t.N * t.N + t.M * t.N + n * t.S + j;
}
__device__ __forceinline__ int l_spine_leaf(const FsTopo& t, int j, int m) {
  return t.M * t.N * t.N + t.M * t.N + t.N * t.S + j * t.N + m;
}
__device__ __forceinline__ int l_nic_down(const FsTopo& t, int f, int m) {
  return t.M * t.N * t.N + t.M * t.N + 2 * t.N * t.S + f * t.N + m;
}
__device__ __forceinline__ int l_gpu_down(const FsTopo& t, int f, int n, int m) {
  return t.M * t.N * t.N + 2 * t.M * t.N + 2 * t.N * t.S + (f * t.N + n) * t.N + m;
}
__device__ __forceinline__ double l_cap(const FsTopo& t, int l) {
  const int a = t.M * t.N * t.N, b = t.M * t.N, c = t.N * t.S;
  if (l < a) return t.R1;
  if (l < a + b) return t.R2;
  if (l < a + b + 2 * c) return t.Rs;
  if (l < a + 2 * b + 2 * c) return t.R2;
  return t.R1;
}
// rail path of rail n: [GPU_UP] NIC_UP NIC_DOWN [GPU_DOWN]
__device__ __forceinline__ int rail_path(const FsTopo& t, int k, int g, int f, int m, int n,
                                         int* p) {
  int c = 0;
  if (g != n) p[c++] = l_gpu_up(t, k, g, n);
  p[c++] = l_nic_up(t, k, n);
  p[c++] = l_nic_down(t, f, n);
  if (m != n) p[c++] = l_gpu_down(t, f, n, m);
  return c;
}
// spine path from NIC g to NIC m through spine j (direct leaf path when g == m)
__device__ __forceinline__ int spine_path(const FsTopo& t, int k, int g, int f, int m, int j,
                                          int* p) {
  if (g == m) return rail_path(t, k, g, f, m, g, p);
  p[0] = l_nic_up(t, k, g);
  p[1] = l_leaf_spine(t, g, j);
  p[2] = l_spine_leaf(t, j, m);
  p[3] = l_nic_down(t, f, m);
  return 4;
}

// ---------------------------------------------------------------- workspace
// Per simulation, `stride` bytes holding (each array 256-byte aligned):
struct FsWs {
  long long* foff;   // [Q+1] first flow of each message
  long long* soff;   // [Q+1] first subflow of each message
  double* fbytes;    // [capF]
  int* fmsg;         // [capF] message index
  int* fsub0;        // [capF+1]
  double* sw;        // [capS] share-weight
  int* snl;          // [capS] links on the path (0 until MinRTT routes it)
  int* slink;        // [capS][4]
  uint32_t* kA;      // [4 capS] CSR sort keys / values
  uint32_t* kB;
  uint32_t* iA;
  uint32_t* iB;
  int* loff;         // [L+1]
  int* lsub;         // [4 capS] subflows per link, ascending
  double* rem;       // [capF]
  double* frate;     // [capF]
  double* done;      // [capF] completion time
  uint8_t* fact;     // [capF] flow active
  double* rate;      // [capS]
  int* swi;          // [capS] share-weight in units of 1/S
  uint8_t* sact;     // [capS] subflow active
  int* fep;          // [capS] event at which the subflow was last frozen
  uint64_t* cA;      // [Q] CCT sort keys
  uint64_t* cB;
  uint32_t* ciA;     // [Q]
  uint32_t* ciB;
  double* simstat;   // [4] max pair fraction, events, flows, subflows
  unsigned long long* pair;  // [M*M] per-event domain-pair rate, fixed point
  uint8_t* sinit;    // [capS] active at t = 0 (PLB's spare spine paths are not)
  uint8_t* shit;     // [capS] frozen by a spine-layer bottleneck (PLB signal)
  int* fcur;         // [capF] PLB: the flow's active subflow
  int* fatt;         // [capF] PLB: re-hash attempts
  int* flast;        // [capF] PLB: event of the last re-hash
  // o[33]: link state of k_fs_sim<true> (L * 40 bytes)
};

static inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct FsLayout {
  size_t o[40];
  size_t stride;
};

static FsLayout fs_layout(long long Q, int L, long long capF, long long capS) {
  const size_t sz[] = {
      (size_t)(Q + 1) * 8, (size_t)(Q + 1) * 8, (size_t)capF * 8, (size_t)capF * 4,
      (size_t)(capF + 1) * 4, (size_t)capS * 8, (size_t)capS * 4, (size_t)capS * 16,
      (size_t)capS * 16, (size_t)capS * 16, (size_t)capS * 16, (size_t)capS * 16,
      (size_t)(L + 1) * 4, (size_t)capS * 16, (size_t)capF * 8, (size_t)capF * 8,
      (size_t)capF * 8, (size_t)capF, (size_t)capS * 8, (size_t)capS * 4, (size_t)capS,
      (size_t)capS * 4, (size_t)Q * 8, (size_t)Q * 8, (size_t)Q * 4, (size_t)Q * 4, 64, (size_t)Q * 8, (size_t)capS, (size_t)capS,
      (size_t)capF * 4, (size_t)capF * 4, (size_t)capF * 4,
      (size_t)L * 41 + 2 * (size_t)((capS + 31) / 32) * 4 + 64};
  FsLayout lo;
  size_t off = 0;
  const int n = (int)(sizeof(sz) / sizeof(sz[0]));
  for (int i = 0; i < n; ++i) {
    lo.o[i] = off;
    off += al256(sz[i] + 16);
  }
  lo.stride = off;
  return lo;
}

__device__ __forceinline__ FsWs fs_ws(uint8_t* base, const size_t* o) {
  FsWs w;
  w.foff = (long long*)(base + o[0]);
  w.soff = (long long*)(base + o[1]);
  w.fbytes = (double*)(base + o[2]);
  w.fmsg = (int*)(base + o[3]);
  w.fsub0 = (int*)(base + o[4]);
  w.sw = (double*)(base + o[5]);
  w.snl = (int*)(base + o[6]);
  w.slink = (int*)(base + o[7]);
  w.kA = (uint32_t*)(base + o[8]);
  w.kB = (uint32_t*)(base + o[9]);
  w.iA = (uint32_t*)(base + o[10]);
  w.iB = (uint32_t*)(base + o[11]);
  w.loff = (int*)(base + o[12]);
  w.lsub = (int*)(base + o[13]);
  w.rem = (double*)(base + o[14]);
  w.frate = (double*)(base + o[15]);
  w.done = (double*)(base + o[16]);
  w.fact = base + o[17];
  w.rate = (double*)(base + o[18]);
  w.swi = (int*)(base + o[19]);
  w.sact = base + o[20];
  w.fep = (int*)(base + o[21]);
  w.cA = (uint64_t*)(base + o[22]);
  w.cB = (uint64_t*)(base + o[23]);
  w.ciA = (uint32_t*)(base + o[24]);
  w.ciB = (uint32_t*)(base + o[25]);
  w.simstat = (double*)(base + o[26]);
  w.pair = (unsigned long long*)(base + o[27]);
  w.sinit = base + o[28];
  w.shit = base + o[29];
  w.fcur = (int*)(base + o[30]);
  w.fatt = (int*)(base + o[31]);
  w.flast = (int*)(base + o[32]);
  return w;
}

struct FsOffsets {
  size_t o[40];
};

__device__ __forceinline__ double fs_inf() { return __longlong_as_double(0x7ff0000000000000LL); }

// ---------------------------------------------------------------- block helpers
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
// block reductions: scratch >= 32 doubles; result broadcast to every thread
__device__ double block_min_d(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_min_d(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = lane < nw ? scratch[lane] : fs_inf();
  r = warp_min_d(r);
  return r;
}
__device__ double block_max_d(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max_d(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = lane < nw ? scratch[lane] : -DBL_MAX;
  return warp_max_d(r);
}
__device__ double block_sum_d(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = lane < nw ? scratch[lane] : 0.0;
  return warp_sum_d(r);
}
__device__ long long block_sum_ll(long long v, long long* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  long long r = lane < nw ? scratch[lane] : 0;
  return warp_sum(r);
}

// ---------------------------------------------------------------- flow counts
// Flows and subflows each message becomes under the policy (R#36).
__device__ __forceinline__ void msg_counts(const FsTopo& t, int pol, long long q, long long B,
                                           long long& nf, long long& ns) {
  nf = ns = 0;
  if (B <= 0) return;
  const int g = (int)((q / t.G) % t.N), m = (int)((q % t.G) % t.N);
  switch (pol) {
    case RAILS_POL_LPT:
    case RAILS_POL_MINRTT:
      nf = ns = (B + t.C - 1) / t.C;
      break;
    case RAILS_POL_UNIFORM:
      nf = ns = t.N;
      break;
    case RAILS_POL_ECMP:
      nf = ns = 1;
      break;
    default:  // REPS, PLB
      nf = 1;
      ns = (g == m) ? 1 : t.S;
  }
}

// One CTA per simulation: exclusive scans of the per-message flow / subflow counts
// in message order; plan mode writes only the totals.
__global__ void __launch_bounds__(FS_THREADS)
    k_fs_count(FsTopo t, const int32_t* __restrict__ policy, const int64_t* __restrict__ msg,
               uint8_t* ws, FsOffsets lo, size_t stride, int64_t* __restrict__ totals,
               int plan, int* err) {
  __shared__ long long scr[33];
  const long long sim = blockIdx.x;
  const int pol = policy[sim];
  const int64_t* __restrict__ ms = msg + sim * t.Q;
  FsWs w = fs_ws(ws + sim * stride, lo.o);
  long long cf = 0, cs = 0;
  if (pol < RAILS_POL_LPT || pol > RAILS_POL_PLB) {  // unknown policy: no flows
    if (threadIdx.x == 0) {
      flag_error(err, ERR_RANGE);
      if (plan) totals[2 * sim] = totals[2 * sim + 1] = 0;
    }
    if (!plan)
      for (long long q = threadIdx.x; q <= t.Q; q += FS_THREADS) w.foff[q] = w.soff[q] = 0;
    return;
  }
  for (long long q0 = 0; q0 < t.Q; q0 += FS_THREADS) {
    const long long q = q0 + threadIdx.x;
    long long nf = 0, ns = 0;
    if (q < t.Q) msg_counts(t, pol, q, ms[q], nf, ns);
    long long tf, ts;
    const long long ef = block_excl_scan(nf, scr, &tf);
    const long long es = block_excl_scan(ns, scr, &ts);
    if (!plan && q < t.Q) {
      w.foff[q] = cf + ef;
      w.soff[q] = cs + es;
    }
    cf += tf;
    cs += ts;
  }
  if (threadIdx.x == 0) {
    if (plan) {
      totals[2 * sim] = cf;
      totals[2 * sim + 1] = cs;
    } else {
      w.foff[t.Q] = cf;
      w.soff[t.Q] = cs;
    }
  }
}

// ---------------------------------------------------------------- flow build
__global__ void __launch_bounds__(FS_THREADS)
    k_fs_build(FsTopo t, const int32_t* __restrict__ policy, const int64_t* __restrict__ msg,
               const int64_t* __restrict__ full_base, const int8_t* __restrict__ rem_rail,
               uint8_t* ws, FsOffsets lo, size_t stride, long long capF, long long capS,
               int* err) {
  const long long sim = blockIdx.x;
  const int pol = policy[sim];
  const int64_t* __restrict__ ms = msg + sim * t.Q;
  FsWs w = fs_ws(ws + sim * stride, lo.o);
  const long long nflow = w.foff[t.Q], nsub = w.soff[t.Q];
  if (nflow > capF || nsub > capS) {
    if (threadIdx.x == 0) flag_error(err, ERR_NOSPC);
    return;
  }
  for (long long q = threadIdx.x; q < t.Q; q += FS_THREADS) {
    const long long B = ms[q];
    if (B <= 0) continue;
    const int d = (int)(q / (t.N * t.G)), g = (int)((q / t.G) % t.N);
    const int h = (int)(q % t.G), f = h / t.N, m = h % t.N;
    const long long fo = w.foff[q], so = w.soff[q];
    if (pol == RAILS_POL_LPT || pol == RAILS_POL_MINRTT) {
      const long long nfull = B / t.C, nch = (B + t.C - 1) / t.C;
      const long long fb = full_base ? full_base[sim * t.Q + q] : 0;
      for (long long c = 0; c < nch; ++c) {
        const long long i = fo + c, s = so + c;
        w.fbytes[i] = (double)(c < nfull ? t.C : B - nfull * t.C);
        w.fmsg[i] = (int)q;
        w.fsub0[i] = (int)s;
        w.sw[s] = 1.0;
        w.swi[s] = t.S;
        w.sinit[s] = 1;
        if (pol == RAILS_POL_LPT) {
          const int rail = c < nfull ? (int)((fb + c) % t.N) : (int)rem_rail[sim * t.Q + q];
          w.snl[s] = rail_path(t, d, g, f, m, rail, w.slink + s * FS_MAXL);
        } else {
          w.snl[s] = 0;  // routed by k_fs_minrtt
        }
      }
    } else if (pol == RAILS_POL_UNIFORM) {
      for (int n = 0; n < t.N; ++n) {
        w.fbytes[fo + n] = __ddiv_rn((double)B, (double)t.N);
        w.fmsg[fo + n] = (int)q;
        w.fsub0[fo + n] = (int)(so + n);
        w.sw[so + n] = 1.0;
        w.swi[so + n] = t.S;
        w.sinit[so + n] = 1;
        w.snl[so + n] = rail_path(t, d, g, f, m, n, w.slink + (so + n) * FS_MAXL);
      }
    } else if (pol == RAILS_POL_ECMP) {
      const int j = ecmp_rail(t.seed, (long long)d * t.N + g, h, t.S);
      w.fbytes[fo] = (double)B;
      w.fmsg[fo] = (int)q;
      w.fsub0[fo] = (int)so;
      w.sw[so] = 1.0;
      w.swi[so] = t.S;
      w.sinit[so] = 1;
      w.snl[so] = spine_path(t, d, g, f, m, j, w.slink + so * FS_MAXL);
    } else if (pol == RAILS_POL_PLB) {
      // every spine path is a candidate subflow; the ECMP-hashed one starts
      const int nj = (g == m) ? 1 : t.S;
      const int j0 = ecmp_rail(t.seed, (long long)d * t.N + g, h, t.S);
      w.fbytes[fo] = (double)B;
      w.fmsg[fo] = (int)q;
      w.fsub0[fo] = (int)so;
      w.fcur[fo] = (int)so + (nj == 1 ? 0 : j0);
      w.fatt[fo] = 0;
      w.flast[fo] = -2;
      for (int j = 0; j < nj; ++j) {
        w.sw[so + j] = 1.0;
        w.swi[so + j] = t.S;
        w.sinit[so + j] = (uint8_t)(nj == 1 || j == j0);
        w.snl[so + j] = spine_path(t, d, g, f, m, j, w.slink + (so + j) * FS_MAXL);
      }
    } else {  // REPS
      const int nj = (g == m) ? 1 : t.S;
      w.fbytes[fo] = (double)B;
      w.fmsg[fo] = (int)q;
      w.fsub0[fo] = (int)so;
      for (int j = 0; j < nj; ++j) {
        w.sw[so + j] = __ddiv_rn(1.0, (double)nj);
        w.swi[so + j] = t.S / nj;
        w.sinit[so + j] = 1;
        w.snl[so + j] = spine_path(t, d, g, f, m, j, w.slink + (so + j) * FS_MAXL);
      }
    }
  }
  if (threadIdx.x == 0) w.fsub0[nflow] = (int)nsub;
}

// ---------------------------------------------------------------- MinRTT routes
// One warp per MinRTT simulation walks the chunks in (d, g, h, c) order; lane j
// scores spine j's path (max backlog / capacity over its links), the warp takes the
// lowest-scored lane (lowest j on ties), and the chosen links' backlog grows by the
// chunk's bytes.  Backlog lives in shared memory (L doubles).
__global__ void __launch_bounds__(32)
    k_fs_minrtt(FsTopo t, const int32_t* __restrict__ policy, uint8_t* ws, FsOffsets lo,
                size_t stride, long long capF, long long capS) {
  extern __shared__ double backlog[];
  const long long sim = blockIdx.x;
  if (policy[sim] != RAILS_POL_MINRTT) return;
  const int lane = threadIdx.x;
  FsWs w = fs_ws(ws + sim * stride, lo.o);
  if (w.foff[t.Q] > capF || w.soff[t.Q] > capS) return;
  for (int l = lane; l < t.L; l += 32) backlog[l] = 0.0;
  __syncwarp();
  const long long nflow = w.foff[t.Q];
  for (long long i0 = 0; i0 < nflow; i0 += 32) {
    const long long ii = i0 + lane;
    const int qv = ii < nflow ? w.fmsg[ii] : 0;
    const double bv = ii < nflow ? w.fbytes[ii] : 0.0;
    const int sv = ii < nflow ? w.fsub0[ii] : 0;
    const int cnt = (int)min(32LL, nflow - i0);
    for (int b = 0; b < cnt; ++b) {
      const long long q = __shfl_sync(FULL, qv, b);
      const double bytes = __shfl_sync(FULL, bv, b);
      const int s = __shfl_sync(FULL, sv, b);
      const int d = (int)(q / (t.N * t.G)), g = (int)((q / t.G) % t.N);
      const int h = (int)(q % t.G), f = h / t.N, m = h % t.N;
      const int nj = (g == m) ? 1 : t.S;
      double score = fs_inf();  // +inf for lanes without a candidate
      int p[FS_MAXL];
      int pn = 0;
      if (lane < nj) {
        pn = spine_path(t, d, g, f, m, lane, p);
        score = 0.0;
        for (int a = 0; a < pn; ++a) score = fmax(score, __ddiv_rn(backlog[p[a]], l_cap(t, p[a])));
      }
      double bs = score;
      int bj = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(FULL, bs, o);
        const int oj = __shfl_xor_sync(FULL, bj, o);
        if (os < bs || (os == bs && oj < bj)) {
          bs = os;
          bj = oj;
        }
      }
      __syncwarp();
      if (lane == bj) {
        for (int a = 0; a < pn; ++a) {
          w.slink[(long long)s * FS_MAXL + a] = p[a];
          backlog[p[a]] = __dadd_rn(backlog[p[a]], bytes);
        }
        w.snl[s] = pn;
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------- link index
// Link -> subflows (ascending) by a stable radix sort of (link, subflow) entries.
__global__ void __launch_bounds__(512)
    k_fs_csr(FsTopo t, uint8_t* ws, FsOffsets lo, size_t stride, int nbits, long long capF,
             long long capS) {
  __shared__ int hist[(512 / 32) * 256];
  __shared__ int sc[256];
  __shared__ uint32_t red32[32];
  __shared__ long long scr[33];
  const long long sim = blockIdx.x;
  FsWs w = fs_ws(ws + sim * stride, lo.o);
  if (w.foff[t.Q] > capF || w.soff[t.Q] > capS) return;
  const long long nsub = w.soff[t.Q];
  const int n = (int)(nsub * FS_MAXL);
  uint32_t kor = 0, kand = ~0u;
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const int s = e / FS_MAXL, a = e % FS_MAXL;
    const uint32_t key = a < w.snl[s] ? (uint32_t)w.slink[e] : (uint32_t)t.L;
    w.kA[e] = key;
    w.iA[e] = (uint32_t)s;
    kor |= key;
    kand &= key;
  }
  for (int l = threadIdx.x; l <= t.L; l += blockDim.x) w.loff[l] = 0;
  kor = block_reduce_or(kor, red32);
  kand = block_reduce_and(kand, red32);
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    if (w.kA[e] < (uint32_t)t.L) atomicAdd(&w.loff[w.kA[e]], 1);
  const int which = radix_sort<uint32_t, uint32_t>(w.kA, w.iA, w.kB, w.iB, n, kor, kand, nbits,
                                                   hist, sc);
  const uint32_t* is = which ? w.iB : w.iA;
  const uint32_t* ks = which ? w.kB : w.kA;
  for (int e = threadIdx.x; e < n; e += blockDim.x)
    if (ks[e] < (uint32_t)t.L) w.lsub[e] = (int)is[e];
  // counts -> exclusive offsets, in link order
  long long carry = 0;
  for (int l0 = 0; l0 <= t.L; l0 += blockDim.x) {
    const int l = l0 + threadIdx.x;
    const long long v = l < t.L ? w.loff[l] : 0;
    long long tot;
    const long long ex = block_excl_scan(v, scr, &tot);
    if (l <= t.L) w.loff[l] = (int)(carry + ex);
    carry += tot;
  }
}

// ---------------------------------------------------------------- the event loop
// One CTA per simulation (R#37, R#38).  Link state lives in shared memory and is
// updated incrementally, in integers, so every sum is exact and order-free:
//   wsum[l]  share-weights of the unfrozen active subflows on l, in units of 1/S
//            (weights are 1 or 1/S, R#36), reset each event from wbase[l];
//   used[l]  rates of the frozen subflows on l (B/s).
// Progressive filling: x* = min_l S*(cap - used)/wsum; the links within 1e-12 of
// x* are listed; the CTA walks the listed links' subflows (flattened), claims the
// unfrozen ones (atomicMax on the subflow's epoch), sets rate = w*x* and counts
// their weight per link (32-bit shared atomics: 64-bit ones are CAS loops); then
// each link moves that weight from wsum to used = used + weight * x*/S.  A link is
// listed at most once per event, so an event costs O(iterations * L +
// subflow-links), not O(iterations * subflows).  Link bytes grow by used*dt.

// GL: link state in the simulation's global workspace instead of shared memory
// (fabrics whose L links do not fit, e.g. the paper's 128 domains x 8 rails).
template <bool GL>
__global__ void __launch_bounds__(FS_THREADS)
    k_fs_sim(FsTopo t, const int32_t* __restrict__ policy, uint8_t* ws, FsOffsets lo,
             size_t stride, long long capF, long long capS, double* __restrict__ link_bytes,
             int* err) {
  extern __shared__ __align__(16) uint8_t fs_smem[];
  uint8_t* lbase;
  if constexpr (GL) lbase = ws + blockIdx.x * stride + lo.o[33];
  else lbase = fs_smem;
  double* used = (double*)lbase;                                     // [L]
  double* lb = used + t.L;                                           // [L]
  unsigned* wsum = (unsigned*)(lb + t.L);                            // [L]
  unsigned* wbase = wsum + t.L;                                      // [L]
  unsigned* dnew = wbase + t.L;                                      // [L]
  int* blist = (int*)(dnew + t.L);                                   // [L]
  int* bpre = blist + t.L;                                           // [L]
  int* loffs = bpre + t.L;                                           // [L+1] link offsets
  unsigned* actb = (unsigned*)(loffs + t.L + 1);                     // [capS/32] active bits
  unsigned* frzb = actb + (capS + 31) / 32;                          // [capS/32] frozen bits
  uint8_t* isb = (uint8_t*)(frzb + (capS + 31) / 32);                // [L] listed now
  __shared__ double dscr[32];
  __shared__ long long lscr[32];
  __shared__ long long lscan[33];
  __shared__ int nb;
  const long long sim = blockIdx.x;
  FsWs w = fs_ws(ws + sim * stride, lo.o);
  if (w.foff[t.Q] > capF || w.soff[t.Q] > capS) return;
  const int nflow = (int)w.foff[t.Q], nsub = (int)w.soff[t.Q];
  const double Sd = (double)t.S;
  unsigned long long* pair = w.pair;  // [M*M], global
  const int nwords = (nsub + 31) / 32;
  for (int l = threadIdx.x; l < t.L; l += FS_THREADS) {
    wbase[l] = 0;
    dnew[l] = 0;
    lb[l] = 0.0;
  }
  for (int l = threadIdx.x; l <= t.L; l += FS_THREADS) loffs[l] = w.loff[l];
  for (int q = threadIdx.x; q < nwords; q += FS_THREADS) actb[q] = 0u;
  for (int i = threadIdx.x; i < nflow; i += FS_THREADS) {
    w.rem[i] = w.fbytes[i];
    w.done[i] = 0.0;
    w.fact[i] = 1;
  }
  __syncthreads();
  const bool plb = policy[sim] == RAILS_POL_PLB;
  const int ls0 = l_leaf_spine(t, 0, 0), ls1 = l_nic_down(t, 0, 0);  // spine layer
  for (int s = threadIdx.x; s < nsub; s += FS_THREADS) {
    if (!w.sinit[s]) continue;
    atomicOr(&actb[s >> 5], 1u << (s & 31));
    const int nl = w.snl[s];
    for (int a = 0; a < nl; ++a) atomicAdd(&wbase[w.slink[(long long)s * FS_MAXL + a]], w.swi[s]);
  }
  __syncthreads();
  double tnow = 0.0, maxpair = 0.0;
  int events = 0;
  long long active = nflow;
  const double NR2 = __dmul_rn((double)t.N, t.R2);
  while (active > 0) {
    if (events > nflow + 1) {
      if (threadIdx.x == 0) flag_error(err, ERR_RANGE);
      break;
    }
    // ---- progressive filling (R#37)
    for (int l = threadIdx.x; l < t.L; l += FS_THREADS) {
      wsum[l] = wbase[l];
      used[l] = 0.0;
    }
    for (int q = threadIdx.x; q < nwords; q += FS_THREADS) frzb[q] = 0u;
    __syncthreads();
    double xu = 0.0;  // x*/S of the previous iteration, for its pending dnew
    for (int it = 0;; ++it) {
      if (it > t.L + 1) {
        if (threadIdx.x == 0) flag_error(err, ERR_RANGE);
        break;
      }
      // the last iteration's newly frozen weight leaves wsum and joins used at its
      // x* (each link is owned by one thread here and in the listing below)
      double lmin = fs_inf();
      for (int l = threadIdx.x; l < t.L; l += FS_THREADS) {
        const unsigned dn = dnew[l];
        if (dn != 0) {
          wsum[l] -= dn;
          used[l] = __dadd_rn(used[l], __dmul_rn((double)dn, xu));
          dnew[l] = 0;
        }
        isb[l] = 0;
        if (wsum[l] == 0) continue;
        const double r = fmax(__dsub_rn(l_cap(t, l), used[l]), 0.0);
        lmin = fmin(lmin, __ddiv_rn(__dmul_rn(Sd, r), (double)wsum[l]));
      }
      if (threadIdx.x == 0) nb = 0;
      const double xs = block_min_d(lmin, dscr);
      if (!(xs < fs_inf())) break;  // every active subflow frozen
      xu = __ddiv_rn(xs, Sd);
      const double thr = __dmul_rn(xs, 1.0 + 1e-12);
      for (int l = threadIdx.x; l < t.L; l += FS_THREADS) {
        if (wsum[l] == 0) continue;
        const double r = fmax(__dsub_rn(l_cap(t, l), used[l]), 0.0);
        if (__ddiv_rn(__dmul_rn(Sd, r), (double)wsum[l]) <= thr) {
          blist[atomicAdd(&nb, 1)] = l;
          isb[l] = 1;
        }
      }
      __syncthreads();
      // the listed links' subflow lists, flattened over the whole CTA (a hot
      // receiver's link can carry thousands of subflows)
      const int nbl = nb;
      int ntot;
      if (nbl <= 32) {  // usual case: one warp scans the list lengths
        if (threadIdx.x < 32) {
          const int len = threadIdx.x < nbl ? loffs[blist[threadIdx.x] + 1] - loffs[blist[threadIdx.x]] : 0;
          const int inc = warp_incl_scan(len);
          if (threadIdx.x < nbl) bpre[threadIdx.x] = inc - len;
          if (threadIdx.x == 31) lscan[32] = inc;
        }
        __syncthreads();
        ntot = (int)lscan[32];
      } else {
        long long carry = 0;
        for (int b0 = 0; b0 < nbl; b0 += FS_THREADS) {
          const int b = b0 + threadIdx.x;
          const long long len = b < nbl ? loffs[blist[b] + 1] - loffs[blist[b]] : 0;
          long long tot;
          const long long ex = block_excl_scan(len, lscan, &tot);
          if (b < nbl) bpre[b] = (int)(carry + ex);
          carry += tot;
        }
        __syncthreads();
        ntot = (int)carry;
      }
      for (int x = threadIdx.x; x < ntot; x += FS_THREADS) {
        int lo_ = 0, hi_ = nbl - 1;  // last b with bpre[b] <= x
        while (lo_ < hi_) {
          const int mid = (lo_ + hi_ + 1) >> 1;
          if (bpre[mid] <= x) lo_ = mid;
          else hi_ = mid - 1;
        }
        const int l = blist[lo_];
        const int s = w.lsub[loffs[l] + (x - bpre[lo_])];
        const unsigned bit = 1u << (s & 31);
        if (!(actb[s >> 5] & bit) || (frzb[s >> 5] & bit)) continue;
        if (atomicOr(&frzb[s >> 5], bit) & bit) continue;  // claimed by another link
        w.rate[s] = __dmul_rn(w.sw[s], xs);
        const int nl = w.snl[s];
        bool sp = false;
        for (int a = 0; a < nl; ++a) {
          const int l2 = w.slink[(long long)s * FS_MAXL + a];
          atomicAdd(&dnew[l2], (unsigned)w.swi[s]);
          sp |= isb[l2] && l2 >= ls0 && l2 < ls1;
        }
        w.shit[s] = sp;
      }
      __syncthreads();
    }
    // ---- flow rates, next completion (R#38)
    for (int p = threadIdx.x; p < t.M * t.M; p += FS_THREADS) pair[p] = 0ull;
    __syncthreads();
    double dmin = fs_inf();
    for (int i = threadIdx.x; i < nflow; i += FS_THREADS) {
      if (!w.fact[i]) continue;
      double r = 0.0;
      for (int s = w.fsub0[i]; s < w.fsub0[i + 1]; ++s)
        if (actb[s >> 5] & (1u << (s & 31))) r = __dadd_rn(r, w.rate[s]);
      w.frate[i] = r;
      dmin = fmin(dmin, __ddiv_rn(w.rem[i], r));
      const int q = w.fmsg[i];
      const int d = (int)(q / (t.N * t.G)), f = (int)((q % t.G) / t.N);
      // integer atomics: the per-pair sums (a statistic only) are order-independent
      atomicAdd(&pair[d * t.M + f], __double2ull_rn(__dmul_rn(r, 1024.0)));
    }
    const double dt = block_min_d(dmin, dscr);
    double pm = 0.0;
    for (int p = threadIdx.x; p < t.M * t.M; p += FS_THREADS)
      pm = fmax(pm, __ddiv_rn(__dmul_rn(__ull2double_rn(pair[p]), 1.0 / 1024.0), NR2));
    pm = block_max_d(pm, dscr);
    maxpair = fmax(maxpair, pm);
    tnow = __dadd_rn(tnow, dt);
    for (int l = threadIdx.x; l < t.L; l += FS_THREADS)
      lb[l] = __dadd_rn(lb[l], __dmul_rn(used[l], dt));
    const double fin_thr = __dmul_rn(dt, 1.0 + 1e-9);
    long long ndone = 0;
    for (int i = threadIdx.x; i < nflow; i += FS_THREADS) {
      if (!w.fact[i]) continue;
      const double fr = w.frate[i];
      const double fin = __ddiv_rn(w.rem[i], fr);
      w.rem[i] = __dsub_rn(w.rem[i], __dmul_rn(fr, dt));
      if (fin <= fin_thr) {
        w.done[i] = tnow;
        w.fact[i] = 0;
        ++ndone;
        for (int s = w.fsub0[i]; s < w.fsub0[i + 1]; ++s) {
          if (!(actb[s >> 5] & (1u << (s & 31)))) continue;
          atomicAnd(&actb[s >> 5], ~(1u << (s & 31)));
          const int nl = w.snl[s];
          for (int a = 0; a < nl; ++a)
            atomicSub(&wbase[w.slink[(long long)s * FS_MAXL + a]], (unsigned)w.swi[s]);
        }
      } else if (plb && w.fsub0[i + 1] - w.fsub0[i] > 1 && w.flast[i] != events - 1) {
        // PLB (R#36): a flow held back by a spine bottleneck re-hashes its spine
        const int cur = w.fcur[i];
        if (w.shit[cur]) {
          const int q = w.fmsg[i];
          const int att = ++w.fatt[i];
          const int j = ecmp_rail(t.seed + (uint64_t)att * 0x9E3779B97F4A7C15ull, q / t.G,
                                  q % t.G, t.S);
          w.flast[i] = events;
          const int nxt = w.fsub0[i] + j;
          if (nxt != cur) {
            atomicAnd(&actb[cur >> 5], ~(1u << (cur & 31)));
            atomicOr(&actb[nxt >> 5], 1u << (nxt & 31));
            w.fcur[i] = nxt;
            for (int a = 0; a < w.snl[cur]; ++a)
              atomicSub(&wbase[w.slink[(long long)cur * FS_MAXL + a]], (unsigned)w.swi[cur]);
            for (int a = 0; a < w.snl[nxt]; ++a)
              atomicAdd(&wbase[w.slink[(long long)nxt * FS_MAXL + a]], (unsigned)w.swi[nxt]);
          }
        }
      }
    }
    ++events;
    active -= block_sum_ll(ndone, lscr);
    __syncthreads();
  }
  for (int l = threadIdx.x; l < t.L; l += FS_THREADS) link_bytes[sim * t.L + l] = lb[l];
  if (threadIdx.x == 0) {
    w.simstat[0] = maxpair;
    w.simstat[1] = (double)events;
    w.simstat[2] = (double)nflow;
    w.simstat[3] = (double)nsub;
  }
}

// ---------------------------------------------------------------- results (R#39)
__global__ void __launch_bounds__(FS_THREADS)
    k_fs_finish(FsTopo t, const int64_t* __restrict__ msg, uint8_t* ws, FsOffsets lo,
                size_t stride, long long capF, long long capS, double* __restrict__ msg_cct,
                double* __restrict__ stats) {
  __shared__ int hist[(FS_THREADS / 32) * 256];
  __shared__ int sc[256];
  __shared__ uint64_t red64[32];
  __shared__ double dscr[32];
  __shared__ long long scr[33];
  const long long sim = blockIdx.x;
  const int64_t* __restrict__ ms = msg + sim * t.Q;
  FsWs w = fs_ws(ws + sim * stride, lo.o);
  if (w.foff[t.Q] > capF || w.soff[t.Q] > capS) return;
  double* cct = msg_cct + sim * t.Q;
  // per message: completion of its last flow; compacted keys of B > 0 messages
  long long carry = 0;
  double tmax = 0.0, csum = 0.0;
  long long total = 0;
  uint64_t kor = 0, kand = ~0ull;
  for (long long q0 = 0; q0 < t.Q; q0 += FS_THREADS) {
    const long long q = q0 + threadIdx.x;
    double c = 0.0;
    long long B = 0;
    if (q < t.Q) {
      B = ms[q];
      for (long long i = w.foff[q]; i < w.foff[q + 1]; ++i) c = fmax(c, w.done[i]);
      cct[q] = c;
    }
    const long long has = B > 0 ? 1 : 0;
    long long tot;
    const long long ex = block_excl_scan(has, scr, &tot);
    if (has) {
      const uint64_t key = (uint64_t)__double_as_longlong(c);
      w.cA[carry + ex] = key;
      w.ciA[carry + ex] = (uint32_t)(carry + ex);
      kor |= key;
      kand &= key;
      total += B;
      csum = __dadd_rn(csum, c);
      tmax = fmax(tmax, c);
    }
    carry += tot;
  }
  const long long nm = carry;
  tmax = block_max_d(tmax, dscr);
  __syncthreads();
  csum = block_sum_d(csum, dscr);
  __syncthreads();
  total = block_sum_ll(total, scr);
  __syncthreads();
  kor = block_reduce_or(kor, red64);
  kand = block_reduce_and(kand, red64);
  __syncthreads();
  const int which = radix_sort<uint64_t, uint32_t>(w.cA, w.ciA, w.cB, w.ciB, (int)nm, kor, kand,
                                                   64, hist, sc);
  const uint64_t* ks = which ? w.cB : w.cA;
  if (threadIdx.x == 0) {
    double* st = stats + sim * FS_NSTATS;
    const double ps[3] = {0.80, 0.95, 0.99};
    st[0] = tmax;
    st[1] = (double)total;
    st[2] = tmax > 0.0 ? __ddiv_rn((double)total, tmax) : 0.0;
    st[3] = nm > 0 ? __ddiv_rn(csum, (double)nm) : 0.0;
    for (int a = 0; a < 3; ++a) {
      double v = 0.0;
      if (nm > 0) {
        long long r = (long long)ceil(__dmul_rn(ps[a], (double)nm));
        if (r < 1) r = 1;
        v = __longlong_as_double((long long)ks[r - 1]);
      }
      st[4 + a] = v;
    }
    st[7] = w.simstat[0];
    st[8] = w.simstat[1];
    st[9] = w.simstat[2];
  }
}

// ---------------------------------------------------------------- host side
static FsTopo fs_topo(const rails_topo_t& tp, const rails_fabric_t& fb) {
  FsTopo t;
  t.M = tp.M;
  t.N = tp.N;
  t.S = fb.S;
  t.L = 2 * tp.M * tp.N * tp.N + 2 * tp.M * tp.N + 2 * tp.N * fb.S;
  t.G = (long long)tp.M * tp.N;
  t.Q = (long long)tp.M * tp.N * t.G;
  t.R1 = fb.R1;
  t.R2 = tp.R2;
  t.Rs = fb.Rs;
  t.C = tp.chunk_bytes;
  t.seed = tp.ecmp_seed;
  return t;
}

size_t flowsim_workspace_bytes(const rails_topo_t& tp, const rails_fabric_t& fb, int n_sim,
                               long long capF, long long capS) {
  const FsTopo t = fs_topo(tp, fb);
  const FsLayout lo = fs_layout(t.Q, t.L, capF, capS);
  const size_t sched = schedule_workspace_bytes(n_sim, tp.M, tp.M, tp.N);
  const size_t sarr = al256((size_t)n_sim * t.Q * 8) + al256((size_t)n_sim * t.Q) +
                      al256((size_t)n_sim * t.Q * 8) + al256((size_t)n_sim * tp.M * tp.N * 8) +
                      al256((size_t)n_sim * tp.M * 8) + al256((size_t)n_sim * tp.M * 4);
  return 256 + lo.stride * (size_t)n_sim + al256(sched) + sarr;
}

size_t flowsim_smem_bytes(const rails_topo_t& tp, const rails_fabric_t& fb, long long capS) {
  const FsTopo t = fs_topo(tp, fb);
  const size_t bits = 2 * (size_t)((capS + 31) / 32) * 4;
  return (size_t)t.L * (8 + 8 + 4 + 4 + 4 + 4 + 4 + 4 + 1) + 4 + bits + 16;
}

cudaError_t launch_flowsim_plan(const LaunchCtx& c, const rails_topo_t& tp,
                                const rails_fabric_t& fb, int n_sim, const int32_t* policy,
                                const int64_t* msg, int64_t* totals) {
  const FsTopo t = fs_topo(tp, fb);
  FsOffsets o{};
  k_fs_count<<<n_sim, FS_THREADS, 0, c.stream>>>(t, policy, msg, nullptr, o, 0, totals, 1,
                                                 c.err);
  count_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_flowsim(const LaunchCtx& c, const rails_topo_t& tp, const rails_fabric_t& fb,
                           int n_sim, const int32_t* policy, const int64_t* msg, long long capF,
                           long long capS, void* ws_, double* msg_cct, double* link_bytes,
                           double* stats) {
  const FsTopo t = fs_topo(tp, fb);
  const FsLayout lay = fs_layout(t.Q, t.L, capF, capS);
  FsOffsets o;
  for (int i = 0; i < 40; ++i) o.o[i] = lay.o[i];
  uint8_t* base = (uint8_t*)ws_ + 256;
  uint8_t* sims = base;
  uint8_t* schw = sims + lay.stride * (size_t)n_sim;
  const size_t schb = al256(schedule_workspace_bytes(n_sim, tp.M, tp.M, tp.N));
  uint8_t* sa = schw + schb;
  rails_sched_t s;
  s.full_base = (int64_t*)sa;
  sa += al256((size_t)n_sim * t.Q * 8);
  s.rem_rail = (int8_t*)sa;
  sa += al256((size_t)n_sim * t.Q);
  s.rem_off = (int64_t*)sa;
  sa += al256((size_t)n_sim * t.Q * 8);
  s.send_load = (int64_t*)sa;
  sa += al256((size_t)n_sim * tp.M * tp.N * 8);
  s.n_full = (int64_t*)sa;
  sa += al256((size_t)n_sim * tp.M * 8);
  s.n_rem = (int32_t*)sa;
  cudaError_t e;
  // the LPT schedule of every (simulation, node); only LPT simulations use it
  if ((e = launch_node(c, n_sim, tp.M, 0, tp.M, tp.N, tp.chunk_bytes, tp.ecmp_seed, tp.R2, msg,
                       s, schw, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr)) !=
      cudaSuccess)
    return e;
  k_fs_count<<<n_sim, FS_THREADS, 0, c.stream>>>(t, policy, msg, sims, o, lay.stride, nullptr, 0,
                                                 c.err);
  k_fs_build<<<n_sim, FS_THREADS, 0, c.stream>>>(t, policy, msg, s.full_base, s.rem_rail, sims,
                                                 o, lay.stride, capF, capS, c.err);
  const size_t bsm = (size_t)t.L * 8;
  if (bsm > 48 * 1024) {
    if ((e = cudaFuncSetAttribute(k_fs_minrtt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)bsm)) != cudaSuccess)
      return e;
  }
  k_fs_minrtt<<<n_sim, 32, bsm, c.stream>>>(t, policy, sims, o, lay.stride, capF, capS);
  int nbits = 1;
  while ((1LL << nbits) <= t.L) ++nbits;
  k_fs_csr<<<n_sim, 512, 0, c.stream>>>(t, sims, o, lay.stride, nbits, capF, capS);
  const size_t ssm = flowsim_smem_bytes(tp, fb, capS);
  const char* gv = getenv("RAILS_FS_GLOBAL");
  if (ssm > 200 * 1024 || (gv && gv[0] == '1')) {
    k_fs_sim<true><<<n_sim, FS_THREADS, 0, c.stream>>>(t, policy, sims, o, lay.stride, capF,
                                                       capS, link_bytes, c.err);
  } else {
    if (ssm > 48 * 1024) {
      if ((e = cudaFuncSetAttribute(k_fs_sim<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ssm)) != cudaSuccess)
        return e;
    }
    k_fs_sim<false><<<n_sim, FS_THREADS, ssm, c.stream>>>(t, policy, sims, o, lay.stride, capF,
                                                          capS, link_bytes, c.err);
  }
  k_fs_finish<<<n_sim, FS_THREADS, 0, c.stream>>>(t, msg, sims, o, lay.stride, capF, capS,
                                                  msg_cct, stats);
  count_launch(6);
  return cudaGetLastError();
}

}  // namespace rails
