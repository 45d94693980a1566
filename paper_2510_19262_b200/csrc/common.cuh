// common.cuh -- internal helpers of the B200 RailS kernels (sm_100a only).
// Not part of the ABI; see include/rails.h.  No code here is shared with oracle/.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rails.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "librails is written for sm_100a (B200) only"
#endif

namespace rails {

constexpr unsigned FULL = 0xffffffffu;

// Device error bits, OR-ed into the flag word passed to every kernel.
enum : int { ERR_RANGE = 1, ERR_NOSPC = 2, ERR_OVERFLOW = 4, ERR_TIMEOUT = 8 };

__device__ __forceinline__ void flag_error(int* err, int bit) {
  if ((*(volatile int*)err & bit) == 0) atomicOr(err, bit);
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes of the warp holding the same key (a "multi-split" match): one ballot per
// key bit, so the cost is nbits ballots whatever the number of distinct keys
// (__match_any_sync serialises over distinct values).  All 32 lanes must call it;
// invalid lanes get 0 and are excluded from every valid lane's mask.
__device__ __forceinline__ unsigned warp_match_bits(unsigned key, int nbits, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll 4
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (key >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? bal : ~bal;
  }
  return valid ? peers : 0u;
}

// Same with the key width known at compile time (fully unrolled: one VOTE and one
// LOP3 per bit plus the bit-mask extraction).
template <int NB>
__device__ __forceinline__ unsigned warp_match_nb(unsigned key, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const unsigned m = (unsigned)(((int)(key << (31 - b))) >> 31);  // bit b -> 0 / ~0
    const unsigned bal = __ballot_sync(0xffffffffu, m != 0u);
    peers &= ~(bal ^ m);
  }
  return valid ? peers : 0u;
}

// Warp-inclusive scan helpers (int64 and int32).
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T n = __shfl_xor_sync(FULL, v, o);
    v = n > v ? n : v;
  }
  return v;
}

// Block-wide exclusive scan of one int64 per thread; returns the exclusive prefix
// and writes the block total to *total.  scratch: >= 33 int64 in shared memory.
__device__ __forceinline__ long long block_excl_scan(long long v, long long* scratch,
                                                     long long* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  long long inc = warp_incl_scan(v);
  if (lane == 31) scratch[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    long long s = lane < nw ? scratch[lane] : 0;
    long long si = warp_incl_scan(s);
    if (lane < nw) scratch[lane] = si - s;
    if (lane == 31) scratch[32] = si;
  }
  __syncthreads();
  long long r = scratch[wid] + inc - v;
  *total = scratch[32];
  __syncthreads();
  return r;
}

// ---- system-scope flags of the peer-memory exchanges (k_eval.cu, k_owner.cu)
__device__ __forceinline__ void st_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// A rank waits at most this long for a peer's flag.  Generous on purpose: ranks
// sharing one GPU (the single-GPU multi-rank tests) only progress when the GPU's
// time slicing runs their context.
constexpr unsigned long long PEER_TIMEOUT_NS = 30ull * 1000000000ull;

// Wait until the monotonic call counter at f reaches gen (wrap-safe compare).  On
// timeout: ERR_TIMEOUT in the device flag and false; the exchange is then out of
// step and must be rebuilt (include/rails.h, rails_eval_finalize_peer).
__device__ __forceinline__ bool wait_flag_ge(const uint32_t* f, uint32_t gen, int* err) {
  if ((int)(ld_acquire_sys(f) - gen) >= 0) return true;
  const unsigned long long t0 = globaltimer_ns();
  while ((int)(ld_acquire_sys(f) - gen) < 0) {
    __nanosleep(128);
    if (globaltimer_ns() - t0 > PEER_TIMEOUT_NS) {
      flag_error(err, ERR_TIMEOUT);
      return false;
    }
  }
  return true;
}

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream
// serialization may start while the previous kernel of its stream runs; pdl_wait()
// blocks until that kernel has completed and its memory is visible.  The previous
// kernel's pdl_trigger() lets the dependent grid be scheduled early (its CTAs then
// sit in pdl_wait() on SMs the previous grid leaves free).  Both are no-ops for
// ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Eight consecutive int64 per thread as two 256-bit accesses (sm_100 LDG/STG.256):
// a warp's 2 KiB then moves in 64 whole sectors instead of 256 partial ones when
// each thread owns 8 consecutive elements.  p must be 32-byte aligned.
__device__ __forceinline__ void ld8_s64(const int64_t* p, long long (&v)[8]) {
  asm volatile("ld.global.v4.s64 {%0,%1,%2,%3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
  asm volatile("ld.global.v4.s64 {%0,%1,%2,%3}, [%4];"
               : "=l"(v[4]), "=l"(v[5]), "=l"(v[6]), "=l"(v[7]) : "l"(p + 4));
}
__device__ __forceinline__ void st8_s64(int64_t* p, const long long (&v)[8]) {
  asm volatile("st.global.v4.s64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v[0]), "l"(v[1]),
               "l"(v[2]), "l"(v[3]) : "memory");
  asm volatile("st.global.v4.s64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4), "l"(v[4]), "l"(v[5]),
               "l"(v[6]), "l"(v[7]) : "memory");
}
__device__ __forceinline__ bool aligned32(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 31) == 0;
}

// ECMP rail (R#14): splitmix64 output step, this library's own copy.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ int ecmp_rail(uint64_t seed, long long src, long long dst, int N) {
  uint64_t key = ((uint64_t)src << 32) | (uint64_t)dst;
  uint32_t hi = (uint32_t)(mix64(key ^ seed) >> 32);
  return (int)(hi % (uint32_t)N);
}

// Division by the chunk size C: shift when C is a power of two.
struct ChunkDiv {
  long long C;
  int shift;  // >= 0 when C == 1 << shift, else -1
  __device__ __forceinline__ long long div(long long b) const {
    return shift >= 0 ? (b >> shift) : (b / C);
  }
};

// Streaming 16-byte global accesses (opaque payload bytes; never touched as floats).
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_cs(uint4* p, const uint4& v) {  // evict-first store
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

}  // namespace rails

// ---------------------------------------------------------------- host launchers
// (defined in the kernel .cu files, called by abi.cu after validation)
namespace rails {
struct LaunchCtx {
  cudaStream_t stream;
  int* err;      // device error flag
  int num_sms;
};

cudaError_t launch_histogram(const LaunchCtx&, int U, int nd, int d0, int M, int N, int ngs,
                             int T, int k, const int32_t* topk, const int32_t* lut, int n_inst,
                             long long row_bytes, int32_t* counts, int64_t* msg,
                             int32_t* rank);

size_t schedule_workspace_bytes(int U, int nd, int M, int N);
cudaError_t launch_node(const LaunchCtx&, int U, int nd, int d0, int M, int N, long long C,
                        uint64_t seed, double R2, const int64_t* msg, const rails_sched_t& s,
                        void* ws, int32_t* rem_qp, int qps_per_rail, const rails_eval_t* ev,
                        const rails_final_t* fin, int64_t* rail_base, int64_t* rail_total,
                        bool* fused);

cudaError_t launch_chains(const LaunchCtx&, int U, int nd, int d0, int M, int N, long long C,
                          const int64_t* msg, const rails_sched_t& s, uint64_t* ws_res,
                          uint32_t* ws_qp, uint32_t* ws_w, int32_t* ws_inv, uint8_t* scratch,
                          int32_t* rem_qp, int qps_per_rail, int cshift, int nbits,
                          bool defer_expand = false);

void schedule_workspace_ptrs(void* ws, int U, int nd, int M, int N, int64_t** acc,
                             unsigned** cnt, uint64_t** res);
size_t assign_workspace_bytes(int n_seg, long long F);
cudaError_t launch_assign(const LaunchCtx&, int N, int n_seg, const int64_t* seg_off,
                          long long F, const int64_t* w, int32_t* rail, int64_t* off,
                          int64_t* load, void* ws);

// ex_inv / ex_res (optional): the chains' inverse permutation and sorted-order
// results; the evaluation then also expands them into s.rem_rail / s.rem_off (the
// k_expand pass fused into its message loop) instead of reading s.rem_rail.
cudaError_t launch_eval(const LaunchCtx&, int U, int nd, int d0, int M, int N, long long C,
                        uint64_t seed, const int64_t* msg, const rails_sched_t& s,
                        const rails_eval_t& e, const int32_t* ex_inv = nullptr,
                        const uint64_t* ex_res = nullptr);
cudaError_t launch_finalize(const LaunchCtx&, int U, int M, int N, double R2,
                            const int64_t* red_sum, const int64_t* red_max,
                            const rails_final_t& f);

size_t peer_buffer_bytes(int U, int world, long long rsl);
void owner_exchange_layout(int U, int world, long long N, long long G, size_t* bytes,
                           size_t* gflag_off, size_t* msg_off);
cudaError_t launch_gather_rows_peer(const LaunchCtx&, int U, int N, long long G, int ng,
                                    const int64_t* const* msg_loc, const int* g0,
                                    const rails_peer_t& peer, int nplay);
cudaError_t launch_peer_barrier(const LaunchCtx&, const rails_peer_t& peer, int nplay);
cudaError_t launch_finalize_peer(const LaunchCtx&, int U, int M, int N, double R2,
                                 int64_t* const* red_sum, int64_t* const* red_max,
                                 const rails_peer_t& peer, const rails_final_t* f, int nplay);

cudaError_t launch_rail_offsets(const LaunchCtx&, long long n, const int64_t* send_load,
                                int64_t* rail_base, int64_t* total);
cudaError_t launch_pack(const LaunchCtx&, int U, int nd, int d0, int M, int N, int T, int k,
                        long long C, const void* x, const int32_t* topk, const int32_t* lut,
                        int n_inst, const int32_t* rank, const int64_t* msg,
                        long long row_bytes, const rails_sched_t& s, const int64_t* rail_base,
                        void* out, long long out_cap);

cudaError_t launch_pack_owner(const LaunchCtx&, int U, int nd, int d0, int M, int N, int g0,
                              int ng, int T, int k, long long C, const void* x,
                              const int32_t* topk, const int32_t* lut, int n_inst,
                              const int32_t* rank, const int64_t* msg, long long row_bytes,
                              const rails_sched_t& s, const int64_t* rail_base,
                              void* const* rail_ptr, const int64_t* rail_cap);
cudaError_t launch_rail_offsets_owner(const LaunchCtx&, long long ublk, int N,
                                      const int64_t* send_load, int64_t* rail_base,
                                      int64_t* rail_total);

cudaError_t launch_transpose(const LaunchCtx&, int U, long long G, const int64_t* src,
                             int64_t* dst);
cudaError_t launch_recv_offsets(const LaunchCtx&, int U, long long G, const int32_t* counts,
                                int64_t* in_off, int64_t* rows_in);
cudaError_t launch_pack_combine(const LaunchCtx&, int U, int nd, int d0, int M, int N,
                                long long Rcap, long long C, const void* y,
                                const int64_t* in_off, const int64_t* rows_in,
                                const int64_t* msgc, const rails_sched_t& s,
                                const int64_t* rail_base, void* out, long long out_cap,
                                long long RB);
cudaError_t launch_unpack_combine(const LaunchCtx&, int U, int nd, int d0, int M, int N, int T,
                                  int k, long long C, const int32_t* topk, const int32_t* lut,
                                  int n_inst, const int32_t* rank, const float* w, const void* y,
                                  long long Rcap, const int64_t* in_off, const int64_t* msgc,
                                  const rails_sched_t& s, const int64_t* rail_base_c,
                                  const void* comb_out, float* out, long long RB);

size_t flowsim_workspace_bytes(const rails_topo_t& tp, const rails_fabric_t& fb, int n_sim,
                               long long capF, long long capS);
size_t flowsim_smem_bytes(const rails_topo_t& tp, const rails_fabric_t& fb, long long capS);
cudaError_t launch_flowsim_plan(const LaunchCtx&, const rails_topo_t& tp,
                                const rails_fabric_t& fb, int n_sim, const int32_t* policy,
                                const int64_t* msg, int64_t* totals);
cudaError_t launch_flowsim(const LaunchCtx&, const rails_topo_t& tp, const rails_fabric_t& fb,
                           int n_sim, const int32_t* policy, const int64_t* msg, long long capF,
                           long long capS, void* ws, double* msg_cct, double* link_bytes,
                           double* stats);

void count_launch(int n);

// Grid of a row-streaming kernel (one warp per row inside a grid-stride loop):
// about `rpw` rows per warp, the CTAs running in waves, instead of one persistent
// wave of resident CTAs striding over every row.  On B200 the persistent grid held
// the C3 pack at 90% of the copy peak, 8 rows per warp reach 99-100% (DESIGN.md
// section 12); one row per warp pays a CTA launch per row.  rpw = 0: the persistent
// grid (one wave of resident CTAs).
inline long long wave_grid(int num_sms, int per_sm, long long need_ctas, long long rpw) {
  const long long resident = (long long)num_sms * (per_sm < 1 ? 1 : per_sm);
  long long grid = rpw >= 1 ? (need_ctas + rpw - 1) / rpw : resident;
  if (grid < resident) grid = resident;
  if (grid > need_ctas) grid = need_ctas;
  if (grid > 0x7fffffffLL) grid = 0x7fffffffLL;
  return grid < 1 ? 1 : grid;
}

}  // namespace rails
