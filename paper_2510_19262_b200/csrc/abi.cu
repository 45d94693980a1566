// abi.cu -- the extern "C" boundary declared in include/rails.h.
//
// Host-side argument validation (nothing is enqueued on an argument error), the
// device error flag behind rails_check, the thread-local last-error string and the
// launch counter.  All compute is in k_*.cu; this file only validates and launches.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

__device__ int g_rails_err;  // process-wide device error flag (per device)

namespace rails {
static thread_local char t_err[512] = "";
static thread_local long long t_launches = 0;
void count_launch(int n) { t_launches += n; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return code;
}

static std::mutex g_mu;
static int* g_err_ptr[64];
static int g_sms[64];

static int ctx(void* stream, LaunchCtx* c) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(RAILS_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  if (dev < 0 || dev >= 64) return fail(RAILS_ECUDA, "device index %d unsupported", dev);
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_err_ptr[dev]) {
    void* p = nullptr;
    e = cudaGetSymbolAddress(&p, g_rails_err);
    if (e != cudaSuccess)
      return fail(RAILS_ECUDA, "cudaGetSymbolAddress: %s (is this an sm_100 device?)",
                  cudaGetErrorString(e));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_err_ptr[dev] = (int*)p;
    g_sms[dev] = sms > 0 ? sms : 148;
  }
  c->stream = (cudaStream_t)stream;
  c->err = g_err_ptr[dev];
  c->num_sms = g_sms[dev];
  return RAILS_OK;
}

static int cuda_rc(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return RAILS_OK;
  return fail(RAILS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

static int check_topo(const rails_topo_t* t) {
  if (!t) return fail(RAILS_EINVAL, "topo is NULL");
  if (t->M < 2) return fail(RAILS_EINVAL, "M=%d: need at least 2 nodes (P:184)", t->M);
  if (t->N < 1 || t->N > 32) return fail(RAILS_EINVAL, "N=%d: need 1 <= N <= 32", t->N);
  if ((long long)t->M * t->N > (1LL << 20))
    return fail(RAILS_EINVAL, "M*N=%lld exceeds 2^20 GPUs", (long long)t->M * t->N);
  if (t->chunk_bytes < 1 || t->chunk_bytes > (1LL << 31))
    return fail(RAILS_EINVAL, "chunk_bytes=%lld: need 1 <= C <= 2^31", (long long)t->chunk_bytes);
  if (!(t->R2 > 0) || !std::isfinite(t->R2)) return fail(RAILS_EINVAL, "R2 must be > 0");
  if (t->R1 != 0 && !(t->R1 > t->R2))
    return fail(RAILS_EINVAL, "R1 must exceed R2 (P:333) or be 0");
  return RAILS_OK;
}

static int check_shard(const rails_topo_t* t, const rails_shard_t* s) {
  if (!s) return fail(RAILS_EINVAL, "shard is NULL");
  if (s->U < 1) return fail(RAILS_EINVAL, "U=%d: need >= 1", s->U);
  if (s->nd < 1 || s->d0 < 0 || (long long)s->d0 + s->nd > t->M)
    return fail(RAILS_EINVAL, "shard nodes [%d, %d) outside [0, %d)", s->d0, s->d0 + s->nd, t->M);
  const long long NG = (long long)t->N * t->M * t->N;
  if ((long long)s->U * s->nd * NG > (1LL << 40))
    return fail(RAILS_EINVAL, "U*nd*N*G too large");
  return RAILS_OK;
}

static bool al(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

}  // namespace rails

using namespace rails;

extern "C" {

int32_t rails_version(void) { return 200; }



const char* rails_last_error(void) { return t_err; }

int64_t rails_launch_count(int32_t reset) {
  long long v = t_launches;
  if (reset) t_launches = 0;
  return v;
}

int rails_check(void* stream) {
  LaunchCtx c;
  int rc = ctx(stream, &c);
  if (rc) return rc;
  cudaError_t e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) return cuda_rc(e, "stream");
  int flag = 0;
  e = cudaMemcpy(&flag, c.err, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_rc(e, "read error flag");
  if (flag) {
    int zero = 0;
    cudaMemcpy(c.err, &zero, sizeof(int), cudaMemcpyHostToDevice);
  }
  if (flag & ERR_TIMEOUT)
    return fail(RAILS_ETIMEDOUT,
                "device: a peer rank's flag did not arrive within %llu s; the peer exchange is "
                "out of step -- rebuild it (PeerFinalize / RailOwnerNode) before the next call",
                (unsigned long long)(PEER_TIMEOUT_NS / 1000000000ull));
  if (flag & ERR_RANGE) return fail(RAILS_ERANGE, "device: value out of range (routing id, LUT, rank or byte count)");
  if (flag & ERR_NOSPC) return fail(RAILS_ENOSPC, "device: output buffer too small");
  if (flag & ERR_OVERFLOW) return fail(RAILS_EOVERFLOW, "device: load overflow");
  return RAILS_OK;
}

int rails_histogram(const rails_topo_t* topo, const rails_shard_t* sh, int32_t T, int32_t k,
                    const int32_t* topk_inst, const int32_t* inst_to_gpu, int32_t n_inst,
                    int64_t row_bytes, int32_t* counts, int64_t* msg_bytes, int32_t* row_rank,
                    void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (T < 1 || k < 1 || k > 32) return fail(RAILS_EINVAL, "need T >= 1 and 1 <= k <= 32");
  if ((long long)T * k > (1LL << 30)) return fail(RAILS_EINVAL, "T*k too large");
  if (n_inst < 1 || row_bytes < 1) return fail(RAILS_EINVAL, "need n_inst >= 1, row_bytes >= 1");
  if (!topk_inst || !inst_to_gpu || !counts || !msg_bytes)
    return fail(RAILS_EINVAL, "NULL array argument");
  if ((long long)topo->M * topo->N > 49152)
    return fail(RAILS_ENOSPC, "G=%lld: histogram bins exceed shared memory",
                (long long)topo->M * topo->N);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_histogram(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, topo->N, T, k,
                                  topk_inst,
                                  inst_to_gpu, n_inst, row_bytes, counts, msg_bytes, row_rank),
                 "rails_histogram launch");
}

int rails_schedule_workspace(const rails_topo_t* topo, const rails_shard_t* sh, size_t* bytes) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (!bytes) return fail(RAILS_EINVAL, "bytes is NULL");
  *bytes = schedule_workspace_bytes(sh->U, sh->nd, topo->M, topo->N);
  return RAILS_OK;
}

static int schedule_impl(const rails_topo_t* topo, const rails_shard_t* sh,
                         const int64_t* msg_bytes, const rails_sched_t* out, void* ws,
                         size_t ws_bytes, int32_t* rem_qp, int32_t qps, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (!msg_bytes || !out || !out->full_base || !out->rem_rail || !out->rem_off ||
      !out->send_load || !out->n_full || !out->n_rem || !ws)
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(ws, 256)) return fail(RAILS_EINVAL, "workspace must be 256-byte aligned");
  const size_t need = schedule_workspace_bytes(sh->U, sh->nd, topo->M, topo->N);
  if (ws_bytes < need) return fail(RAILS_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_node(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, topo->chunk_bytes,
                             topo->ecmp_seed, topo->R2, msg_bytes, *out, ws, rem_qp, qps, nullptr,
                             nullptr, nullptr, nullptr, nullptr),
                 "rails_lpt_schedule launch");
}

int rails_lpt_schedule(const rails_topo_t* topo, const rails_shard_t* sh,
                       const int64_t* msg_bytes, const rails_sched_t* out, void* ws,
                       size_t ws_bytes, void* stream) {
  return schedule_impl(topo, sh, msg_bytes, out, ws, ws_bytes, nullptr, 0, stream);
}

int rails_lpt_schedule_qp(const rails_topo_t* topo, const rails_shard_t* sh,
                          const int64_t* msg_bytes, const rails_sched_t* out,
                          int32_t qps_per_rail, int32_t* rem_qp, void* ws, size_t ws_bytes,
                          void* stream) {
  if (qps_per_rail < 1) return fail(RAILS_EINVAL, "qps_per_rail %d < 1", (int)qps_per_rail);
  if (!rem_qp) return fail(RAILS_EINVAL, "rem_qp is NULL");
  return schedule_impl(topo, sh, msg_bytes, out, ws, ws_bytes, rem_qp, qps_per_rail, stream);
}

int rails_assign_workspace(int32_t n_seg, int64_t F, size_t* bytes) {
  if (n_seg < 1 || F < 0 || !bytes) return fail(RAILS_EINVAL, "bad arguments");
  *bytes = assign_workspace_bytes(n_seg, F);
  return RAILS_OK;
}

int rails_lpt_assign(int32_t N, int32_t n_seg, const int64_t* seg_off, int64_t F,
                     const int64_t* w, int32_t* rail, int64_t* off, int64_t* load, void* ws,
                     size_t ws_bytes, void* stream) {
  if (N < 1 || N > 32) return fail(RAILS_EINVAL, "N=%d: need 1 <= N <= 32", N);
  if (n_seg < 1 || F < 0 || F > (1LL << 31) - 1) return fail(RAILS_EINVAL, "bad n_seg or F");
  if (!seg_off || !load || !ws || (F > 0 && (!w || !rail || !off)))
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(ws, 256)) return fail(RAILS_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < assign_workspace_bytes(n_seg, F))
    return fail(RAILS_ENOSPC, "workspace too small");
  LaunchCtx c;
  int rc;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_assign(c, N, n_seg, seg_off, F, w, rail, off, load, ws),
                 "rails_lpt_assign launch");
}

static bool eval_ok(const rails_eval_t* e) {
  return e && e->S && e->S_e && e->S_u && e->mse && e->nmse && e->red_sum && e->red_max;
}

int rails_eval(const rails_topo_t* topo, const rails_shard_t* sh, const int64_t* msg_bytes,
               const rails_sched_t* sched, const rails_eval_t* out, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (!msg_bytes || !sched || !sched->full_base || !sched->rem_rail || !sched->n_full ||
      !eval_ok(out))
    return fail(RAILS_EINVAL, "NULL argument");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_eval(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, topo->chunk_bytes,
                             topo->ecmp_seed, msg_bytes, *sched, *out),
                 "rails_eval launch");
}

int rails_eval_finalize(const rails_topo_t* topo, int32_t U, const int64_t* red_sum,
                        const int64_t* red_max, const rails_final_t* out, void* stream) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if (U < 1 || !red_sum || !red_max || !out) return fail(RAILS_EINVAL, "bad argument");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_finalize(c, U, topo->M, topo->N, topo->R2, red_sum, red_max, *out),
                 "rails_eval_finalize launch");
}

int rails_schedule_eval(const rails_topo_t* topo, const rails_shard_t* sh,
                        const int64_t* msg_bytes, const rails_sched_t* sched,
                        const rails_eval_t* ev, const rails_final_t* fin, int64_t* rail_base,
                        int64_t* rail_total, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (!msg_bytes || !sched || !sched->full_base || !sched->rem_rail || !sched->rem_off ||
      !sched->send_load || !sched->n_full || !sched->n_rem || !ws || !eval_ok(ev))
    return fail(RAILS_EINVAL, "NULL argument");
  if (fin && (sh->d0 != 0 || sh->nd != topo->M))
    return fail(RAILS_EINVAL, "final needs every node of the units (d0 = 0, nd = M); "
                              "finalize after the a6 exchange instead");
  if ((rail_base == nullptr) != (rail_total == nullptr))
    return fail(RAILS_EINVAL, "rail_base and rail_total go together");
  if (!al(ws, 256)) return fail(RAILS_EINVAL, "workspace must be 256-byte aligned");
  const size_t need = schedule_workspace_bytes(sh->U, sh->nd, topo->M, topo->N);
  if (ws_bytes < need) return fail(RAILS_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  bool fused = false;
  cudaError_t e = launch_node(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, topo->chunk_bytes,
                              topo->ecmp_seed, topo->R2, msg_bytes, *sched, ws, nullptr, 0, ev,
                              fin, rail_base, rail_total, &fused);
  if (e == cudaSuccess && !fused) {  // node too large for the fused evaluation
    e = launch_eval(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, topo->chunk_bytes,
                    topo->ecmp_seed, msg_bytes, *sched, *ev);
    if (e == cudaSuccess && fin)
      e = launch_finalize(c, sh->U, topo->M, topo->N, topo->R2, ev->red_sum, ev->red_max, *fin);
    if (e == cudaSuccess && rail_base)
      e = launch_rail_offsets(c, (long long)sh->U * sh->nd * topo->N, sched->send_load,
                              rail_base, rail_total);
  }
  return cuda_rc(e, "rails_schedule_eval launch");
}

int rails_histogram_schedule_eval(const rails_topo_t* topo, const rails_shard_t* sh, int32_t T,
                                  int32_t k, const int32_t* topk_inst, const int32_t* inst_to_gpu,
                                  int32_t n_inst, int64_t row_bytes, int32_t* counts,
                                  int64_t* msg_bytes, int32_t* row_rank,
                                  const rails_sched_t* sched, const rails_eval_t* ev,
                                  const rails_final_t* fin, int64_t* rail_base,
                                  int64_t* rail_total, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (T < 1 || k < 1 || k > 32) return fail(RAILS_EINVAL, "need T >= 1 and 1 <= k <= 32");
  if ((long long)T * k > (1LL << 30)) return fail(RAILS_EINVAL, "T*k too large");
  if (n_inst < 1 || row_bytes < 1) return fail(RAILS_EINVAL, "need n_inst >= 1, row_bytes >= 1");
  if (!topk_inst || !inst_to_gpu || !counts || !msg_bytes)
    return fail(RAILS_EINVAL, "NULL array argument");
  if ((long long)topo->M * topo->N > 49152)
    return fail(RAILS_ENOSPC, "G=%lld: histogram bins exceed shared memory",
                (long long)topo->M * topo->N);
  if (!sched || !sched->full_base || !sched->rem_rail || !sched->rem_off || !sched->send_load ||
      !sched->n_full || !sched->n_rem || !ws || !eval_ok(ev))
    return fail(RAILS_EINVAL, "NULL argument");
  if (fin && (sh->d0 != 0 || sh->nd != topo->M))
    return fail(RAILS_EINVAL, "final needs every node of the units (d0 = 0, nd = M); "
                              "finalize after the a6 exchange instead");
  if ((rail_base == nullptr) != (rail_total == nullptr))
    return fail(RAILS_EINVAL, "rail_base and rail_total go together");
  if (!al(ws, 256)) return fail(RAILS_EINVAL, "workspace must be 256-byte aligned");
  const size_t need = schedule_workspace_bytes(sh->U, sh->nd, topo->M, topo->N);
  if (ws_bytes < need) return fail(RAILS_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  // the histogram, then the fused schedule + eval kernel (launched with PDL behind it)
  cudaError_t e = launch_histogram(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, topo->N, T, k,
                                   topk_inst, inst_to_gpu, n_inst, row_bytes, counts, msg_bytes,
                                   row_rank);
  if (e != cudaSuccess) return cuda_rc(e, "rails_histogram_schedule_eval launch");
  return rails_schedule_eval(topo, sh, msg_bytes, sched, ev, fin, rail_base, rail_total, ws,
                             ws_bytes, stream);
}

int rails_rail_offsets(const rails_topo_t* topo, const rails_shard_t* sh,
                       const int64_t* send_load, int64_t* rail_base, int64_t* total,
                       void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (!send_load || !rail_base || !total) return fail(RAILS_EINVAL, "NULL argument");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_rail_offsets(c, (long long)sh->U * sh->nd * topo->N, send_load,
                                     rail_base, total),
                 "rails_rail_offsets launch");
}

int rails_pack(const rails_topo_t* topo, const rails_shard_t* sh, int32_t T, int32_t k,
               const void* x, const int32_t* topk_inst, const int32_t* inst_to_gpu,
               int32_t n_inst, const int32_t* row_rank, const int64_t* msg_bytes,
               int64_t row_bytes, const rails_sched_t* sched, const int64_t* rail_base,
               void* out, int64_t out_cap, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (T < 1 || k < 1 || k > 32 || n_inst < 1) return fail(RAILS_EINVAL, "bad T, k or n_inst");
  if (row_bytes < 16 || row_bytes % 16 || row_bytes > (1LL << 30))
    return fail(RAILS_EINVAL, "row_bytes=%lld must be a positive multiple of 16",
                (long long)row_bytes);
  if (topo->chunk_bytes % 16)
    return fail(RAILS_EINVAL, "pack needs chunk_bytes %% 16 == 0 (16-byte vector copies)");
  if (!x || !topk_inst || !inst_to_gpu || !row_rank || !msg_bytes || !sched ||
      !sched->full_base || !sched->rem_rail || !sched->rem_off || !rail_base ||
      (!out && out_cap > 0))
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(x, 16) || (out && !al(out, 16))) return fail(RAILS_EINVAL, "x/out must be 16-byte aligned");
  if (out_cap < 0) return fail(RAILS_EINVAL, "out_cap < 0");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_pack(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, T, k, topo->chunk_bytes,
                             x, topk_inst, inst_to_gpu, n_inst, row_rank, msg_bytes, row_bytes,
                             *sched, rail_base, out, out_cap),
                 "rails_pack launch");
}

int rails_histogram_gpus(const rails_topo_t* topo, const rails_shard_t* sh, int32_t g0,
                         int32_t ng, int32_t T, int32_t k, const int32_t* topk_inst,
                         const int32_t* inst_to_gpu, int32_t n_inst, int64_t row_bytes,
                         int32_t* counts, int64_t* msg_bytes, int32_t* row_rank, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (g0 < 0 || ng < 1 || g0 + ng > topo->N)
    return fail(RAILS_EINVAL, "GPU range [%d, %d) outside [0, %d)", g0, g0 + ng, topo->N);
  if (T < 1 || k < 1 || k > 32) return fail(RAILS_EINVAL, "need T >= 1 and 1 <= k <= 32");
  if ((long long)T * k > (1LL << 30)) return fail(RAILS_EINVAL, "T*k too large");
  if (n_inst < 1 || row_bytes < 1) return fail(RAILS_EINVAL, "need n_inst >= 1, row_bytes >= 1");
  if (!topk_inst || !inst_to_gpu || !counts || !msg_bytes)
    return fail(RAILS_EINVAL, "NULL array argument");
  if ((long long)topo->M * topo->N > 49152)
    return fail(RAILS_ENOSPC, "G=%lld: histogram bins exceed shared memory",
                (long long)topo->M * topo->N);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_histogram(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, ng, T, k,
                                  topk_inst, inst_to_gpu, n_inst, row_bytes, counts, msg_bytes,
                                  row_rank),
                 "rails_histogram_gpus launch");
}

int rails_rail_offsets_owner(const rails_topo_t* topo, const rails_shard_t* sh,
                             const int64_t* send_load, int64_t* rail_base, int64_t* rail_total,
                             void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (!send_load || !rail_base || !rail_total) return fail(RAILS_EINVAL, "NULL argument");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_rail_offsets_owner(c, (long long)sh->U * sh->nd, topo->N, send_load,
                                           rail_base, rail_total),
                 "rails_rail_offsets_owner launch");
}

int rails_pack_owner(const rails_topo_t* topo, const rails_shard_t* sh, int32_t g0, int32_t ng,
                     int32_t T, int32_t k, const void* x, const int32_t* topk_inst,
                     const int32_t* inst_to_gpu, int32_t n_inst, const int32_t* row_rank,
                     const int64_t* msg_bytes, int64_t row_bytes, const rails_sched_t* sched,
                     const int64_t* rail_base, void* const* rail_ptr, const int64_t* rail_cap,
                     void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (g0 < 0 || ng < 1 || g0 + ng > topo->N)
    return fail(RAILS_EINVAL, "GPU range [%d, %d) outside [0, %d)", g0, g0 + ng, topo->N);
  if (T < 1 || k < 1 || k > 32 || n_inst < 1) return fail(RAILS_EINVAL, "bad T, k or n_inst");
  if (row_bytes < 16 || row_bytes % 16 || row_bytes > (1LL << 30))
    return fail(RAILS_EINVAL, "row_bytes=%lld must be a positive multiple of 16",
                (long long)row_bytes);
  if (topo->chunk_bytes % 16)
    return fail(RAILS_EINVAL, "pack needs chunk_bytes %% 16 == 0 (16-byte vector copies)");
  if (!x || !topk_inst || !inst_to_gpu || !row_rank || !msg_bytes || !sched ||
      !sched->full_base || !sched->rem_rail || !sched->rem_off || !rail_base || !rail_ptr ||
      !rail_cap)
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(x, 16)) return fail(RAILS_EINVAL, "x must be 16-byte aligned");
  for (int j = 0; j < topo->N; ++j) {
    if (rail_cap[j] < 0 || (rail_cap[j] > 0 && (!rail_ptr[j] || !al(rail_ptr[j], 16))))
      return fail(RAILS_EINVAL, "rail %d: pointer NULL/misaligned or negative capacity", j);
  }
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_pack_owner(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, g0, ng, T, k,
                                   topo->chunk_bytes, x, topk_inst, inst_to_gpu, n_inst,
                                   row_rank, msg_bytes, row_bytes, *sched, rail_base, rail_ptr,
                                   rail_cap),
                 "rails_pack_owner launch");
}

int rails_transpose_traffic(const rails_topo_t* topo, int32_t U, const int64_t* msg,
                            int64_t* msg_t, void* stream) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if (U < 1 || !msg || !msg_t || msg == msg_t) return fail(RAILS_EINVAL, "bad argument");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_transpose(c, U, (long long)topo->M * topo->N, msg, msg_t),
                 "rails_transpose_traffic launch");
}

int rails_recv_offsets(const rails_topo_t* topo, int32_t U, const int32_t* counts,
                       int64_t* in_off, int64_t* rows_in, void* stream) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if (U < 1 || !counts || !in_off || !rows_in) return fail(RAILS_EINVAL, "bad argument");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_recv_offsets(c, U, (long long)topo->M * topo->N, counts, in_off, rows_in),
                 "rails_recv_offsets launch");
}

int rails_pack_combine(const rails_topo_t* topo, const rails_shard_t* sh, int64_t row_bytes,
                       int64_t rows_cap, const void* y, const int64_t* in_off,
                       const int64_t* rows_in, const int64_t* msg_comb,
                       const rails_sched_t* sched, const int64_t* rail_base, void* out,
                       int64_t out_cap, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (row_bytes < 16 || row_bytes % 16 || topo->chunk_bytes % 16 || rows_cap < 0)
    return fail(RAILS_EINVAL, "row_bytes and chunk_bytes must be multiples of 16");
  if (!y || !in_off || !rows_in || !msg_comb || !sched || !sched->full_base || !sched->rem_rail ||
      !sched->rem_off || !rail_base || (!out && out_cap > 0))
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(y, 16) || (out && !al(out, 16))) return fail(RAILS_EINVAL, "y/out must be 16-byte aligned");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_pack_combine(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, rows_cap,
                                     topo->chunk_bytes, y, in_off, rows_in, msg_comb, *sched,
                                     rail_base, out, out_cap, row_bytes),
                 "rails_pack_combine launch");
}

int rails_unpack_combine(const rails_topo_t* topo, const rails_shard_t* sh, int32_t T, int32_t k,
                         const int32_t* topk_inst, const int32_t* inst_to_gpu, int32_t n_inst,
                         const int32_t* row_rank, const float* w, const void* y,
                         int64_t rows_cap, const int64_t* in_off, const int64_t* msg_comb_all,
                         const rails_sched_t* sched_all, const int64_t* rail_base_all,
                         const void* comb_out, float* out, int64_t row_bytes, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_shard(topo, sh))) return rc;
  if (T < 1 || k < 1 || k > 32 || n_inst < 1) return fail(RAILS_EINVAL, "bad T, k or n_inst");
  if (row_bytes < 16 || row_bytes % 16 || topo->chunk_bytes % 16 || rows_cap < 0)
    return fail(RAILS_EINVAL, "row_bytes and chunk_bytes must be multiples of 16");
  if (!topk_inst || !inst_to_gpu || !row_rank || !w || !y || !in_off || !msg_comb_all ||
      !sched_all || !sched_all->full_base || !sched_all->rem_rail || !sched_all->rem_off ||
      !rail_base_all || !comb_out || !out)
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(y, 16) || !al(comb_out, 16) || !al(out, 16))
    return fail(RAILS_EINVAL, "y/comb_out/out must be 16-byte aligned");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_unpack_combine(c, sh->U, sh->nd, sh->d0, topo->M, topo->N, T, k,
                                       topo->chunk_bytes, topk_inst, inst_to_gpu, n_inst,
                                       row_rank, w, y, rows_cap, in_off, msg_comb_all, *sched_all,
                                       rail_base_all, comb_out, out, row_bytes),
                 "rails_unpack_combine launch");
}

int rails_ipc_alloc(int64_t bytes, void** dptr, void* handle) {
  if (bytes < 1 || !dptr || !handle) return fail(RAILS_EINVAL, "bad argument");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e != cudaSuccess) return cuda_rc(e, "cudaMalloc");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_rc(e, "cudaIpcGetMemHandle");
  }
  memcpy(handle, &h, sizeof(h));
  *dptr = p;
  return RAILS_OK;
}

int rails_ipc_open(const void* handle, void** dptr) {
  if (!handle || !dptr) return fail(RAILS_EINVAL, "bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_rc(e, "cudaIpcOpenMemHandle");
  *dptr = p;
  return RAILS_OK;
}

int rails_ipc_close(void* dptr) {
  if (!dptr) return fail(RAILS_EINVAL, "NULL pointer");
  return cuda_rc(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
}

int rails_ipc_free(void* dptr) {
  if (!dptr) return fail(RAILS_EINVAL, "NULL pointer");
  return cuda_rc(cudaFree(dptr), "cudaFree");
}

static int check_peer(const rails_peer_t* peer) {
  if (!peer) return fail(RAILS_EINVAL, "peer is NULL");
  if (peer->world < 1 || peer->world > RAILS_PEER_MAX || peer->rank < 0 ||
      peer->rank >= peer->world || peer->gen == 0)
    return fail(RAILS_EINVAL, "bad peer descriptor (rank %d, world %d, gen %u)", (int)peer->rank,
                (int)peer->world, (unsigned)peer->gen);
  for (int p = 0; p < peer->world; ++p)
    if (!peer->buf[p] || !al(peer->buf[p], 256))
      return fail(RAILS_EINVAL, "peer buffer %d NULL or not 256-byte aligned", p);
  return RAILS_OK;
}

int rails_peer_buffer_bytes(const rails_topo_t* topo, int32_t U, int32_t world, size_t* bytes) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if (U < 1 || world < 1 || world > RAILS_PEER_MAX || !bytes)
    return fail(RAILS_EINVAL, "bad arguments");
  *bytes = peer_buffer_bytes(U, world, RAILS_RED_SUM_LEN(topo->M, topo->N));
  return RAILS_OK;
}

int rails_eval_finalize_peer(const rails_topo_t* topo, int32_t U, int64_t* red_sum,
                             int64_t* red_max, const rails_peer_t* peer,
                             const rails_final_t* out, void* stream) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if (U < 1 || !red_sum || !red_max || !out) return fail(RAILS_EINVAL, "NULL argument");
  if ((rc = check_peer(peer))) return rc;
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_finalize_peer(c, U, topo->M, topo->N, topo->R2, &red_sum, &red_max, *peer,
                                      out, 1),
                 "rails_eval_finalize_peer launch");
}

int rails_eval_finalize_peer_local(const rails_topo_t* topo, int32_t U, int64_t* const* red_sum,
                                   int64_t* const* red_max, const rails_peer_t* peer,
                                   const rails_final_t* out, void* stream) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if ((rc = check_peer(peer))) return rc;
  if (U < 1 || !red_sum || !red_max || !out) return fail(RAILS_EINVAL, "NULL argument");
  for (int p = 0; p < peer->world; ++p)
    if (!red_sum[p] || !red_max[p]) return fail(RAILS_EINVAL, "rank %d: NULL red_sum/red_max", p);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_finalize_peer(c, U, topo->M, topo->N, topo->R2, red_sum, red_max, *peer,
                                      out, peer->world),
                 "rails_eval_finalize_peer_local launch");
}

int rails_owner_exchange_layout(const rails_topo_t* topo, int32_t U, int32_t world,
                                size_t* bytes, size_t* msg_offset) {
  int rc = check_topo(topo);
  if (rc) return rc;
  if (U < 1 || world < 1 || world > RAILS_PEER_MAX || !bytes || !msg_offset)
    return fail(RAILS_EINVAL, "bad arguments");
  size_t gf;
  owner_exchange_layout(U, world, topo->N, (long long)topo->M * topo->N, bytes, &gf, msg_offset);
  return RAILS_OK;
}

int rails_gather_rows_peer(const rails_topo_t* topo, int32_t U, int32_t g0, int32_t ng,
                           const int64_t* msg_loc, const rails_peer_t* peer, void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_peer(peer))) return rc;
  if (U < 1 || !msg_loc || g0 < 0 || ng < 1 || g0 + ng > topo->N)
    return fail(RAILS_EINVAL, "bad arguments");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_gather_rows_peer(c, U, topo->N, (long long)topo->M * topo->N, ng,
                                         &msg_loc, &g0, *peer, 1),
                 "rails_gather_rows_peer launch");
}

int rails_gather_rows_peer_local(const rails_topo_t* topo, int32_t U, int32_t ng,
                                 const int64_t* const* msg_loc, const rails_peer_t* peer,
                                 void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_peer(peer))) return rc;
  if (U < 1 || !msg_loc || ng < 1 || (long long)ng * peer->world != topo->N)
    return fail(RAILS_EINVAL, "need ng * world == N");
  int g0[RAILS_PEER_MAX];
  for (int p = 0; p < peer->world; ++p) {
    if (!msg_loc[p]) return fail(RAILS_EINVAL, "rank %d: NULL msg_loc", p);
    g0[p] = p * ng;
  }
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_gather_rows_peer(c, U, topo->N, (long long)topo->M * topo->N, ng, msg_loc,
                                         g0, *peer, peer->world),
                 "rails_gather_rows_peer_local launch");
}

int rails_peer_barrier(const rails_peer_t* peer, void* stream) {
  int rc = check_peer(peer);
  if (rc) return rc;
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_peer_barrier(c, *peer, 1), "rails_peer_barrier launch");
}

int rails_peer_barrier_local(const rails_peer_t* peer, void* stream) {
  int rc = check_peer(peer);
  if (rc) return rc;
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_peer_barrier(c, *peer, peer->world), "rails_peer_barrier_local launch");
}

static int check_fabric(const rails_topo_t* topo, const rails_fabric_t* fb) {
  if (!fb) return fail(RAILS_EINVAL, "fabric is NULL");
  if (fb->S < 1 || fb->S > 32) return fail(RAILS_EINVAL, "spines S=%d not in 1..32", (int)fb->S);
  if (!(fb->R1 > topo->R2)) return fail(RAILS_EINVAL, "R1 must exceed R2 (P:333)");
  if (!(fb->Rs > 0.0)) return fail(RAILS_EINVAL, "Rs must be > 0");
  const long long L = 2LL * topo->M * topo->N * topo->N + 2LL * topo->M * topo->N +
                      2LL * topo->N * fb->S;
  if (L > (1 << 20) || (long long)topo->M * topo->N * topo->M * topo->N > (1LL << 30))
    return fail(RAILS_ENOSPC, "fabric too large for the simulator");
  if (L * 8 > 200 * 1024)  // MinRTT's per-link backlog lives in shared memory
    return fail(RAILS_ENOSPC, "L=%lld links exceed the simulator's shared memory", L);
  return RAILS_OK;
}

int rails_flowsim_plan(const rails_topo_t* topo, const rails_fabric_t* fb, int32_t n_sim,
                       const int32_t* policy, const int64_t* msg, int64_t* totals,
                       void* stream) {
  int rc = check_topo(topo);
  if (rc || (rc = check_fabric(topo, fb))) return rc;
  if (n_sim < 1 || !policy || !msg || !totals) return fail(RAILS_EINVAL, "bad arguments");
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_flowsim_plan(c, *topo, *fb, n_sim, policy, msg, totals),
                 "rails_flowsim_plan launch");
}

int rails_flowsim_workspace(const rails_topo_t* topo, const rails_fabric_t* fb, int32_t n_sim,
                            int64_t max_flows, int64_t max_subflows, size_t* bytes) {
  int rc = check_topo(topo);
  if (rc || (rc = check_fabric(topo, fb))) return rc;
  if (n_sim < 1 || max_flows < 0 || max_subflows < 0 || !bytes)
    return fail(RAILS_EINVAL, "bad arguments");
  if (max_flows > (1LL << 28) || max_subflows > (1LL << 28))
    return fail(RAILS_ENOSPC, "too many flows per simulation");
  *bytes = flowsim_workspace_bytes(*topo, *fb, n_sim, max_flows, max_subflows);
  return RAILS_OK;
}

int rails_flowsim(const rails_topo_t* topo, const rails_fabric_t* fb, int32_t n_sim,
                  const int32_t* policy, const int64_t* msg, int64_t max_flows,
                  int64_t max_subflows, void* ws, size_t ws_bytes, double* msg_cct,
                  double* link_bytes, double* stats, void* stream) {
  size_t need = 0;
  int rc = rails_flowsim_workspace(topo, fb, n_sim, max_flows, max_subflows, &need);
  if (rc) return rc;
  if (!policy || !msg || !ws || !msg_cct || !link_bytes || !stats)
    return fail(RAILS_EINVAL, "NULL argument");
  if (!al(ws, 256)) return fail(RAILS_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < need) return fail(RAILS_ENOSPC, "workspace %zu < %zu bytes", ws_bytes, need);
  LaunchCtx c;
  if ((rc = ctx(stream, &c))) return rc;
  return cuda_rc(launch_flowsim(c, *topo, *fb, n_sim, policy, msg, max_flows, max_subflows, ws,
                                msg_cct, link_bytes, stats),
                 "rails_flowsim launch");
}

int rails_enable_peer_access(int32_t peer_device) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_rc(e, "cudaGetDevice");
  if (peer_device == dev) return RAILS_OK;
  int can = 0;
  e = cudaDeviceCanAccessPeer(&can, dev, peer_device);
  if (e != cudaSuccess) return cuda_rc(e, "cudaDeviceCanAccessPeer");
  if (!can) return fail(RAILS_ECUDA, "device %d cannot access device %d", dev, peer_device);
  e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RAILS_OK;
  }
  return cuda_rc(e, "cudaDeviceEnablePeerAccess");
}

}  // extern "C"
