/*
 * rails.h -- C ABI of the B200-native RailS hot path (arXiv 2510.19262).
 *
 * The library (paper_2510_19262_b200/librails.so) implements, in hand-written
 * sm_100a CUDA kernels, the per-node LPT spraying scheduler of RailS and the
 * payload packing it drives:
 *
 *   a1 rails_histogram      MoE top-k routing -> per-node D^(1) send histogram
 *   a2-a4 rails_lpt_schedule chunking, size-descending sort, greedy LPT on N rails
 *   a5 rails_eval/_finalize per-rail send/receive loads, completion time, T*,
 *                           bus bandwidth, MSE, ECMP-hash baseline
 *   a7 rails_pack           token rows -> rail-ordered send buffers
 *
 * Citations: P:n = PAPER.md line n; R#n = reading n of DESIGN.md section 3.
 *
 * Conventions (all entry points):
 *  - Array arguments are DEVICE pointers owned by the caller (e.g. torch tensors);
 *    the library never allocates, frees or retains them.  Struct arguments
 *    (rails_topo_t etc.) are HOST pointers read during the call only.
 *  - Every compute call is asynchronous on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and returns after enqueueing.
 *  - Return value: RAILS_OK or a negative code.  Argument errors are detected on
 *    the host before anything is enqueued (nothing is written).  Errors that
 *    depend on device data (out-of-range routing ids, undersized output buffers)
 *    are recorded in a device-side flag; the affected items are skipped, and
 *    rails_check() reports the first such error after synchronising.
 *  - rails_last_error() returns a thread-local message for the last failure.
 *  - No exceptions cross the ABI; calls on distinct streams may run concurrently
 *    (the device error flag is process-wide; see rails_check).
 *
 * Index notation: M nodes (domains), N rails = GPUs = NICs
 * per node, G = M*N global GPUs, h = f*N + m a global destination
 * GPU on node f, g a local source GPU, U units (all-to-all rounds, R#6).
 * A call covers the source nodes d0 .. d0+nd-1 of U units; arrays indexed by
 * source node use the LOCAL node index dl = d - d0, outermost dims [U][nd].
 */
#ifndef RAILS_H
#define RAILS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    RAILS_OK = 0,
    RAILS_EINVAL = -1,    /* bad argument (null pointer, size, alignment, topology) */
    RAILS_ERANGE = -2,    /* routing id / LUT value / negative byte count out of range */
    RAILS_ENOSPC = -3,    /* workspace or output buffer too small, or size limit hit */
    RAILS_EOVERFLOW = -4, /* a load would overflow int64 */
    RAILS_ECUDA = -5,     /* CUDA launch or runtime failure (see rails_last_error) */
    RAILS_ETIMEDOUT = -6  /* a peer rank of a peer-memory exchange never arrived */
};

/* Topology and method parameters -- the paper's problem statement (section 4.1). */
typedef struct {
    int32_t M;            /* nodes (computing domains), >= 2   */
    int32_t N;            /* rails = GPUs = NICs per node, 1..32 */
    int64_t chunk_bytes;  /* C: fixed chunk size, 1 .. 2^31   */
    double R2;            /* inter-domain rate per rail and direction, B/s, > 0 */
    double R1;            /* intra-domain rate; 0 = unspecified, else must be > R2 */
    uint64_t ecmp_seed;   /* seed of the ECMP-hash baseline (R#14)   */
} rails_topo_t;

/* Which (unit, source node) block a call covers. */
typedef struct {
    int32_t U;   /* units (all-to-all rounds) in the call, >= 1   (R#6) */
    int32_t d0;  /* first source node held by the caller, >= 0          */
    int32_t nd;  /* number of source nodes held, >= 1, d0 + nd <= M     */
} rails_shard_t;

/* ------------------------------------------------------------------ a1 */
/* Per-node send histogram (D^(1) row block; Alg. 1 "Select input slices
 * for local experts according to Gate and E") with the stable in-bucket
 * rank the pack needs (R#18).
 *   topk_inst  int32 [U][nd][N][T][k]  expert-instance id of slot s of token t of
 *              local GPU g (values in [0, n_inst));
 *   inst_to_gpu int32 [n_inst]         instance -> global destination GPU in [0, G);
 *   row_bytes  payload bytes per token row (RB), >= 1;
 *   counts     int32 [U][nd][N][G]     number of (t,s) of GPU g routed to GPU h,
 *              intra-node included (R#2);
 *   msg_bytes  int64 [U][nd][N][G]     counts * RB for remote h, 0 when h is on the
 *              source node (R#2);
 *   row_rank   int32 [U][nd][N][T][k]  number of earlier (t',s') (in (t,s) order)
 *              of the same GPU g with the same destination h; may be NULL.
 *   T, k       tokens per GPU >= 1, slots per token 1..32, T*k <= 2^30 (else
 *              RAILS_EINVAL before any launch).
 * Out-of-range ids set RAILS_ERANGE in the device flag; such slots are skipped. */
int rails_histogram(const rails_topo_t* topo, const rails_shard_t* shard,
                    int32_t T, int32_t k, const int32_t* topk_inst,
                    const int32_t* inst_to_gpu, int32_t n_inst, int64_t row_bytes,
                    int32_t* counts, int64_t* msg_bytes, int32_t* row_rank,
                    void* stream);

/* ------------------------------------------------------------------ a2-a4 */
/* Compact LPT schedule of every (unit, node).  Chunking (R#3): message
 * B = msg_bytes[u][dl][g][h] is cut into floor(B/C) full chunks and one remainder
 * chunk of B mod C bytes when nonzero.  Sort (Alg. 2 step 2): size
 * descending, ties by (g, h, chunk index) ascending (R#4).  Assignment (Alg. 2
 * step 3): LoadState[0..N) = 0; each chunk goes to the lowest-index
 * argmin rail (R#5) at byte offset LoadState[j*] (R#19); LoadState[j*] += size.
 * Because every full chunk is larger than every remainder and full chunks come in
 * (g,h,c) order, the i-th full chunk of a node (i = full_base[g][h] + c) lands on
 * rail i mod N at offset floor(i/N)*C; remainders are recorded per message.
 *   full_base  int64 [U][nd][N][G]  full chunks of the node emitted before (g,h);
 *   rem_rail   int8  [U][nd][N][G]  rail of the remainder chunk, -1 if none;
 *   rem_off    int64 [U][nd][N][G]  its byte offset in the rail buffer, 0 if none;
 *   send_load  int64 [U][nd][N]     final LoadState (= S[d][.], Eq. 4);
 *   n_full     int64 [U][nd]        number of full chunks of the node;
 *   n_rem      int32 [U][nd]        number of remainder chunks of the node.     */
typedef struct {
    int64_t* full_base;
    int8_t* rem_rail;
    int64_t* rem_off;
    int64_t* send_load;
    int64_t* n_full;
    int32_t* n_rem;
} rails_sched_t;

/* Device workspace (bytes) rails_lpt_schedule / rails_schedule_eval need for this
 * topology/shard.  Zero-fill it once before its first use (rails_schedule_eval). */
int rails_schedule_workspace(const rails_topo_t* topo, const rails_shard_t* shard,
                             size_t* workspace_bytes);

/* msg_bytes int64 [U][nd][N][G] (>= 0; negative values flag RAILS_ERANGE and
 * count as 0).  workspace: device buffer of at least rails_schedule_workspace()
 * bytes, 256-byte aligned, not used concurrently by another call. */
int rails_lpt_schedule(const rails_topo_t* topo, const rails_shard_t* shard,
                       const int64_t* msg_bytes, const rails_sched_t* out,
                       void* workspace, size_t workspace_bytes, void* stream);

/* NEXT f2 -- QP map (Alg. 2 step 4: "select port p from NIC j* by
 * round-robin; map (j*, p) to a QP"; R#34).  Same as rails_lpt_schedule (same
 * outputs, same workspace) plus the QP index of every remainder chunk: per rail,
 * chunks take QP indices round-robin over qps_per_rail in assignment (Step 3)
 * order, one counter per rail and (unit, node) round.  Because full chunks are
 * assigned first and in emission order, the i-th full chunk of a node
 * (i = full_base[g][h] + c) is the floor(i/N)-th chunk of rail i mod N and gets
 * QP floor(i/N) mod qps_per_rail (closed form, not stored).
 *   qps_per_rail  >= 1 (ports x QPs per port; the paper uses up to 256);
 *   rem_qp        int32 [U][nd][N][G]  QP of the message's remainder chunk, -1 if
 *                 none.  Errors: RAILS_EINVAL for qps_per_rail < 1 or NULL rem_qp. */
int rails_lpt_schedule_qp(const rails_topo_t* topo, const rails_shard_t* shard,
                          const int64_t* msg_bytes, const rails_sched_t* out,
                          int32_t qps_per_rail, int32_t* rem_qp,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Generic atomic-flow LPT ("small application-layer messages" P:603):
 * n_seg independent flow sets, set s = flows seg_off[s] .. seg_off[s+1]-1
 * (seg_off: device int64 [n_seg+1], non-decreasing, seg_off[0] = 0, last = F).
 * Order within a set: weight descending, then flow index ascending; each flow to
 * the lowest-index argmin rail.  w int64 [F] >= 0; rail int8-range int32 [F];
 * off int64 [F] (LoadState before the update); load int64 [n_seg][N]. */
int rails_assign_workspace(int32_t n_seg, int64_t F, size_t* workspace_bytes);
int rails_lpt_assign(int32_t N, int32_t n_seg, const int64_t* seg_off, int64_t F,
                     const int64_t* w, int32_t* rail, int64_t* off, int64_t* load,
                     void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ a5 */
/* Loads and balance of the shard's nodes plus reduction buffers for the global
 * quantities.  Load model (R#7): a chunk of node d on rail j bound for node
 * f = h/N adds to S[d][j] (Eq. 4) and R[f][j] (Eq. 5).  Two baselines on the same
 * load model:
 *   ECMP (R#13, R#14): each whole message (d,g,h) goes on rail ecmp(d*N+g, h);
 *   uniform (Theorem 3's continuous optimum P* = 1/N; R#41): each
 *     message of B bytes is split over all N rails, rail j taking floor(B/N) bytes
 *     plus one more when j < B mod N.
 *   S, S_e, S_u int64 [U][nd][N]  send loads (LPT, ECMP, uniform) of the shard's nodes;
 *   mse, nmse double [U][nd]     Eq. 6 of S[d][.] about its mean, exact
 *                                form sum_j (N*S_j - sum S)^2 / N^3 (R#11); nMSE =
 *                                mse / (sum S)^2, 0 if sum S = 0 (R#12);
 *   red_sum   int64 [U][RAILS_RED_SUM_LEN(M,N)]  PARTIAL sums over the shard's
 *             nodes, layout: R[M][N], R_e[M][N], R_u[M][N], colsum[M] (bytes into
 *             node f), total, total_e.  Overwritten by the call.
 *   red_max   int64 [U][RAILS_RED_MAX_LEN]  PARTIAL maxima: max S, max S_e, max row
 *             sum (bytes out of one node), max S_u.
 * With the nodes of a unit split over ranks, all-reduce red_sum (SUM) and
 * red_max (MAX) across ranks before rails_eval_finalize (a6). */
#define RAILS_RED_SUM_LEN(M, N) (3 * (int64_t)(M) * (int64_t)(N) + (int64_t)(M) + 2)
#define RAILS_RED_MAX_LEN 4
typedef struct {
    int64_t* S;
    int64_t* S_e;
    int64_t* S_u;
    double* mse;
    double* nmse;
    int64_t* red_sum;
    int64_t* red_max;
} rails_eval_t;

int rails_eval(const rails_topo_t* topo, const rails_shard_t* shard,
               const int64_t* msg_bytes, const rails_sched_t* sched,
               const rails_eval_t* out, void* stream);

/* Per-unit results from fully reduced red_sum / red_max ([U][...] as above):
 *   maxload   = max(max S, max R)        (most loaded NIC, send or receive)
 *   T         = maxload / R2             (R#8)
 *   total     = inter-node bytes;  busbw = total / T, 0 if total = 0   (R#10, R#40)
 *   rowmax, colmax = max row / column sum of D^(2) (Eq. 1);
 *   T_star    = max(rowmax, colmax) / (N * R2)   (Thm 2 + Thm 3)
 *   *_e       = the same for the ECMP-hash baseline;
 *   *_u       = the same for the uniform split (R#41; T_u >= T_star, equal when
 *               every message is a multiple of N bytes: Theorem 3).
 * All outputs are device arrays of length U (int64 or double); any may be NULL. */
typedef struct {
    int64_t* maxload;
    int64_t* maxload_e;
    int64_t* maxload_u;
    int64_t* total;
    int64_t* rowmax;
    int64_t* colmax;
    double* T;
    double* T_e;
    double* T_u;
    double* T_star;
    double* busbw;
    double* busbw_e;
    double* busbw_u;
} rails_final_t;

int rails_eval_finalize(const rails_topo_t* topo, int32_t U, const int64_t* red_sum,
                        const int64_t* red_max, const rails_final_t* out, void* stream);

/* a2-a5 fused (the hot path): ONE kernel computes the compact LPT schedule
 * (exactly as rails_lpt_schedule), the evaluation of the shard's nodes (exactly as
 * rails_eval: S, S_e, S_u, mse, nmse, partial red_sum / red_max) and, optionally,
 * the per-unit finalize and the rail offsets:
 *   final      NULL, or the rails_eval_finalize outputs -- only when the shard holds
 *              every node of its units (d0 = 0, nd = M); with nodes split over ranks
 *              pass NULL and finalize after the a6 exchange;
 *   rail_base, rail_total  NULL, or the rails_rail_offsets outputs.
 * workspace: rails_schedule_workspace() bytes, zero-filled before the FIRST call
 * (the kernel keeps per-unit accumulators and arrival counters there and leaves them
 * zeroed after every call).  Falls back to two launches (schedule, then eval) when
 * N*M*N exceeds the fused kernel's shared-memory limit; the results are identical. */
int rails_schedule_eval(const rails_topo_t* topo, const rails_shard_t* shard,
                        const int64_t* msg_bytes, const rails_sched_t* sched,
                        const rails_eval_t* eval, const rails_final_t* final,
                        int64_t* rail_base, int64_t* rail_total, void* workspace,
                        size_t workspace_bytes, void* stream);

/* a1-a5, the dispatch hot path in one call: rails_histogram followed by
 * rails_schedule_eval on the same stream (the schedule kernel is launched with
 * programmatic dependent launch, so it is scheduled while the histogram runs).
 * Arguments and outputs are exactly those of the two calls (same workspace contract
 * as rails_schedule_eval). */
int rails_histogram_schedule_eval(const rails_topo_t* topo, const rails_shard_t* shard,
                                  int32_t T, int32_t k, const int32_t* topk_inst,
                                  const int32_t* inst_to_gpu, int32_t n_inst, int64_t row_bytes,
                                  int32_t* counts, int64_t* msg_bytes, int32_t* row_rank,
                                  const rails_sched_t* sched, const rails_eval_t* eval,
                                  const rails_final_t* final, int64_t* rail_base,
                                  int64_t* rail_total, void* workspace, size_t workspace_bytes,
                                  void* stream);


/* a6 fused with the finalize over NVLink peer memory (one process per GPU of a
 * box): every rank pushes its partial red_sum / red_max of each unit into every
 * rank's exchange buffer (remote stores through CUDA-IPC mappings), publishes a
 * per-(unit, rank) flag with a system-scope release, waits for all ranks' flags,
 * sums / maxes the partials (written back into red_sum / red_max, as an
 * all-reduce would) and finalizes -- one kernel, no NCCL call.
 *   buf[p]  rank p's exchange buffer as mapped in this process (own included),
 *           rails_peer_buffer_bytes() bytes, zero-filled before the first call;
 *   gen     call number: >= 1, equal on all ranks, +1 per call (flags are waited on
 *           as ">= gen"; partials are double-buffered by gen parity, so back-to-back
 *           calls need no other synchronisation).
 * A rank that waits 30 s for a peer's flag gives up: it records RAILS_ETIMEDOUT in the
 * device flag (rails_check reports it) and finalizes what it has, which is then
 * undefined.  The exchange is out of step after a timeout (the call counters of the
 * ranks disagree): free and rebuild the exchange buffers on every rank before the
 * next call.  The call counter lives on the host, so a call captured into a CUDA
 * graph would replay a stale gen: never capture these calls. */
#define RAILS_PEER_MAX 8
typedef struct {
    int32_t rank;
    int32_t world;   /* 1 .. RAILS_PEER_MAX */
    uint32_t gen;
    void* buf[RAILS_PEER_MAX];
} rails_peer_t;
int rails_peer_buffer_bytes(const rails_topo_t* topo, int32_t U, int32_t world, size_t* bytes);
int rails_eval_finalize_peer(const rails_topo_t* topo, int32_t U, int64_t* red_sum,
                             int64_t* red_max, const rails_peer_t* peer,
                             const rails_final_t* out, void* stream);

/* The same exchange with EVERY rank driven by one process on one device (the
 * single-GPU tests; one process serving several ranks).  Rank p's partials are
 * red_sum[p] / red_max[p] and its outputs out[p] (host arrays of `world` entries);
 * peer->buf[p] is rank p's exchange buffer (plain device memory, all in this
 * process); peer->rank is ignored.  ONE cooperative launch plays every rank (CTA
 * (u, p) is rank p), so the ranks' flag waits run co-resident: separate spinning
 * launches or processes sharing one GPU are not guaranteed to run concurrently.
 * RAILS_ECUDA if U * world CTAs cannot be co-resident. */
int rails_eval_finalize_peer_local(const rails_topo_t* topo, int32_t U, int64_t* const* red_sum,
                                   int64_t* const* red_max, const rails_peer_t* peer,
                                   const rails_final_t* out, void* stream);

/* ------------------------------------------------------------------ a7 */
/* Rail buffer placement: rail_base int64 [U][nd][N] = exclusive prefix sum of
 * send_load in (u, dl, j) order, i.e. the byte offset of rail j of node d in one
 * contiguous output buffer; total int64 [1] = the buffer size needed. */
int rails_rail_offsets(const rails_topo_t* topo, const rails_shard_t* shard,
                       const int64_t* send_load, int64_t* rail_base, int64_t* total,
                       void* stream);

/* Scatter token rows into rail-ordered send buffers (R#18-R#20).  Message (g,h)
 * is the concatenation, in ascending (t,s), of the RB-byte rows x[g][t] of every
 * REMOTE slot routed to h; the copy with rank rho occupies message bytes
 * [rho*RB, (rho+1)*RB).  Chunk c of the message (bytes [c*C, c*C+size)) is
 * written to out + rail_base[u][dl][rail(c)] + off(c) with (rail, off) from the
 * compact schedule.  Each source row is read once.  Payload is opaque bytes.
 *   x         [U][nd][N][T][row_bytes] device bytes, 16-byte aligned;
 *   row_bytes multiple of 16; chunk_bytes multiple of 16;
 *   topk_inst, inst_to_gpu, row_rank, msg_bytes: as produced/consumed above;
 *   out       device buffer of out_cap bytes, 16-byte aligned.
 * A destination beyond out_cap sets RAILS_ENOSPC (that piece is skipped). */
int rails_pack(const rails_topo_t* topo, const rails_shard_t* shard, int32_t T,
               int32_t k, const void* x, const int32_t* topk_inst,
               const int32_t* inst_to_gpu, int32_t n_inst, const int32_t* row_rank,
               const int64_t* msg_bytes, int64_t row_bytes, const rails_sched_t* sched,
               const int64_t* rail_base, void* out, int64_t out_cap, void* stream);

/* ------------------------------------------------------------------ NEXT f1 */
/* Combine all-to-all (Alg. 1 step 4): expert outputs go back from
 * expert GPU h = f*N+m to the token's GPU a = d*N+g as a SECOND all-to-all round
 * with its own LoadState.  Readings R#28-R#31.
 *
 * rails_transpose_traffic: combine traffic msg_t[u][f][m][a] = msg[u][a/N][a%N][f*N+m]
 *   for every node (msg, msg_t: int64 [U][M][N][G]; R#28).  The combine schedule and
 *   evaluation are then rails_lpt_schedule / rails_eval on msg_t, unchanged. */
int rails_transpose_traffic(const rails_topo_t* topo, int32_t U, const int64_t* msg,
                            int64_t* msg_t, void* stream);

/* Expert-output buffer layout (R#29): GPU b holds the rows it received in dispatch,
 * message by message in ascending source GPU a, each in dispatch rank order.
 * counts: dispatch counts int32 [U][M][N][G] (all nodes); in_off int64 [U][G][G]:
 * in_off[u][b][a] = first row of message a in b's buffer; rows_in int64 [U][G]. */
int rails_recv_offsets(const rails_topo_t* topo, int32_t U, const int32_t* counts,
                       int64_t* in_off, int64_t* rows_in, void* stream);

/* Combine pack of the shard's SENDER nodes f (R#30): message (m, a) = rows
 * in_off[u][f*N+m][a] .. of y (bytes [U][nd][N][rows_cap][row_bytes]), chunked by
 * the combine schedule (msg_comb [U][nd][N][G], sched) into out at
 * rail_base[u][dl][j] + off (as rails_pack).  Intra-node messages are skipped. */
int rails_pack_combine(const rails_topo_t* topo, const rails_shard_t* shard, int64_t row_bytes,
                       int64_t rows_cap, const void* y, const int64_t* in_off,
                       const int64_t* rows_in, const int64_t* msg_comb,
                       const rails_sched_t* sched, const int64_t* rail_base, void* out,
                       int64_t out_cap, void* stream);

/* Unpack + top-k weighted combine on the shard's RECEIVER nodes d (R#31):
 *   out[u][dl][g][t][e] = sum_{s<k} w[t][s] * row(t,s)[e],  e < row_bytes/2 (bf16)
 * accumulated in fp32 in slot order, every product and sum rounded (no FMA).
 * row(t,s): expert h = inst_to_gpu[topk[t][s]] on node f; rank rho = row_rank[t][s];
 * f == d: y row in_off[u][h][a] + rho of GPU h (never railed); f != d: message
 * bytes [rho*RB, (rho+1)*RB) of combine message (h -> a), read from comb_out with
 * node f's combine schedule (msg_comb_all/sched_all/rail_base_all cover ALL M
 * sender nodes: [U][M][N][G] / [U][M][N]).  w: float [U][nd][N][T][k];
 * out: float [U][nd][N][T][row_bytes/2]. */
int rails_unpack_combine(const rails_topo_t* topo, const rails_shard_t* shard, int32_t T,
                         int32_t k, const int32_t* topk_inst, const int32_t* inst_to_gpu,
                         int32_t n_inst, const int32_t* row_rank, const float* w, const void* y,
                         int64_t rows_cap, const int64_t* in_off, const int64_t* msg_comb_all,
                         const rails_sched_t* sched_all, const int64_t* rail_base_all,
                         const void* comb_out, float* out, int64_t row_bytes, void* stream);

/* ------------------------------------------------------------------ NEXT f2 */
/* Rail-owner variant (one multi-GPU box = one RailS node): NIC j hangs off GPU j
 * (P:184), so rail j's send buffer lives in GPU j's HBM and traffic of GPU g on
 * rail j != g crosses the intra-domain network first.  A
 * process holding source GPUs g0 .. g0+ng-1 of each node histograms its own rows,
 * the node's msg_bytes rows are all-gathered (caller, NCCL), every process runs the
 * same node-wide rails_lpt_schedule, and rails_pack_owner writes each chunk piece
 * straight into the rail owner's buffer through peer-mapped pointers (NVLink /
 * NVSwitch): the intra-node hop is fused into the pack.
 *
 * rails_histogram_gpus: as rails_histogram for source GPUs g0..g0+ng-1 only;
 *   topk_inst/row_rank [U][nd][ng][T][k], counts/msg_bytes [U][nd][ng][G].        */
int rails_histogram_gpus(const rails_topo_t* topo, const rails_shard_t* shard, int32_t g0,
                         int32_t ng, int32_t T, int32_t k, const int32_t* topk_inst,
                         const int32_t* inst_to_gpu, int32_t n_inst, int64_t row_bytes,
                         int32_t* counts, int64_t* msg_bytes, int32_t* row_rank, void* stream);

/* rail_base int64 [U][nd][N]: offset of block (u, dl) inside RAIL j's own buffer
 * (exclusive prefix of send_load over (u, dl) for each j); rail_total int64 [N]:
 * bytes each rail buffer needs. */
int rails_rail_offsets_owner(const rails_topo_t* topo, const rails_shard_t* shard,
                             const int64_t* send_load, int64_t* rail_base, int64_t* rail_total,
                             void* stream);

/* Pack the rows of source GPUs g0..g0+ng-1 (x, topk_inst, row_rank in the local
 * [U][nd][ng][...] layout) into the rail buffers rail_ptr[j] (host array of N
 * device pointers, peer-mapped where rail j is owned by another GPU; each 16-byte
 * aligned, rail_cap[j] bytes, host array).  msg_bytes and sched are node-wide
 * ([U][nd][N][G]); a piece of chunk c on rail j goes to
 * rail_ptr[j] + rail_base[u][dl][j] + off(c).  Beyond rail_cap -> RAILS_ENOSPC. */
int rails_pack_owner(const rails_topo_t* topo, const rails_shard_t* shard, int32_t g0,
                     int32_t ng, int32_t T, int32_t k, const void* x, const int32_t* topk_inst,
                     const int32_t* inst_to_gpu, int32_t n_inst, const int32_t* row_rank,
                     const int64_t* msg_bytes, int64_t row_bytes, const rails_sched_t* sched,
                     const int64_t* rail_base, void* const* rail_ptr, const int64_t* rail_cap,
                     void* stream);

/* NVLink-native exchange of the rail-owner node (replaces NCCL in its step).
 * Each rank owns an exchange buffer (rails_owner_exchange_layout bytes, zero-filled
 * before first use, IPC-exported and mapped by every rank; rails_peer_t.buf[p] =
 * rank p's buffer as mapped here; gen as for rails_eval_finalize_peer):
 *   rails_gather_rows_peer: one kernel (one CTA per unit) stores this rank's
 *     msg_bytes rows (msg_loc [U][1][ng][G], source GPUs g0..g0+ng-1) into every
 *     rank's node-wide msg table at msg_offset ([U][1][N][G] int64), flags, and
 *     returns when all ranks' rows are in this rank's table (the schedule input);
 *   rails_peer_barrier: after rails_pack_owner, every rank's packed pieces are in
 *     their owners' buffers when the barrier kernel of every rank has completed.
 * A peer missing for 30 s sets RAILS_ETIMEDOUT in the device flag; the exchange must
 * then be rebuilt (as for rails_eval_finalize_peer).  Not graph-capturable (gen). */
int rails_owner_exchange_layout(const rails_topo_t* topo, int32_t U, int32_t world,
                                size_t* bytes, size_t* msg_offset);
int rails_gather_rows_peer(const rails_topo_t* topo, int32_t U, int32_t g0, int32_t ng,
                           const int64_t* msg_loc, const rails_peer_t* peer, void* stream);
int rails_peer_barrier(const rails_peer_t* peer, void* stream);
/* Both for every rank driven by one process on one device (as
 * rails_eval_finalize_peer_local): rank p holds source GPUs p*ng .. p*ng+ng-1
 * (ng * world == N), msg_loc[p] is its [U][1][ng][G] rows; one cooperative launch. */
int rails_gather_rows_peer_local(const rails_topo_t* topo, int32_t U, int32_t ng,
                                 const int64_t* const* msg_loc, const rails_peer_t* peer,
                                 void* stream);
int rails_peer_barrier_local(const rails_peer_t* peer, void* stream);

/* Inter-process rail buffers for rails_pack_owner (one process per GPU): the
 * owner allocates with rails_ipc_alloc (device memory of the current device, 256-B
 * aligned, plus a 64-byte cudaIpcMemHandle_t written to `handle`), ships the
 * handle to the other processes of the box, and each of them maps it with
 * rails_ipc_open while ITS OWN device is current (peer access enabled lazily), so
 * its kernels can store into the owner's HBM over NVLink.  rails_ipc_close unmaps
 * an opened buffer; rails_ipc_free releases an owned one. */
int rails_ipc_alloc(int64_t bytes, void** dptr, void* handle);
int rails_ipc_open(const void* handle, void** dptr);
int rails_ipc_close(void* dptr);
int rails_ipc_free(void* dptr);

/* Enable direct loads/stores from kernels on the current device to memory of
 * `peer_device` (cudaDeviceEnablePeerAccess; "already enabled" is not an error).
 * RAILS_ECUDA if the devices cannot reach each other. */
int rails_enable_peer_access(int32_t peer_device);

/* ------------------------------------------------------------------ NEXT f4 */
/* Fluid (flow-level) simulation of one all-to-all round per simulation (SPEC
 * flowsim S:464-537 in place of the paper's Mininet testbed), with the
 * paper's comparison policies and its metrics (CCT avg/p80/p95/p99,
 * BusBw).  Readings R#35-R#39.
 *
 * Fabric (R#35): topo gives M, N, R2 (NIC<->leaf rate), chunk_bytes C and the
 * ECMP seed; the fabric adds S spines, the intra-domain GPU<->NIC rate R1 (> R2)
 * and the leaf<->spine rate Rs.  Directed links, in this order:
 *   GPU_UP[M][N][N] (g -> NIC n, R1), NIC_UP[M][N] (R2), LEAF_SPINE[N][S] (Rs),
 *   SPINE_LEAF[S][N] (Rs), NIC_DOWN[M][N] (R2), GPU_DOWN[M][N][N] (NIC n -> m, R1);
 *   L = 2MN^2 + 2MN + 2NS.
 * Policies (R#36): LPT chunks of the node's LPT schedule on rail paths; UNIFORM
 * N flows of B/N per message (Theorem 3's P* = 1/N); ECMP whole message on one
 * hashed spine path; REPS whole message split evenly over every spine path;
 * MINRTT LPT-sized chunks each on the least backlogged spine path at t = 0;
 * PLB as ECMP, re-hashing the spine of a flow whose rate a spine link set, at a
 * completion event (not at two consecutive events).  Unknown policy values set
 * RAILS_ERANGE and give no flows.
 * Rates are max-min fair (progressive filling, R#37); a flow completes at the
 * event where its remaining / rate reaches the step (R#38). */
enum {
    RAILS_POL_LPT = 0,
    RAILS_POL_UNIFORM = 1,
    RAILS_POL_ECMP = 2,
    RAILS_POL_REPS = 3,
    RAILS_POL_MINRTT = 4,
    RAILS_POL_PLB = 5
};
#define RAILS_FS_NSTATS 10
typedef struct {
    int32_t S;    /* spines, >= 1 (default N) */
    double R1;    /* intra-domain GPU<->NIC rate, B/s, > R2 (default 8*R2) */
    double Rs;    /* leaf<->spine rate, B/s, > 0 (default M*R2/S) */
} rails_fabric_t;

/* Flows and subflows each simulation makes: totals int64 [n_sim][2] (device).
 *   policy int32 [n_sim] (device), msg int64 [n_sim][M][N][G] (device, >= 0, zero
 *   for intra-node pairs).  Use the maxima to size the workspace. */
int rails_flowsim_plan(const rails_topo_t* topo, const rails_fabric_t* fabric, int32_t n_sim,
                       const int32_t* policy, const int64_t* msg, int64_t* totals,
                       void* stream);
int rails_flowsim_workspace(const rails_topo_t* topo, const rails_fabric_t* fabric,
                            int32_t n_sim, int64_t max_flows, int64_t max_subflows,
                            size_t* workspace_bytes);
/* Run n_sim simulations, one CTA each.  Outputs (device):
 *   msg_cct    double [n_sim][M][N][G]  completion time (s) of each message, 0 if none;
 *   link_bytes double [n_sim][L]        bytes carried per directed link;
 *   stats      double [n_sim][RAILS_FS_NSTATS]  T, total bytes, busbw = total / T,
 *              CCT mean, p80, p95, p99 (nearest rank over messages with bytes),
 *              max over events of the largest domain-pair rate / (N*R2) (Theorem 1),
 *              events, flows.
 * A simulation whose flows exceed max_flows / max_subflows sets RAILS_ENOSPC and
 * leaves its outputs unwritten. */
int rails_flowsim(const rails_topo_t* topo, const rails_fabric_t* fabric, int32_t n_sim,
                  const int32_t* policy, const int64_t* msg, int64_t max_flows,
                  int64_t max_subflows, void* workspace, size_t workspace_bytes,
                  double* msg_cct, double* link_bytes, double* stats, void* stream);

/* ------------------------------------------------------------------ misc */
/* Synchronise `stream`, then return (and clear) the first device-side error
 * recorded since the last check: RAILS_OK, RAILS_ERANGE, RAILS_ENOSPC,
 * RAILS_EOVERFLOW or RAILS_ETIMEDOUT; RAILS_ECUDA if the stream reports a CUDA
 * error. */
int rails_check(void* stream);

/* Thread-local description of the last failed call ("" if none). */
const char* rails_last_error(void);

/* Number of kernel launches this thread's calls have enqueued since the last
 * reset (reset = nonzero).  For benchmark accounting. */
int64_t rails_launch_count(int32_t reset);

/* ABI version (major*100 + minor). */
int32_t rails_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RAILS_H */
