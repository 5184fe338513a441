/*
 * slf_lce.h — C ABI of libslf_lce.so: the fused linear-cross-entropy (LCE) hot
 * path on B200 (sm_100a).
 *
 * The operation (§3.3 "Optimized Triton Kernels"): the fused
 * LinearCrossEntropy kernel "fuses the projection and loss calculation,
 * computing gradients in small chunks to avoid materializing the full logits
 * tensor", "without sacrificing accuracy" against the "torch standard method"
 * (Fig. fig:lce caption).  With
 *
 *   X = hidden [N, H] bf16 row-major, W = LM-head weight [V, H] bf16 row-major,
 *   t = targets [N] int32, Z = X W^T (never stored),
 *   lse_i = log sum_v exp Z_iv, valid_i = (t_i != ignore_index),
 *   l_i = valid_i ? lse_i - Z_{i,t_i} : 0,
 *   coef_i = scale * valid_i * (1/n_valid if MEAN else 1),
 *   G = coef (softmax(Z) - onehot(t)),
 *
 * the library returns loss (fp32; sum, mean or per-row), dhidden = G W and
 * dweight = G^T X (bf16), with device memory for intermediates bounded by the
 * caller-provided workspace (no N x V buffer exists).  Readings of the paper
 * (ignore_index equality, MEAN with n_valid = 0 -> 0, `scale` scales gradients
 * only, out-of-range targets are a data error) are DESIGN.md R1-R9.
 *
 * Conventions for every entry point
 *  - All pointers except `loss_out` / host outputs documented as host are
 *    DEVICE pointers to caller-owned memory (allocated e.g. by torch).  The
 *    library never allocates device memory; its only device scratch is
 *    `workspace`.  Device pointers must be 16-byte aligned (SLF_ERR_ALIGN).
 *  - Calls enqueue work on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and return without synchronising.  Argument and launch errors are
 *    synchronous return codes; the message is in slf_last_error_string().
 *    Data errors (a valid target outside [0, V_global)) are asynchronous: the
 *    loss becomes NaN and slf_lce_status() reports the count.
 *  - No global mutable state except a thread-local last-error string, a
 *    per-device attribute cache, a per-device 8 MB pinned HOST ring that
 *    stages the per-call tile tables (allocated on first use, never freed),
 *    the host-input call's per-device copy stream, events and staging-buffer
 *    release events, and memoised tile tables; communicators (slf_comm) and
 *    Layer-Adam handles (slf_adam.h) are explicit objects.  Calls on different
 *    streams are independent provided they use different workspaces.  The
 *    calls are not CUDA-graph-capture safe (they copy tile tables from that
 *    host ring).
 *  - Requirements: H % 8 == 0 (16-byte TMA row strides), N >= 1, V_local >= 1,
 *    an sm_100 device (SLF_ERR_UNSUPPORTED otherwise).
 */
#ifndef SLF_LCE_H_
#define SLF_LCE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int slf_status;
#define SLF_OK 0
#define SLF_ERR_ARG 1           /* null required pointer, bad size or enum */
#define SLF_ERR_ALIGN 2         /* a device pointer is not 16-byte aligned */
#define SLF_ERR_WORKSPACE 3     /* workspace_bytes smaller than required   */
#define SLF_ERR_CUDA 4          /* CUDA launch / driver error              */
#define SLF_ERR_UNSUPPORTED 5   /* not an sm_100 device                    */
#define SLF_ERR_UNIMPLEMENTED 6 /* requested schedule not built yet        */
#define SLF_ERR_COMM 7          /* collective transport (NCCL / callback)  */

typedef enum { SLF_SUM = 0, SLF_MEAN = 1, SLF_NONE = 2 } slf_reduction;

/* Schedules.  R: forward statistics pass over all vocabulary
 * tiles, then recompute the logits tile by tile in backward (8·N·H·V tensor
 * FLOPs; the only schedule of the split / shard entry points).  S (fused call
 * only): per row chunk, one forward pass whose epilogue stashes
 * p~ = bf16(exp(z - m_tile)), then dX and dW straight from the stash, the
 * one-hot term applied exactly (6·N·H·V).  AUTO: S when its plan fits the
 * budget, else R; slf_lce_workspace_bytes(AUTO) is enough for every entry
 * point. */
typedef enum { SLF_SCHED_AUTO = 0, SLF_SCHED_R = 1, SLF_SCHED_S = 2 } slf_schedule;

/* Per-row statistics record ("RowStat", 16 bytes) exchanged between the
 * forward and backward halves: lse2 = lse * log2(e); coef as above;
 * tloc = t - vocab_start if the target lies in this vocab shard else -1;
 * valid = 1 if t != ignore_index. */
typedef struct {
  float lse2;
  float coef;
  int32_t tloc;
  int32_t valid;
} slf_rowstat;

/* Per-row shard statistics ("ShardStat", 16 bytes) for vocab-parallel use:
 * m = max_v Z_iv and s = sum_v exp(Z_iv - m) over this shard's columns,
 * zt = Z_{i,t_i} if t_i is in this shard else 0, hit = 1.0f if it is. */
typedef struct {
  float m;
  float s;
  float zt;
  float hit;
} slf_shardstat;

/* Library version (major*10000 + minor*100 + patch). */
int slf_lce_version(void);

/* Message for the last error on this thread ("" if none).  Host string owned
 * by the library, valid until the next call on this thread. */
const char* slf_last_error_string(void);

/* Workspace bytes the planner needs for a problem of this shape when it must
 * stay within `budget_bytes` (0 = default budget: max(5% of N*V_local*2, 16 MiB),
 * the BASELINE.json "extra memory <= 5% of the materialised-logits footprint"
 * target).  Returns 0 if no plan fits the budget or the shape is invalid. */
size_t slf_lce_workspace_bytes(int64_t N, int64_t H, int64_t V_local, int schedule, size_t budget_bytes);

/* Writes a one-line description of the plan (schedule, row block, vocab chunk,
 * launches) into the HOST buffer `out` of `cap` bytes.  Returns SLF_OK or
 * SLF_ERR_ARG / SLF_ERR_WORKSPACE. */
slf_status slf_lce_plan_describe(int64_t N, int64_t H, int64_t V_local, int schedule, size_t budget_bytes,
                                 char* out, size_t cap);

/* The whole hot path on one GPU (V_local = V_global, vocab_start = 0):
 * forward statistics, loss, and both gradients.
 *   hidden   [N, H] bf16, row-major (ld = H)               (read)
 *   weight   [V, H] bf16, row-major (ld = H)               (read)
 *   targets  [N] int32                                     (read)
 *   loss_out DEVICE fp32: [1] for SUM/MEAN, [N] for NONE   (written)
 *   dhidden  [N, H] bf16 (may be NULL to skip)             (overwritten)
 *   dweight  [V, H] bf16 (may be NULL to skip)             (overwritten)
 *   workspace, workspace_bytes: >= slf_lce_workspace_bytes(N,H,V,schedule,budget)
 * Gradients are those of scale*loss (SUM/MEAN) or of scale*sum_i l_i (NONE).
 * Rows with t_i == ignore_index get dhidden rows of exactly +0.0.
 * Under schedule S the rows of dhidden that are not written yet also serve as stash scratch
 * (extended row chunks): dhidden must not alias hidden, weight or the workspace,
 * and its contents before the call are irrelevant. */
slf_status slf_lce_fwd_bwd(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                           int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                           void* dhidden, void* dweight, void* workspace, size_t workspace_bytes, int schedule,
                           size_t budget_bytes, void* stream);

/* slf_lce_fwd_bwd with flags (gradient accumulation across micro-batches):
 *   SLF_FLAG_ACCUMULATE_DW: dweight += dL/dW instead of = (each partial is rounded to bf16 and
 *   added to dweight by the L2: TMA reduce-add).
 * flags = 0 is exactly slf_lce_fwd_bwd. */
#define SLF_FLAG_ACCUMULATE_DW 1u
slf_status slf_lce_fwd_bwd_ex(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                              int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                              void* dhidden, void* dweight, void* workspace, size_t workspace_bytes, int schedule,
                              size_t budget_bytes, uint32_t flags, void* stream);

/* The fused call with HOST inputs and loss (the path as a training step sees it:
 * the batch arrives from the host).  Per step it copies targets, then hidden row chunk by row chunk
 * on an internal copy stream, and the schedule-S chunk c waits only for its own rows, so the
 * host->device transfer overlaps the GEMMs; the loss is copied back at the end.
 *   hidden_host  [N, H] bf16 HOST (pinned for overlap; pageable works, serialised)   (read)
 *   targets_host [N] int32 HOST                                                      (read)
 *   loss_host    HOST fp32 [1] (SUM/MEAN) or [N] (NONE); valid after `stream` syncs  (written)
 *   weight, dhidden, dweight, workspace: as slf_lce_fwd_bwd_ex (DEVICE)
 *   hidden_dev [N, H] bf16, targets_dev [N] int32, loss_dev fp32 [1] / [N]: caller-owned DEVICE
 *       staging buffers (the library allocates no device memory); overwritten.
 * The copies into a staging buffer start once the last call that used the same hidden_dev has
 * finished with it (tracked per staging pointer; the first time: once the work already enqueued
 * on `stream` has completed), so alternating two staging sets lets step k+1's input copy run
 * under step k.  Schedule R (when S does not fit) copies
 * everything up front.  Not thread-safe against another host call on the same device at once
 * (the copy stream and its events are per device). */
slf_status slf_lce_fwd_bwd_host(const void* hidden_host, const void* weight, const int32_t* targets_host, int64_t N,
                                int64_t H, int64_t V, int32_t ignore_index, int reduction, float scale,
                                float* loss_host, void* dhidden, void* dweight, void* hidden_dev,
                                int32_t* targets_dev, float* loss_dev, void* workspace, size_t workspace_bytes,
                                int schedule, size_t budget_bytes, uint32_t flags, void* stream);

/* Forward half (schedule R split; also the vocab-shard seam).  Computes the
 * loss and the RowStat array [N] (16 B/row, DEVICE, caller-owned) that
 * slf_lce_bwd consumes.  `scale` enters coef only.  Single GPU form. */
slf_status slf_lce_fwd(const void* hidden, const void* weight, const int32_t* targets, int64_t N, int64_t H,
                       int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                       slf_rowstat* rowstat, void* workspace, size_t workspace_bytes, size_t budget_bytes,
                       void* stream);

/* Vocab-shard forward, part 1: this shard's per-row statistics.
 *   weight_shard [V_local, H] bf16 = rows [vocab_start, vocab_start+V_local) of W
 *   shardstat    [N] slf_shardstat (DEVICE, written)
 * No loss is formed; gather the g shards' arrays (e.g. NCCL all-gather, rank
 * order) and call slf_lce_stats_combine. */
slf_status slf_lce_fwd_shard_stats(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                                   int64_t H, int64_t V_local, int64_t vocab_start, int32_t ignore_index,
                                   slf_shardstat* shardstat, void* workspace, size_t workspace_bytes,
                                   size_t budget_bytes, void* stream);

/* Vocab-shard forward, part 2: merge g shards' statistics (`stats` is
 * [g][N] slf_shardstat, DEVICE, shard order) into the loss and this shard's
 * RowStat (tloc relative to vocab_start, V_local wide).  Targets are range
 * checked against V_global.  Deterministic (fixed shard order). */
slf_status slf_lce_stats_combine(const slf_shardstat* stats, int g, const int32_t* targets, int64_t N,
                                 int64_t vocab_start, int64_t V_local, int64_t V_global, int32_t ignore_index,
                                 int reduction, float scale, float* loss_out, slf_rowstat* rowstat,
                                 void* workspace, size_t workspace_bytes, void* stream);

/* Backward half: recompute the logits tile by tile, form
 * G = grad_scale * coef * (softmax - onehot) in fp32, round to bf16, and feed
 * it to the dweight and dhidden GEMMs.
 *   rowstat  [N] from slf_lce_fwd / slf_lce_stats_combine (read)
 *   dhidden  [N, H]: bf16 if dhidden_fp32 == 0, else fp32 (the shard partial
 *            to be summed across shards)               (overwritten; may be NULL)
 *   dweight  [V_local, H] bf16                          (overwritten; may be NULL)
 * grad_scale multiplies coef (the autograd grad_output). */
slf_status slf_lce_bwd(const void* hidden, const void* weight, const int32_t* targets, const slf_rowstat* rowstat,
                       int64_t N, int64_t H, int64_t V_local, float grad_scale, void* dhidden, int dhidden_fp32,
                       void* dweight, void* workspace, size_t workspace_bytes, size_t budget_bytes,
                       void* stream);

/* ---- schedule S split for vocab shards ----
 * Each rank owns W rows [vocab_start, vocab_start + V_local).  Per step:
 *   slf_lce_s_begin                                  targets scan + this shard's target CSR
 *   for chunk c in [0, n_chunks):   (rows [c*chunk_rows, min(N, (c+1)*chunk_rows)))
 *     slf_lce_s_chunk_stats(c) -> shardstat_chunk [rows_c]      stash GEMM + local row merge
 *     caller: gather the g shards' shardstat_chunk in rank order -> stats [g][rows_c]
 *     slf_lce_s_chunk_bwd(c, stats, g) -> dhidden rows of the chunk (fp32 partial: sum it across
 *         shards, then slf_lce_dx_finalize those rows with the chunk's RowStat), dW (+)=
 *   slf_lce_s_end                                    one-hot dW correction, loss
 * The same workspace must be used for all calls of a step; chunk_rows / n_chunks come from
 * slf_lce_s_plan for the same (N, H, V_local, budget).  Rowstats of the step are kept in the
 * workspace; slf_lce_s_rowstat returns a device pointer to them (for slf_lce_dx_finalize). */
slf_status slf_lce_s_plan(int64_t N, int64_t H, int64_t V_local, size_t budget_bytes, int64_t* chunk_rows,
                          int64_t* n_chunks);
slf_status slf_lce_s_begin(const int32_t* targets, int64_t N, int64_t H, int64_t V_local, int64_t vocab_start,
                           int64_t V_global, int32_t ignore_index, int need_dweight, void* workspace,
                           size_t workspace_bytes, size_t budget_bytes, void* stream);
slf_status slf_lce_s_chunk_stats(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                                 int64_t H, int64_t V_local, int64_t vocab_start, int64_t V_global,
                                 int32_t ignore_index, int64_t chunk, slf_shardstat* shardstat_chunk, void* workspace,
                                 size_t workspace_bytes, size_t budget_bytes, void* stream);
/* dhidden_chunk: row 0 of the chunk's rows ([rows_c, H]; fp32 if dhidden_fp32 else bf16; may be
 * NULL); dweight: [V_local, H] bf16 (may be NULL; must be the same buffer for every chunk);
 * loss_rows: DEVICE fp32 [N] for SUM/MEAN may be NULL (kept in the workspace), for NONE the
 * caller's per-row loss buffer. */
slf_status slf_lce_s_chunk_bwd(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                               int64_t H, int64_t V_local, int64_t vocab_start, int64_t V_global,
                               int32_t ignore_index, int reduction, float scale, int64_t chunk,
                               const slf_shardstat* stats, int g, float* loss_rows, void* dhidden_chunk,
                               int dhidden_fp32, void* dweight, void* workspace, size_t workspace_bytes,
                               size_t budget_bytes, void* stream);
slf_status slf_lce_s_end(const void* hidden, int64_t N, int64_t H, int64_t V_local, int reduction, float scale,
                         float* loss_out, void* dweight, void* workspace, size_t workspace_bytes, size_t budget_bytes,
                         void* stream);
/* DEVICE pointer (in *out) to the step's RowStat array [N] inside `workspace` (schedule S). */
slf_status slf_lce_s_rowstat(int64_t N, int64_t H, int64_t V_local, size_t budget_bytes, void* workspace,
                             const slf_rowstat** out);

/* ---- vocab-sharded LCE in one call, collectives inside the library (SURVEY §8(b) "Comm", §8(e)) ----
 * BASELINE.json north_star: "the LM head is vocab-sharded (V/g rows per GPU): NCCL over NVLink
 * all-reduces the per-token (max, sum-exp, target-logit) triples in forward and dhidden in backward,
 * and dW stays local to its shard" — PAPER.md l.273's fused LCE split across the g GPUs of one box.
 *
 * A communicator (slf_comm) binds one process = one GPU = one rank.  Transports:
 *   slf_comm_init:           NCCL (loaded at run time: the libnccl.so.2 already in the process,
 *                            e.g. PyTorch's, else the system one; SLF_ERR_COMM if none).  Bootstrap:
 *                            rank 0 calls slf_comm_get_unique_id (128 HOST bytes) and the caller
 *                            ships them to every rank (e.g. torch.distributed broadcast).
 *   slf_comm_init_callbacks: caller-provided collectives (tests: gloo through host copies).  The
 *                            callbacks are invoked on the calling thread with the library's stream;
 *                            they must leave the result visible to later work on that stream
 *                            (e.g. synchronise it, copy, copy back) and return 0 on success.
 * The communicator keeps one internal CUDA stream and four events (NCCL transport); it must be
 * destroyed with slf_comm_destroy on the device it was created on.  Not thread-safe: one call at a
 * time per communicator. */
typedef struct slf_comm_s* slf_comm;
/* recv[r * bytes_per_rank ...] = rank r's send[0 .. bytes_per_rank), r = 0..world-1 (DEVICE). */
typedef int (*slf_allgather_fn)(const void* send, void* recv, size_t bytes_per_rank, void* stream, void* user);
/* buf[0 .. count) fp32 (DEVICE) := elementwise sum over ranks, identical on every rank. */
typedef int (*slf_allreduce_f32_fn)(void* buf, size_t count, void* stream, void* user);
slf_status slf_comm_get_unique_id(void* id128);
slf_status slf_comm_init(slf_comm* out, const void* id128, int rank, int world, int device);
slf_status slf_comm_init_callbacks(slf_comm* out, int rank, int world, slf_allgather_fn allgather,
                                   slf_allreduce_f32_fn allreduce, void* user);
slf_status slf_comm_destroy(slf_comm comm);
/* HOST *rank, *world of the communicator. */
slf_status slf_comm_rank(slf_comm comm, int* rank, int* world);
/* P2P exchanges over CUDA IPC instead of the transport's collectives;
 * `enable` is a bit mask: 1 = the per-chunk statistics all-gather (below), 2 = the dX exchange
 * kernel (per chunk, one kernel on the communicator's stream sums the g ranks' fp32 partials of
 * this rank's row slice in rank order from peer memory and stores the bf16 rows into every rank's
 * dhidden — reduce-scatter + all-gather + finalize; the workspace and dhidden are exported as IPC
 * allocation base + offset each call, so they must come from cudaMalloc, e.g. PyTorch's caching
 * allocator), 3 = both, 0 = off.
 * Statistics (bit 1): instead of the transport's all-gather.  At the next sharded call every rank allocates a receive buffer
 * [256 B flags | 2 x world x C x 16 B] with cudaMalloc (communicator-owned, like NCCL's own
 * buffers; freed by slf_comm_destroy or enable = 0), the CUDA IPC handles are exchanged through the
 * transport and mapped (cudaIpcMemLazyEnablePeerAccess; NVLink peers, or other processes on the
 * same GPU).  Per chunk one kernel stores the rank's statistics into slot `rank` of every rank's
 * buffer and bumps a per-source counter there (system-scope release); the consumer waits on its own
 * counters (acquire).  A wait that exceeds ~30 s gives up instead of hanging: the call's loss is
 * then NaN (every element for NONE), slf_comm_status reports it, and every later
 * slf_lce_fwd_bwd_sharded call on this communicator returns SLF_ERR_COMM (sticky; recreate it).
 * All ranks must set the same mode.  world <= 16. */
slf_status slf_comm_set_p2p(slf_comm comm, int enable);
/* Synchronising: HOST *p2p_timeouts = 1 if a P2P wait ever timed out on this rank (results of
 * that call are invalid, its loss NaN), else 0. */
slf_status slf_comm_status(slf_comm comm, int32_t* p2p_timeouts);

/* Rank k of g owns W rows [V_global*k/g, V_global*(k+1)/g) (contiguous, as even as possible). */
slf_status slf_shard_bounds(int64_t V_global, int world, int rank, int64_t* vocab_start, int64_t* V_local);

/* Workspace of slf_lce_fwd_bwd_sharded for rank `rank` of `world`: the schedule-S workspace and
 * the local / gathered per-row statistics (2C*16 and world*2C*16 bytes), plus — only when that
 * placement cuts fewer row chunks — a dedicated fp32 dX partial [2C, H]; otherwise each chunk's
 * fp32 partial lives in dhidden's not-yet-written top rows, or (the last chunks) in the tail of the
 * workspace stash.  All within `budget_bytes` (0: 5 % of the GLOBAL N*V_global*2
 * logits per GPU).  Host only; 0 if nothing fits. */
size_t slf_lce_sharded_workspace_bytes(int64_t N, int64_t H, int64_t V_global, int world, int rank,
                                       size_t budget_bytes);
/* Writes the plan (chunk rows, chunks, partial placement, planner budget, workspace bytes) into
 * HOST `out`. */
slf_status slf_lce_sharded_plan_describe(int64_t N, int64_t H, int64_t V_global, int world, int rank,
                                         size_t budget_bytes, char* out, size_t cap);
/* The row chunks the sharded call cuts when dhidden is requested (the same on every rank), as HOST
 * int64 rows of 6: (first row, rows, extended-stash rows in dhidden, partial placement: byte offset
 * into dhidden or -1 = workspace stash tail or -2 = workspace region, end in bytes of the dhidden
 * rows X'^T may use, stash row pitch used for the extension).  At most `cap` rows are written;
 * *n_chunks = the count.  Host only (planning; for tests and tools). */
slf_status slf_lce_sharded_chunk_table(int64_t N, int64_t H, int64_t V_global, int world, int rank,
                                       size_t budget_bytes, int64_t* out, int64_t cap, int64_t* n_chunks);

/* The whole vocab-sharded step on this rank (schedule S, per row chunk c):
 *   stash GEMM + this shard's row statistics -> all-gather (16 B/row/rank, rank order)
 *   -> shard-order merge, loss rows, in-place G_P, grouped dX-partial (fp32) / dW (+)= launch
 *   -> all-reduce of the chunk's fp32 dX (comm stream, overlaps chunk c+1's stash GEMM) -> bf16
 *   dhidden rows (the partial may live in dhidden's unwritten rows: slf_lce_sharded_chunk_table);
 *   after the chunks: one-hot dW correction (local targets) and the loss.
 *   hidden [N, H] bf16, targets [N] int32: identical on every rank            (read)
 *   weight_shard [V_local, H] bf16: this rank's rows (slf_shard_bounds)       (read)
 *   loss_out DEVICE fp32 [1] (SUM/MEAN) or [N] (NONE): the global loss, every rank
 *   dhidden [N, H] bf16: the full (all-reduced) gradient, every rank          (overwritten)
 *   dweight_shard [V_local, H] bf16: this rank's rows of dW                   (overwritten)
 *   workspace >= slf_lce_sharded_workspace_bytes(N, H, V_global, world, rank, budget_bytes)
 * Every rank must make the same sequence of calls with the same N, H, V_global, ignore_index,
 * reduction and budget.  Results are those of slf_lce_fwd_bwd on the whole W within the
 * BASELINE tolerance (the shards' dX partials are summed in fp32).  Errors: SLF_ERR_COMM for a
 * transport failure (the other ranks may then block inside their collectives). */
slf_status slf_lce_fwd_bwd_sharded(const void* hidden, const void* weight_shard, const int32_t* targets, int64_t N,
                                   int64_t H, int64_t V_global, int32_t ignore_index, int reduction, float scale,
                                   float* loss_out, void* dhidden, void* dweight_shard, void* workspace,
                                   size_t workspace_bytes, size_t budget_bytes, slf_comm comm, void* stream);

/* Data-parallel (token-sharded) form (SURVEY §8(e) "alternative partition", §8(f) NEXT-3): rank k
 * holds its own tokens (hidden [N_local, H], targets [N_local]) and the FULL weight [V, H].  The
 * fused call runs with the MEAN denominator summed across ranks on the device right after the
 * target scan (so coef and the loss use the GLOBAL valid count, no host round trip); the loss
 * (SUM / MEAN) is all-reduced, so every rank returns the global loss; dhidden stays local;
 * dweight is this rank's partial, or with sync_dweight = 1 the all-reduced sum (bf16, NCCL
 * transport only: SLF_ERR_UNSUPPORTED otherwise).  Workspace as slf_lce_fwd_bwd for N_local. */
slf_status slf_lce_fwd_bwd_dp(const void* hidden, const void* weight, const int32_t* targets, int64_t N_local,
                              int64_t H, int64_t V, int32_t ignore_index, int reduction, float scale, float* loss_out,
                              void* dhidden, void* dweight, void* workspace, size_t workspace_bytes, int schedule,
                              size_t budget_bytes, int sync_dweight, slf_comm comm, void* stream);

/* Debug: copy the per-tile clock64 trace recorded for the launch selected by the environment
 * variable SLF_DEBUG_TRACE=k (the k-th GEMM launch of the process) into HOST `host` (n values,
 * 8 per tile: MMA tile start / after TMEM-free wait / issued, epilogue start / accumulator ready /
 * TMEM released / end, problem index), followed by 256 x 8 per-unit counters of that launch
 * (MMA cycles waiting on full stages / on a free accumulator, first / last clock, K-blocks,
 * producer cycles waiting on empty stages, tiles).  Synchronises the device. */
slf_status slf_debug_trace_read(uint64_t* host, int64_t n);

/* p[i] = bf16(p[i] * s) for a DEVICE bf16 array of n elements (n % 8 == 0, 16-byte aligned):
 * applies an autograd grad_output to gradients formed during the forward (LCEFunctionFused). */
slf_status slf_scale_bf16(void* p, int64_t n, float s, void* stream);
/* The same with the factor in DEVICE memory (s_dev[0], fp32): no host read of an autograd
 * grad_output; a no-op pass when it is exactly 1. */
slf_status slf_scale_bf16_dev(void* p, int64_t n, const float* s_dev, void* stream);
/* RowStat out[i] = in[i] with coef multiplied by grad[0] (per_row = 0: SUM / MEAN grad_output) or
 * grad[i] (per_row = 1: reduction NONE, one upstream gradient per row); DEVICE pointers, N rows,
 * in / out may alias.  slf_lce_bwd on `out` with grad_scale = 1 then yields the gradients of
 * sum_i grad_i * loss_i: the autograd backward without a host synchronisation (LCEFunction). */
slf_status slf_rowstat_scale(const slf_rowstat* in, const float* grad, int per_row, int64_t N, slf_rowstat* out,
                             void* stream);

/* Debug: number of clusters of `cluster` CTAs of the GEMM kernel that can be co-resident (HOST
 * *out), from cudaOccupancyMaxActiveClusters with the kernel's shared-memory footprint. */
slf_status slf_debug_max_active_clusters(int cluster, int* out);

/* ---- the final RMSNorm that feeds the LM head ----
 * y = bf16(x * rstd * g), rstd = 1/sqrt(mean_h x^2 + eps) (fp32, [N]); backward with the LCE's
 * dhidden as dy: dx = rstd * (g*dy - xhat * mean_h(xhat*g*dy)), xhat = x*rstd, and
 * dg = sum_rows dy*xhat (fp32 [H], fixed-order, deterministic).  x, y, dy, dx: [N, H] bf16;
 * g: [H] bf16; dy and dx may be the same buffer.  H % 8 == 0, H <= 16384.  The backward needs a
 * workspace of slf_rmsnorm_workspace_bytes(N, H) bytes. */
size_t slf_rmsnorm_workspace_bytes(int64_t N, int64_t H);
slf_status slf_rmsnorm_fwd(const void* x, const void* g, int64_t N, int64_t H, float eps, void* y, float* rstd,
                           void* stream);
slf_status slf_rmsnorm_bwd(const void* x, const void* g, const float* rstd, const void* dy, int64_t N, int64_t H,
                           void* dx, float* dg, void* workspace, size_t workspace_bytes, void* stream);

/* The final RMSNorm fused into the LCE (PAPER.md l.273 lists RMSNorm among the
 * fused Triton kernels): loss, dx = d loss / d x, dg = d loss / d g and dW of
 *     loss = LCE(rmsnorm(x, g, eps) W^T, targets)
 * in one call, schedule S, without the [N, H] normalised activations: per row chunk one launch
 * forms the chunk's y = bf16(x * rstd * g) (the same bits as slf_rmsnorm_fwd) into a chunk buffer
 * in the workspace, the stash / dX / dW GEMMs read it there, and the next launch turns the chunk's
 * dy (the group's bf16 dX output, in `dx`) into dx in place and accumulates dg (fp32, fixed order).
 * The one-hot dW term recomputes y from x, rstd and g.
 *   x [N, H] bf16, g [H] bf16, weight [V, H] bf16, targets [N] int32                    (read)
 *   loss_out [1] (SUM/MEAN) or [N] (NONE) fp32; dx [N, H] bf16; dg [H] fp32; dweight [V, H] bf16
 *                                                                                        (overwritten)
 *   workspace >= slf_rmsnorm_lce_workspace_bytes(N, H, V, budget_bytes): budget 0 = the LCE's default
 *   plan (5 % of N*V*2) plus the chunk buffers; else the whole layout fits within budget_bytes.
 * All DEVICE pointers, 16-byte aligned, non-null; H % 8 == 0, H <= 16384.  Errors as slf_lce_fwd_bwd
 * (SLF_ERR_WORKSPACE if no schedule-S plan fits). */
size_t slf_rmsnorm_lce_workspace_bytes(int64_t N, int64_t H, int64_t V, size_t budget_bytes);
slf_status slf_rmsnorm_lce_plan_describe(int64_t N, int64_t H, int64_t V, size_t budget_bytes, char* out, size_t cap);
slf_status slf_rmsnorm_lce_fwd_bwd(const void* x, const void* g, float eps, const void* weight, const int32_t* targets,
                                   int64_t N, int64_t H, int64_t V, int32_t ignore_index, int reduction, float scale,
                                   float* loss_out, void* dx, float* dg, void* dweight, void* workspace,
                                   size_t workspace_bytes, size_t budget_bytes, void* stream);

/* Synchronises `stream` and returns (in *bad_targets, HOST) the number of
 * valid targets outside [0, V_global) seen by the last call that used this
 * workspace, and (in *n_valid, HOST, may be NULL) the number of valid rows. */
slf_status slf_lce_status(const void* workspace, void* stream, int32_t* bad_targets, int64_t* n_valid);

/* Target CSR of one vocabulary shard (the schedule-S one-hot dW correction reads
 * it): a stable counting sort of the valid tokens whose target falls in [vocab_start,
 * vocab_start + V_local) by t_i - vocab_start.  The method itself needs no CSR (PAPER.md l.273 only
 * fixes the result); it is how dW[v] -= coef * sum_{t_i = v} x_i is formed exactly once per row.
 *   targets   DEVICE int32 [N], 16-byte aligned                                     (read)
 *   offsets   DEVICE int32 [V_local + 2]: offsets[v] .. offsets[v+1] delimit row v's tokens in
 *             token_idx; offsets[V_local] = number of such tokens, offsets[V_local + 1] = number
 *             of rows with at least one                                             (overwritten)
 *   token_idx DEVICE int32 [N]: its first offsets[V_local] entries are the token indices grouped by
 *             row, increasing within a row (stable)                                 (overwritten)
 *   scratch   DEVICE, >= slf_target_csr_scratch_bytes(N, V_local) bytes, 16-byte aligned
 * Integer only, deterministic (no atomics decide positions).  Enqueued on `stream`; errors are
 * synchronous status codes.  The same kernels run inside slf_lce_fwd_bwd (schedule S). */
size_t slf_target_csr_scratch_bytes(int64_t N, int64_t V_local);
slf_status slf_target_csr(const int32_t* targets, int64_t N, int32_t ignore_index, int64_t vocab_start,
                          int64_t V_local, int32_t* offsets, int32_t* token_idx, void* scratch, size_t scratch_bytes,
                          void* stream);

/* Test entry point: a plain bf16 GEMM D[M,N] (fp32, row-major, ld = N) =
 * A * B through the same tcgen05 core, with A [M,K] (a_mn = 0: K contiguous)
 * or stored as [K,M] (a_mn = 1), B stored [N,K] (b_mn = 0) or [K,N] (b_mn = 1).
 * Used by the GPU tests to check the core against torch.matmul. */
slf_status slf_debug_gemm(const void* A, const void* B, float* D, int64_t M, int64_t N, int64_t K, int a_mn,
                          int b_mn, void* stream);

/* Vocab-shard backward, last step: dhidden bf16 [N, H] = RNE(dhidden_fp32 [N, H]) after the
 * caller has summed the shards' fp32 partials (e.g. NCCL all-reduce); rows whose RowStat says
 * ignored are written as +0.0.  All DEVICE pointers, 16-byte aligned. */
slf_status slf_lce_dx_finalize(const float* dhidden_fp32, const slf_rowstat* rowstat, void* dhidden, int64_t N,
                               int64_t H, void* stream);

/* ---- instrumentation (bench.py / profiling only; not needed for correctness) ----
 * slf_profile_begin: from now on, every kernel the library launches FROM THIS THREAD is bracketed
 * by a pair of CUDA events recorded on its stream.  slf_profile_end: synchronises those events and
 * writes per-kind totals into HOST arrays of SLF_PROF_KINDS entries: device milliseconds, launches,
 * algorithmic FLOPs (2*M*N*K of each GEMM launch) and algorithmic bytes (aux kernels: bytes they
 * must read + write).  Kinds: */
#define SLF_PROF_KINDS 18
#define SLF_PROF_GEMM_STATS 0 /* forward logits tile GEMM + stats epilogue          */
#define SLF_PROF_GEMM_GRAD 1  /* backward recompute GEMM + dlogit (G) epilogue      */
#define SLF_PROF_GEMM_DW 2    /* dW = G^T X                                         */
#define SLF_PROF_GEMM_DX 3    /* dX = G W                                           */
#define SLF_PROF_GEMM_DEBUG 4 /* slf_debug_gemm                                     */
#define SLF_PROF_PREP 5       /* target scan                                        */
#define SLF_PROF_LOCAL_COMBINE 6
#define SLF_PROF_FINAL_COMBINE 7
#define SLF_PROF_DX_FINALIZE 8
#define SLF_PROF_GEMM_GROUP 9         /* one launch holding the dW and dX GEMMs of a chunk */
#define SLF_PROF_COMBINE_TRANSFORM 10 /* schedule S: lse, loss, stash -> G_P in place     */
#define SLF_PROF_CSR 11               /* schedule S: target CSR (stable counting sort)    */
#define SLF_PROF_ONEHOT 12            /* schedule S: dW[v] -= coef * sum x_i               */
#define SLF_PROF_LOSS_REDUCE 13       /* schedule S: deterministic loss sum               */
#define SLF_PROF_RMSNORM 14           /* final RMSNorm forward / backward (NEXT-1)        */
#define SLF_PROF_TRANSPOSE 15         /* schedule S: X_chunk^T for the dW GEMM's B operand */
#define SLF_PROF_COMM_ALLGATHER 16    /* NCCL all-gather of per-row statistics (comm stream) */
#define SLF_PROF_COMM_ALLREDUCE 17    /* NCCL all-reduce (dX partials, counts, loss; comm stream) */
slf_status slf_profile_begin(void);
slf_status slf_profile_end(double* ms, int64_t* launches, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif

#endif /* SLF_LCE_H_ */
