/*
 * fsdp.h -- C ABI of the B200-native SimpleFSDP data-parallel hot path.
 *
 * The method (arXiv 2411.00284, "SimpleFSDP"; citations P:<line> are lines of
 * the paper's LaTeX source PAPER.md, S:<line> lines of SPEC.md):
 *   - shard every parameter along dim 0 across N devices;
 *   - all-gather the parameters before forward use, release them, all-gather
 *     them again before backward use;
 *   - reduce-scatter the gradients with an average after backward, in
 *     reduce_dtype;
 *   - bucket the collectives and reorder them for prefetch
 *     (P:182-193), with manual or greedy auto wrapping (Alg. 1).
 *
 * Conventions (all entry points):
 *   - Every function returns fsdp_status; nothing throws or aborts across the
 *     ABI.  On failure fsdp_last_error() returns a thread-local message that
 *     stays valid until the next fsdp_* call on the same thread.
 *   - Arguments are validated before anything is enqueued: a failing call
 *     enqueues nothing.
 *   - "device" pointers are CUDA device pointers of the ctx's device; "host"
 *     pointers are ordinary host memory.  fsdp_stream_t is a cudaStream_t.
 *   - The caller owns every large device buffer (shards, full parameters,
 *     full gradients, gradient shards, staging).  The library owns only the
 *     ctx, bucket handles and their small device run tables, each released by
 *     the matching *_destroy.  The library never frees caller memory; caller
 *     pointers bound in fsdp_bucket_create must outlive the bucket.
 *   - All device work is stream-ordered and asynchronous; only
 *     fsdp_run_schedule with FSDP_SCHED_TIMING and fsdp_proxy_calibrate
 *     synchronise.  A ctx is not thread-safe; distinct ctxs are independent.
 *   - There is no CPU fallback: a call that needs the GPU fails with
 *     FSDP_ERR_CUDA when no device is present.  Host-only calls
 *     (fsdp_shard with NULL data pointers, fsdp_plan_buckets, fsdp_layout,
 *     fsdp_run_schedule with FSDP_SCHED_DRY_RUN on a NULL ctx) work without one.
 */
#ifndef FSDP_B200_FSDP_H
#define FSDP_B200_FSDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FSDP_ABI_VERSION 5  /* 2: schedule.hook; 3: schedule.emulate; 4: p2p_schedule.max_ctas;
                              5: fsdp_bucket_launch_kernel, 80-B NVLS handle, window pointers,
                                 host_io.async_d2h */

typedef void* fsdp_stream_t; /* cudaStream_t */

typedef enum {
  FSDP_OK = 0,
  FSDP_ERR_INVALID_ARG = 1,
  FSDP_ERR_CUDA = 2,
  FSDP_ERR_NCCL = 3,
  FSDP_ERR_OOM = 4,
  FSDP_ERR_UNSUPPORTED = 5
} fsdp_status;

typedef enum { FSDP_BF16 = 0, FSDP_FP32 = 1 } fsdp_dtype; /* param_dtype / grad dtype */

const char* fsdp_last_error(void);
int32_t fsdp_abi_version(void);

/* One parameter p_j of shape [dim0, ...]; row_numel = product of the other
 * dims (1 for 1-D tensors).  module_id tags the wrapping module;
 * array index = forward-use order. */
typedef struct {
  int64_t dim0;
  int64_t row_numel;
  int32_t module_id;
  int32_t reserved; /* must be 0 */
} fsdp_param_desc;

/* Rank r's dim-0 shard: shard_rows = c = ceil(dim0/N); the rank owns rows
 * [row_begin, row_begin + valid_rows) with valid_rows = clamp(dim0 - r*c, 0, c)
 * and row_begin = min(r*c, dim0); shard_numel = c * row_numel.  Rows past
 * valid_rows are padding and hold +0. */
typedef struct {
  int64_t shard_rows;
  int64_t row_begin;
  int64_t valid_rows;
  int64_t shard_numel;
} fsdp_shard_info;

/* ---------------------------------------------------------------- context */
typedef struct fsdp_ctx fsdp_ctx;

/* Writes a 128-byte NCCL unique id (host memory) for an owned communicator. */
fsdp_status fsdp_nccl_get_unique_id(void* uid128);

/* Creates the per-rank context on cuda_device.
 *   nccl_uid (host, 128 B) non-NULL : the ctx owns a new NCCL communicator of
 *                                     `world` ranks (collective call: every rank
 *                                     must call it with the same uid);
 *   borrowed_comm non-NULL          : use this ncclComm_t (never destroyed here);
 *   both NULL                       : layout-only ctx for rank `rank` of a
 *                                     simulated world: ISSUE runs only the pack,
 *                                     WAIT only the copy-out, no collective.
 * world >= 1, 0 <= rank < world.  A ctx with a communicator issues its
 * collectives at every world size (at world 1 NCCL's in-place collectives are
 * local no-ops); a layout-only ctx never issues one. */
fsdp_status fsdp_ctx_create(fsdp_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                            const void* nccl_uid, void* borrowed_comm);
fsdp_status fsdp_ctx_destroy(fsdp_ctx* ctx);

/* The same with NCCL communicator settings (used with nccl_uid only; the
 * library builds the communicator with ncclCommInitRankConfig): bound the SMs
 * NCCL's kernels take from the compute they overlap -- min_ctas /
 * max_ctas per collective, nvls_ctas for NVLS kernels, cta_policy
 * (NCCL_CTA_POLICY_*).  A field <= 0 (cta_policy < 0) keeps NCCL's default.
 * cfg NULL == fsdp_ctx_create.  FSDP_ERR_INVALID_ARG: cfg with a borrowed
 * communicator or no nccl_uid, min_ctas > max_ctas. */
typedef struct {
  int32_t min_ctas;
  int32_t max_ctas;
  int32_t nvls_ctas;
  int32_t cta_policy;
} fsdp_nccl_config;
fsdp_status fsdp_ctx_create_config(fsdp_ctx** out, int32_t world, int32_t rank, int32_t cuda_device,
                                   const void* nccl_uid, const fsdp_nccl_config* cfg);

/* NCCL's own time estimate for one bucket collective on this ctx's
 * communicator (ncclGroupSimulateEnd: NCCL's topology-aware model, nothing is
 * launched) -- a cross-check of the alpha + beta n model (the paper
 * blames auto-wrap misses on that estimate) and an alternative planner
 * input.  op: FSDP_OP_AG (bf16 gather of full_bytes in total) or FSDP_OP_RS
 * (fp32 reduce-scatter, sum, of full_bytes in total).  Writes ns (NCCL's float
 * microseconds x 1000, rounded).  FSDP_ERR_INVALID_ARG without a
 * communicator, for another op, full_bytes not a multiple of world x element
 * size; FSDP_ERR_NCCL if NCCL cannot simulate; FSDP_ERR_UNSUPPORTED if NCCL
 * returns no estimate (it reports none for a 1-rank communicator). */
fsdp_status fsdp_nccl_estimate_ns(fsdp_ctx* ctx, int32_t op, int64_t full_bytes, int64_t* ns);

/* 2-D meshes (Tensor Parallel: a parameter "doubly sharded on both
 * Data Parallel (DP) and Tensor Parallel (TP) dimensions ... is first
 * redistributed (via an all-gather) on the DP sub-mesh"): the FSDP path runs
 * unchanged on the DP sub-mesh over the TP-local tensors.  fsdp_ctx_split
 * creates that sub-mesh ctx from a ctx with a communicator by ncclCommSplit
 * (a collective call over the parent): ranks with equal `color` form one
 * sub-communicator, ordered by `key`; e.g. TP innermost (rank = dp * TP + tp):
 * color = tp, key = dp.  The new ctx owns its communicator (world / rank =
 * the sub-mesh's); color = -1 (NCCL_SPLIT_NOCOLOR) leaves *out NULL.
 * Errors: parent without communicator, color < -1 -> FSDP_ERR_INVALID_ARG. */
fsdp_status fsdp_ctx_split(fsdp_ctx* parent, int32_t color, int32_t key, fsdp_ctx** out);
/* World size and rank of a ctx (host-only; NULL outputs skipped). */
fsdp_status fsdp_ctx_info(const fsdp_ctx* ctx, int32_t* world, int32_t* rank);

/* ------------------------------------------------------------ 1. fsdp_shard
 * P:69 "partitioned per the number of devices ... Each device only holds one of
 * the partitions"; P:133 Shard(0) DTensors.  Always fills *info.  If both
 * full_dev ([dim0, row_numel] row-major, dtype dt) and shard_dev
 * ([shard_rows, row_numel], dtype dt) are non-NULL, also enqueues on `stream`
 * the copy of the owned rows and the zero fill of the padding rows (kernel
 * K0).  Exactly one NULL pointer is FSDP_ERR_INVALID_ARG. */
fsdp_status fsdp_shard(int32_t world, int32_t rank, const fsdp_param_desc* p, fsdp_dtype dt,
                       const void* full_dev, void* shard_dev, fsdp_shard_info* info,
                       fsdp_stream_t stream);

/* ---------------------------------------------------- 2. fsdp_plan_buckets
 * Bucket plan for one phase.  Modes:
 *   PER_PARAM : singletons (the unbucketed baseline);
 *   MANUAL    : one bucket per wrapped module: maximal runs of
 *               equal module_id in the phase's execution order;
 *   SIZE_CAP  : GREEDY with the time constraint disabled;
 *   GREEDY    : Algorithm 1, Table 1 variables:
 *     forward  : merge q_i iff T_AG(open + q_i) <= T_c and M(open) + M_i <= M_max
 *     backward : merge q_i iff T_RS(b_{j-2}) + T_AG(open + q_i) <= T_c and the same memory test
 *     T(n) = alpha_ns + ceil(n * beta_fs_per_byte / 1e6), n = N * segment
 *     bytes of the bucket in its dtype; T_c = sum of t_compute_ns over the
 *     previously closed bucket (0 before the first close); M_i = mem_bytes[i]
 *     or, if mem_bytes is NULL, the padded gathered bytes N * c_i * row_numel_i
 *     * sizeof(param_dtype); ties merge.
 * The phase execution order is forward-use order (FWD) or its reverse (BWD).
 * Output: bucket_begin[0..n_buckets] (caller array of n_params + 1) holds
 * positions in the phase order: bucket b = positions [bucket_begin[b],
 * bucket_begin[b+1]); the forward index of position k is k (FWD) or
 * n_params - 1 - k (BWD).  trace (nullable, n_params - 1 records) receives one
 * record per decision i = 2..P (GREEDY / SIZE_CAP fill every field; other
 * modes fill param and accept only).  Host-only. */
typedef struct {
  int64_t alpha_ns;
  int64_t beta_fs_per_byte;
} fsdp_link;

typedef enum {
  FSDP_PLAN_PER_PARAM = 0,
  FSDP_PLAN_MANUAL = 1,
  FSDP_PLAN_SIZE_CAP = 2,
  FSDP_PLAN_GREEDY = 3
} fsdp_plan_mode;

typedef enum { FSDP_PHASE_FWD = 0, FSDP_PHASE_BWD = 1 } fsdp_phase;

typedef struct {
  const fsdp_param_desc* params; /* n_params, forward order */
  const int64_t* t_compute_ns;   /* n_params, this phase's T_ci, by forward index */
  const int64_t* mem_bytes;      /* n_params or NULL (see above) */
  fsdp_link ag;
  fsdp_link rs;
  int64_t mem_max_bytes;
  int32_t n_params;
  int32_t world;
  int32_t align_bytes;  /* layout alignment A >= 1 (16 default) */
  int32_t mode;         /* fsdp_plan_mode */
  int32_t phase;        /* fsdp_phase */
  int32_t param_dtype;  /* fsdp_dtype of the all-gather */
  int32_t reduce_bytes; /* bytes per reduce_dtype element: 4 (fp32) */
  int32_t reserved;
} fsdp_plan_in;

typedef struct {
  int64_t t_lhs_ns; /* T_AG(open + q_i) (+ T_RS(b_{j-2}) in BWD) */
  int64_t t_rhs_ns; /* T_c */
  int64_t m_lhs;    /* M(open) + M_i */
  int64_t m_rhs;    /* M_max */
  int32_t param;    /* forward index of q_i */
  int32_t accept;   /* 1 = merged into the open bucket */
} fsdp_plan_trace;

fsdp_status fsdp_plan_buckets(const fsdp_plan_in* in, int32_t* bucket_begin, int32_t* n_buckets,
                              fsdp_plan_trace* trace);

/* fsdp_plan_search (beyond Algorithm 1): starting from a plan of
 * the phase (start_begin: n_start + 1 increasing phase positions from 0 to
 * n_params, e.g. fsdp_plan_buckets' output), hill-climb over contiguous
 * partitions scored by the predicted phase time -- fsdp_simulate_schedule over
 * the op sequence fsdp_run_schedule would enqueue with cost->sched_flags, with
 * collectives at alpha + ceil(n beta) (in->ag / in->rs, n = N x segment), the
 * copy-out K3 at 2 x full bytes / unpack_bytes_per_us + copy_launch_ns (none
 * for a direct-gather bucket), the gradient pack K4 at (2 + reduce_bytes) B per
 * element / pack_rs_bytes_per_us + copy_launch_ns, a bucket's compute at the
 * sum of its t_compute_ns + compute_overhead_ns.  Moves, in this order, first
 * strict improvement taken: remove each inner boundary, move it by -1, by +1;
 * then split each bucket at its midpoint, first and last position.  A
 * candidate is feasible when every bucket has M <= in->mem_max_bytes (M as in
 * fsdp_plan_buckets) or a single parameter.  Stops when no move improves or
 * after max_moves improvements (0 = no limit).  Writes the plan like
 * fsdp_plan_buckets (bucket_begin: n_params + 1 entries, caller-allocated) and
 * its predicted phase time.  Deterministic, host-only.  Errors: NULL
 * arguments, a start plan that is not a partition or exceeds the memory cap,
 * non-positive rates -> FSDP_ERR_INVALID_ARG. */
typedef struct {
  int64_t unpack_bytes_per_us;  /* K3 HBM rate, bytes per microsecond (6.47 TB/s = 6470000) */
  int64_t pack_rs_bytes_per_us; /* K4 HBM rate */
  int64_t copy_launch_ns;       /* launch + ramp + tail per copy kernel */
  int64_t compute_overhead_ns;  /* per bucket, on top of its T_c */
  uint32_t sched_flags;         /* FSDP_SCHED_REORDER and placement bits of the schedule to score */
  int32_t max_moves;            /* 0 = until no move improves */
} fsdp_search_cost;
fsdp_status fsdp_plan_search(const fsdp_plan_in* in, const fsdp_search_cost* cost, const int32_t* start_begin,
                             int32_t n_start, int32_t* bucket_begin, int32_t* n_buckets, int64_t* predicted_ns);

/* Bucket layout, host-only: for k members (forward order) of
 * elem_bytes-byte elements at world N, offs[j] = byte offset of member j in a
 * rank segment, *seg_bytes = segment size; off_1 = 0, off_{j+1} =
 * align(off_j + c_j * row_numel_j * elem_bytes), seg = align(end of last). */
fsdp_status fsdp_layout(const fsdp_param_desc* members, int32_t k, int32_t world, int32_t elem_bytes,
                        int32_t align_bytes, int64_t* offs, int64_t* seg_bytes);

/* ------------------------------------------------------------ buckets
 * Binds the device pointers of one bucket's members once (parameters do not
 * move) and builds its device run tables.  Layouts: all-gather segment in
 * param_dtype, reduce-scatter segment in fp32 (reduce_dtype).
 * Pointer arrays have k entries; an array may be NULL if the step that
 * uses it is never called: shards (AG ISSUE), fulls (AG WAIT), full_grads
 * (RS ISSUE), grad_shards (RS WAIT); fsdp_run_schedule needs all four for
 * backward buckets and the first two for forward buckets.  shards[j]: [c_j, R_j] param_dtype; fulls[j]: [d_j, R_j] param_dtype;
 * full_grads[j]: [d_j, R_j] grad_dtype; grad_shards[j]: [c_j, R_j] fp32.
 * The ctx must outlive the bucket. */
typedef struct fsdp_bucket fsdp_bucket;

typedef struct {
  const fsdp_param_desc* params; /* k member descriptors, forward order */
  void* const* shards;
  void* const* fulls;
  const void* const* full_grads;
  void* const* grad_shards;
  int32_t k;
  int32_t align_bytes;
  int32_t param_dtype; /* fsdp_dtype */
  int32_t grad_dtype;  /* fsdp_dtype of full_grads */
  uint32_t flags;      /* FSDP_BUCKET_* below, 0 = plain pointers */
  int32_t reserved;    /* must be 0 */
} fsdp_bucket_desc;

/* Bucket flags: the caller's storage already is this rank's segment (see
 * "Segment-layout storage" below); validated, FSDP_ERR_INVALID_ARG if the
 * pointers do not follow fsdp_layout's offsets. */
enum {
  FSDP_BUCKET_SEGMENT_SHARDS = 1u,
  FSDP_BUCKET_SEGMENT_GRAD_SHARDS = 2u,
  FSDP_BUCKET_FP32_MASTER = 4u,
  FSDP_BUCKET_GROUPED_AG = 8u,
  FSDP_BUCKET_BF16_GRAD_SHARDS = 16u
};
/* FSDP_BUCKET_BF16_GRAD_SHARDS (reading G41; the north star's "1 bf16 ulp
 * after cast"): grad_shards[j] are bf16 [c_j, R_j]; the RS still reduces in
 * fp32 (reduce_dtype) and K6 rounds this rank's fp32 segment to bf16
 * (RNE, one rounding) while copying it out.  Bit-exact against the oracle's
 * rank-order fp32 sum rounded once wherever the fp32 sums agree; within 1 bf16
 * ulp where NCCL's summation order differs.  Excludes
 * FSDP_BUCKET_SEGMENT_GRAD_SHARDS (the fp32 RS cannot land in bf16 storage),
 * gradient accumulation, and the fp32-output peer-memory / NVLS reduce-scatters
 * (K9, K10, FSDP_SCHED_P2P): those return FSDP_ERR_INVALID_ARG. */
/* FSDP_BUCKET_GROUPED_AG (an alternative to copy-in / copy-out bucketing;
 * every member's dim0 divisible by the world size, shards and fulls bound,
 * no FP32_MASTER): the bucket's all-gather is ONE NCCL group of per-member
 * out-of-place all-gathers, shards[j] (c_j rows) -> fulls[j], so NCCL writes
 * every rank's rows straight into the full parameters: no staging, no K1
 * pack, no K3 copy-out, one launch per bucket as with the flat buffer (P:177's
 * goal), same bytes on the wire.  A layout-only ctx's ISSUE copies this rank's
 * rows into the full parameters (K1).  The flat layout stays the default (the
 * paper's design; the grouped form's NCCL efficiency at N > 1 is unmeasured). */
/* FSDP_BUCKET_FP32_MASTER (mixed precision, "parameters are cast to
 * param_dtype"): the shards are fp32 master weights [c_j, R_j] while the
 * all-gather carries param_dtype = FSDP_BF16; the pack (K1) rounds them to
 * bf16 (round to nearest even, cvt.rn.bf16.f32; NaN -> a quiet NaN) while
 * copying.  Needs param_dtype FSDP_BF16; excludes FSDP_BUCKET_SEGMENT_SHARDS
 * (the storage is not the bf16 segment). */

fsdp_status fsdp_bucket_create(fsdp_ctx* ctx, const fsdp_bucket_desc* desc, fsdp_bucket** out,
                               int64_t* ag_seg_bytes, int64_t* rs_seg_bytes);
fsdp_status fsdp_bucket_destroy(fsdp_bucket* b);

/* Segment-layout ("zero-copy") storage, FSDP_BUCKET_SEGMENT_SHARDS: the caller
 * keeps this rank's shards at shards[j] == shards[0] + off_j (off_j = the AG
 * segment offsets of fsdp_layout, shards[0] 16-B aligned), so the storage
 * already is this rank's AG segment: ISSUE launches no pack kernel and the
 * all-gather sends from the storage (out of place; a layout-only ctx's ISSUE
 * then writes nothing); WAIT copies this rank's rows straight from it.
 * FSDP_BUCKET_SEGMENT_GRAD_SHARDS: grad_shards[j] == grad_shards[0] + off'_j
 * (RS segment offsets): the reduce-scatter of a ctx with a communicator writes
 * the averaged gradients directly into the storage (WAIT launches no copy-out;
 * a layout-only ctx still copies its own segment there).  fsdp_bucket_create
 * zeroes the alignment-gap bytes between members of such storage once
 * (synchronously, on the legacy stream).  Reported by fsdp_bucket_query. */
typedef struct {
  int64_t ag_seg_bytes;
  int64_t rs_seg_bytes;
  int64_t kernel_bytes[4]; /* algorithmic HBM bytes per launch of K1 pack, K3 unpack,
                              K4 grad pack, K6 copy-out (0 = kernel not launched) */
  int32_t kernel_chunks[4];
  int32_t ag_zero_copy;
  int32_t rs_zero_copy;
  int64_t p2p_bytes[2];    /* algorithmic bytes per launch of K8 (peer AG) and K9 (peer RS):
                              bytes read from all ranks (local + peers) + bytes written */
  int32_t ag_direct;       /* 1: direct gather (below) */
  int32_t ag_grouped;      /* 1: FSDP_BUCKET_GROUPED_AG */
} fsdp_bucket_info;
/* Direct gather: a one-parameter bucket whose dim 0 divides evenly over the
 * world and whose segment has no alignment gap has a gathered buffer that is
 * byte-identical to the full parameter.  Such a bucket never uses ag_staging:
 * the all-gather writes the full parameter itself (ISSUE packs this rank's
 * rows into it unless the collective sends from segment storage; WAIT has no
 * copy-out).  A layout-only ctx's ISSUE therefore writes this rank's rows of
 * the full parameter only.  Detected automatically. */
fsdp_status fsdp_bucket_query(const fsdp_bucket* b, fsdp_bucket_info* out);

/* ------------------------------------------ 3. fsdp_allgather_bucket
 * copy-in ("flattens and concatenates"), one all-gather AG + wait Wa,
 * copy-out "based on their original tensor size".
 *   FSDP_ISSUE : on `compute`, K1 packs this rank's shards into segment `rank`
 *                of ag_staging (pads zeroed); then on `comm`, after the pack,
 *                an in-place ncclAllGather fills every segment.
 *   FSDP_WAIT  : `compute` waits for the all-gather, then K3 copies the valid
 *                rows of every segment into the full parameters.
 * ag_staging: device, world * ag_seg_bytes, 16-B aligned.  The caller must not
 * re-ISSUE into the same staging before the previous WAIT was enqueued.
 * Layout-only ctx: ISSUE = pack only, WAIT = copy-out only. */
enum { FSDP_ISSUE = 1, FSDP_WAIT = 2, FSDP_NO_COLLECTIVE = 4 };
/* FSDP_NO_COLLECTIVE (with FSDP_ISSUE alone, both bucket calls): run the pack
 * only, no NCCL collective even with a communicator -- for callers that move
 * the bytes themselves (e.g. fsdp_nvls_reduce_scatter_bucket below). */
fsdp_status fsdp_allgather_bucket(fsdp_ctx* ctx, fsdp_bucket* b, void* ag_staging,
                                  fsdp_stream_t compute, fsdp_stream_t comm, uint32_t flags);

/* ------------------------------------- 4. fsdp_reduce_scatter_bucket
 * split each gradient "into chunks based on world size", concatenate
 * chunk q of every member into segment q, one reduce-scatter RS + wait Wr that
 * averages, read out the gradient shards.
 *   FSDP_ISSUE : on `compute`, K4 writes fp32(grad) * fl32(1/N) of chunk q into
 *                segment q of rs_staging (pads +0.0); then on `comm` an in-place
 *                fp32 ncclReduceScatter(sum) leaves rank r's average in segment r.
 *   FSDP_WAIT  : `compute` waits, then K6 copies segment `rank` into grad_shards.
 * rs_staging: device, world * rs_seg_bytes, 16-B aligned.
 * Layout-only ctx: ISSUE = pack only, WAIT = copy-out of segment `rank` only. */
fsdp_status fsdp_reduce_scatter_bucket(fsdp_ctx* ctx, fsdp_bucket* b, void* rs_staging,
                                       fsdp_stream_t compute, fsdp_stream_t comm, uint32_t flags);

/* Gradient accumulation over micro-batches (the
 * read-out of P:179 adds instead of overwriting): with on = 1, every later
 * reduce-scatter of `b` -- fsdp_reduce_scatter_bucket, fsdp_p2p_reduce_scatter_bucket
 * and the RS of fsdp_run_schedule -- leaves grad_shards[j] = grad_shards[j] +
 * (this reduce-scatter's averaged shard), one fp32 addition per element;
 * on = 0 (the default) overwrites.  The mode is latched when the RS is issued
 * (ISSUE / PACK_RS), so toggle it between reduce-scatters, not between an
 * ISSUE and its WAIT.  With FSDP_BUCKET_SEGMENT_GRAD_SHARDS and a
 * communicator an accumulating RS lands in rs_staging and K6 adds it to the
 * storage (the overwrite mode needs no copy-out there).  Host-only; errors:
 * NULL bucket, on not 0/1. */
fsdp_status fsdp_bucket_set_grad_accumulation(fsdp_bucket* b, int32_t on);

/* One data kernel of a bucket, alone (measurement; no event, no collective,
 * no wait): op = FSDP_OP_PACK_AG (K1), FSDP_OP_UNPACK (K3), FSDP_OP_PACK_RS
 * (K4) or FSDP_OP_COPYOUT_RS (K6), launched on `stream` exactly as
 * fsdp_run_schedule launches it for this ctx (same run table, grid and
 * staging slot semantics; skipped where the step skips it, e.g. K1 of
 * segment-layout storage, K6 of segment grad storage with a communicator).
 * *launched (nullable) = 1 if a kernel was enqueued, else 0.  Stream-ordered,
 * capturable into a CUDA graph; the caller orders it against the data it
 * reads.  Errors: NULL ctx / bucket / staging, bucket of another ctx,
 * unaligned staging, an op outside the four, unbound buffers the op needs.
 * (ABI version 5.) */
fsdp_status fsdp_bucket_launch_kernel(fsdp_ctx* ctx, fsdp_bucket* b, int32_t op, void* staging,
                                      fsdp_stream_t stream, int32_t* launched);

/* ------------------------------------------------ 5. fsdp_run_schedule
 * One training step's communication path (Table 6):
 *   reorder on : forward prefetch depth 1 -- AG(k+1) before (default) or after
 *                Wa(k) and its copy-out; backward AG(j+1) after (default) or
 *                before Wa(j); Wr(j-1) before RS(j); first AG and last RS exposed;
 *   reorder off: vanilla -- every collective right before its own wait.
 * Buckets are given in each phase's execution order; bucket b uses staging
 * slot b % 2 (ag_staging[2], rs_staging[2], each >= world * the largest
 * segment).  Compute of bucket b = the caller's hook (fsdp_compute_hook), else
 * linear-layer GEMMs (fsdp_gemm_compute), else compute-proxy kernel K7 with
 * proxy_iters_{fwd,bwd}[b] iterations (NULL or 0 = none).
 * The op sequence is written to report->log (if non-NULL) in host enqueue
 * order as (phase, op, bucket, stream) with op codes FSDP_OP_*; stream 0 =
 * compute, 1 = comm.
 * Flags:
 *   FSDP_SCHED_REORDER            prefetch reordering (else vanilla)
 *   FSDP_SCHED_FWD_AG_BEFORE_WAIT forward AG(k+1) before Wa(k) (else after)
 *   FSDP_SCHED_BWD_AG_BEFORE_WAIT backward AG(j+1) before Wa(j) (else after)
 *   FSDP_SCHED_NO_COMM            run every compute-stream op but no collective
 *                                 and no wait (the compute-only baseline)
 *   FSDP_SCHED_DRY_RUN            write the log only, enqueue nothing (ctx may be NULL)
 *   FSDP_SCHED_TIMING             CUDA events around every op; synchronises at
 *                                 the end and fills step_ns, op_ns/op_count and
 *                                 log[i].ns
 *   FSDP_SCHED_P2P                collectives over peer memory (K8 / K9, see
 *                                 fsdp_p2p_*) instead of NCCL, with `p2p` below:
 *     step start : signal + wait epoch E0 = epoch_base + 1 on the ready flags
 *                  (every rank's shards are final);
 *     PACK_AG    : no kernel (buckets need FSDP_BUCKET_SEGMENT_SHARDS); event;
 *     AG b       : comm stream waits the event, K8 writes the full parameters
 *                  (UNPACK is then empty);
 *     COMPUTE_B b: (b >= 2) first waits the consumed flags >= E(b-2): peers have
 *                  read the gradient slot this bucket's backward overwrites;
 *     PACK_RS b  : signal "gradients of b ready" E(b) = epoch_base + 2 + b;
 *     RS b       : comm stream waits ready flags >= E(b), K9 writes this rank's
 *                  gradient shards, then signals "consumed" E(b);
 *     COPYOUT_RS : no kernel;
 *     step end   : wait consumed >= E(n_bwd - 1), signal + wait epoch_base +
 *                  n_bwd + 2 on the ready flags.
 *   The next step must use epoch_base + n_bwd + 2. */
enum {
  FSDP_OP_PACK_AG = 0, FSDP_OP_AG = 1, FSDP_OP_WAIT_AG = 2, FSDP_OP_UNPACK = 3,
  FSDP_OP_COMPUTE_F = 4, FSDP_OP_COMPUTE_B = 5, FSDP_OP_PACK_RS = 6, FSDP_OP_RS = 7,
  FSDP_OP_WAIT_RS = 8, FSDP_OP_COPYOUT_RS = 9, FSDP_N_OPS = 10
};
enum {
  FSDP_SCHED_REORDER = 1u,
  FSDP_SCHED_FWD_AG_BEFORE_WAIT = 2u,
  FSDP_SCHED_BWD_AG_BEFORE_WAIT = 4u,
  FSDP_SCHED_NO_COMM = 8u,
  FSDP_SCHED_DRY_RUN = 16u,
  FSDP_SCHED_TIMING = 32u,
  FSDP_SCHED_P2P = 64u,
  FSDP_SCHED_KEEP_LAST_GATHERED = 128u,
  FSDP_SCHED_COPY_STREAM = 256u
};
/* FSDP_SCHED_COPY_STREAM (beyond the paper's single compute stream):
 * the pack and copy-out kernels (K1, K3, K4, K6) run on a third, library-
 * owned, highest-priority stream instead of `compute`, so that they overlap
 * the compute of neighbouring buckets rather than sit between them -- the
 * copy-in / copy-out cost the paper blames for bucketing's single-node
 * regression.  Same op sequence, same kernels, same bytes; the data
 * dependencies are kept with events: COMPUTE k waits for UNPACK k; PACK_RS j
 * waits for COMPUTE_B j; an UNPACK (and the all-gather of a direct-gather /
 * grouped bucket, which writes the full parameters itself) waits for the last
 * earlier COMPUTE whose bucket's full-parameter memory overlaps it; a
 * COMPUTE_B waits for the last earlier PACK_RS whose bucket's full-gradient
 * memory overlaps it (overlaps are found from the bound pointers, so any slot
 * layout is safe; adjacent buckets in distinct slots are what lets the copies
 * overlap); the step ends on `compute` after the copy stream's last op.  Log
 * entries of the copy ops carry stream 2.  Not with FSDP_SCHED_P2P (its
 * collectives are the copies). */
/* FSDP_SCHED_KEEP_LAST_GATHERED (reading G42; FSDP2's reshard-after-forward
 * off for the boundary module, which the paper does not describe -- P:137
 * re-gathers every parameter): the first backward bucket reuses the full
 * parameters the last forward bucket gathered, so its re-gather (PACK_AG, AG,
 * WAIT_AG, UNPACK) is left out of the sequence and the log.  Needs
 * bwd[0] to bind the same members and the same full-parameter pointers as
 * fwd[n_fwd - 1] (else FSDP_ERR_INVALID_ARG); those parameters stay live
 * across the forward / backward boundary.  Saves that bucket's all-gather,
 * which is otherwise fully exposed (nothing precedes it in the backward). */

/* Peer tables of one rank for FSDP_SCHED_P2P (device pointers valid in this
 * process; `world` entries per row). */
typedef struct {
  const void* const* ag_peers;  /* (n_fwd + n_bwd) rows: forward buckets then backward
                                   buckets; [q] = rank q's segment storage of that bucket */
  const void* const* rs_peers;  /* n_bwd rows: [q] = rank q's full_grads[0] of that bucket */
  void* const* ready_slots;     /* [q] = this rank's slot in rank q's ready-flag array */
  void* const* done_slots;      /* [q] = this rank's slot in rank q's consumed-flag array */
  const void* ready_flags;      /* this rank's ready-flag array (world uint64) */
  const void* done_flags;       /* this rank's consumed-flag array (world uint64) */
  uint64_t epoch_base;
  int64_t timeout_ns;           /* per wait; 0 = forever */
  int32_t* error_flag;          /* device int set to 1 by a timed-out wait (nullable).  A set
                                   flag means a kernel went ahead without its peers: the step's
                                   results are INVALID.  FSDP_SCHED_TIMING steps read it after
                                   their final synchronisation and fail with FSDP_ERR_CUDA;
                                   otherwise the caller must read it after the step and treat
                                   a nonzero value as a failed step (the flag stays set). */
  uint64_t* epoch_counter;      /* nullable device uint64: if set, every epoch above is
                                   epoch_base + *epoch_counter (read on the device) and the
                                   step's last kernel adds n_bwd + 2 to it -- the step can
                                   then be captured (fsdp_step_graph) and replayed; keep
                                   epoch_base fixed.  Zero it once before the first step. */
  int32_t max_ctas;             /* K8 / K9 grid cap (0 = the library's default, ~8 per SM).  At
                                   N > 1 the peer reads are NVLink-bound and a full-GPU grid
                                   would hold every SM for the link time, starving the compute
                                   stream; a cap like NCCL's channel count leaves the SMs to
                                   compute (57 CTAs carried an 8B block's traffic at N = 8 in
                                   the emulation).  K9 gets twice the cap: it
                                   keeps half of K8's bytes in flight per thread. */
  int32_t grad_slots;           /* gradient slots the backward buckets rotate through (0 = 2):
                                   K9 reads peers' full gradients in place, so the backward of
                                   bucket b first waits until every peer has consumed bucket
                                   b - grad_slots (the same slot); more slots = more slack */
} fsdp_p2p_schedule;

typedef struct {
  fsdp_bucket* const* fwd;      /* n_fwd handles, forward execution order */
  fsdp_bucket* const* bwd;      /* n_bwd handles, backward execution order */
  const int64_t* proxy_iters_fwd; /* n_fwd or NULL */
  const int64_t* proxy_iters_bwd; /* n_bwd or NULL */
  void* ag_staging[2];
  void* rs_staging[2];
  fsdp_stream_t compute;
  fsdp_stream_t comm;
  int32_t n_fwd;
  int32_t n_bwd;
  uint32_t flags;
  int32_t proxy_ctas_per_sm; /* K7 footprint: CTAs per SM (>= 1) */
  int32_t proxy_smem_bytes;  /* K7 footprint: dynamic shared memory per CTA */
  int32_t reserved;
  const fsdp_p2p_schedule* p2p; /* FSDP_SCHED_P2P only, else NULL */
  const struct fsdp_host_io* io; /* host-resident shards / gradient shards, else NULL */
  const struct fsdp_gemm_compute* gemm; /* real linear-layer compute instead of K7, else NULL */
  const struct fsdp_compute_hook* hook; /* caller's model compute instead of K7 / gemm, else NULL */
  const struct fsdp_comm_emulation* emulate; /* emulated N-rank collectives on a layout-only ctx, else NULL */
} fsdp_schedule;

/* Emulated collectives (a measurement device, like the compute proxy K7): on
 * a layout-only ctx (no peers) every AG / RS of the step runs as kernel K11 on
 * the comm stream, with the collective's buffers, SM footprint and duration:
 * `ctas` CTAs of 512 threads (NCCL runs one CTA per channel) move the bytes a
 * rank's HBM sees -- AG: this rank's segment copied into the other N - 1 slots
 * of the gathered buffer; RS: the N fp32 segments summed into this rank's
 * output -- and then hold their SMs until alpha + ceil(n beta / 1e6) ns (n =
 * the collective's full bucket bytes, fsdp_comm_time_ns) have passed since the
 * kernel began.  So the step's exposed time, measured on ONE GPU as (step -
 * compute-only step), includes the SM and HBM contention between the
 * collectives and the compute that the two-stream model leaves out.  The data
 * the emulated collectives leave behind are not the gathered / reduced values
 * (there are no peers): timing only.  With FSDP_SCHED_P2P the peer-memory
 * kernels K8 / K9 themselves do the work (against simulated peers) on a grid
 * of `ctas` CTAs and each CTA stays until the link time has passed (AG: the
 * gathered bucket; RS: the bucket's gradients in their dtype); their results
 * are then the real ones.  Needs a ctx without a communicator, no
 * FSDP_BUCKET_GROUPED_AG buckets; 1 <= ctas <= 4 x SMs (all resident at once). */
typedef struct fsdp_comm_emulation {
  fsdp_link ag;
  fsdp_link rs;
  int32_t ctas;
  int32_t reserved; /* must be 0 */
} fsdp_comm_emulation;

/* Caller-supplied model compute (the real block instead
 * of the proxy).  With `hook` set, the schedule calls
 *     rc = fn(user, phase, bucket, stream)
 * on the host, at the point of the host enqueue order where COMPUTE_F (phase
 * 0) or COMPUTE_B (phase 1) of `bucket` (index in that phase's execution
 * order) belongs, with `stream` = s->compute.  fn must enqueue the bucket's
 * compute on `stream` only (it runs after that bucket's WAIT_AG / UNPACK and
 * before its PACK_RS in stream order): forward reads the gathered full
 * parameters of the bucket's members; backward reads them and writes the
 * members' full_grads, which PACK_RS then averages.  It must not synchronise
 * the comm stream, and it runs once per step.  rc != 0 aborts the step with
 * FSDP_ERR_INVALID_ARG ("compute hook failed"): work enqueued before it stays
 * enqueued, so synchronise before reusing the buffers.  Captured by
 * fsdp_step_graph_create like any other work: a hook that allocates or
 * synchronises must not be used there.  `hook` takes precedence over `gemm`
 * and the proxy iterations. */
typedef int32_t (*fsdp_compute_fn)(void* user, int32_t phase, int32_t bucket, fsdp_stream_t stream);
typedef struct fsdp_compute_hook {
  fsdp_compute_fn fn;
  void* user;
} fsdp_compute_hook;

/* Linear-layer compute instead of the proxy: every
 * member with row_numel > 1 is treated as a linear layer W [d, R] (out = d,
 * in = R, row-major, the gathered full parameter) applied to T tokens with
 * cuBLASLt bf16 GEMMs (fp32 accumulate) on the compute stream:
 *   COMPUTE_F b : Y[T, out]  = X[T, in] . W^T
 *   COMPUTE_B b : dX[T, in]  = dY[T, out] . W,   dW[out, in] = dY^T . X  -> written
 *                 into the member's full_grads (bf16), i.e. the gradients the
 *                 reduce-scatter then averages are real products of the step.
 * 1-D members (norms) take no compute.  No attention / nonlinearity is
 * modelled.  Buffers (device, caller-owned): x [T, max in] and dy [T, max out]
 * bf16 activations, y bf16 scratch of T * max(in, out) elements, a cuBLASLt
 * workspace.  Backward buckets need bf16 gradients. */
typedef struct fsdp_gemm_compute {
  int64_t tokens;
  const void* x;
  const void* dy;
  void* y;
  void* workspace;
  int64_t workspace_bytes;
} fsdp_gemm_compute;

/* Host-resident parameters and gradients (offload): with `io` set, the step
 * streams this rank's shards in from pinned host memory and its averaged
 * gradient shards back out, overlapped bucket by bucket with the device path:
 *   - forward bucket k: on the h2d stream, its segment (ag_seg bytes) is copied
 *     from fwd_host_shards[k] into the bucket's segment-layout shard storage;
 *     PACK_AG k (compute stream) waits for that copy;
 *   - backward bucket j: after its gradient shards are final (COPYOUT_RS j, or
 *     WAIT_RS j with a communicator), the d2h stream copies its gradient-shard
 *     segment (rs_seg bytes) to bwd_host_grads[j]; the step's last
 *     compute-stream work waits for every such copy.
 * The H2D copies (which overwrite the shard storage) are ordered after the
 * previous fsdp_run_schedule step's last reader of that storage -- its last
 * UNPACK on the compute stream -- not after its end, so they overlap the
 * previous step's gradient D2H tail (PCIe is full duplex).  For the first
 * step on a ctx, after a captured or peer-memory step, and after a step with
 * no UNPACK, they wait for everything enqueued on `compute` instead.  Work the
 * caller enqueues between steps that reads the shard storage must be ordered
 * by the caller (e.g. run it before the previous step).
 * Forward buckets need FSDP_BUCKET_SEGMENT_SHARDS and backward buckets
 * FSDP_BUCKET_SEGMENT_GRAD_SHARDS; host memory should be pinned; NULL entries
 * are skipped; h2d / d2h NULL = library-owned streams. */
typedef struct fsdp_host_io {
  const void* const* fwd_host_shards; /* n_fwd */
  void* const* bwd_host_grads;        /* n_bwd */
  fsdp_stream_t h2d;
  fsdp_stream_t d2h;
  int32_t async_d2h;  /* 0: the step's compute stream ends after its gradient D2H (the
                         step is done when the gradients are on the host).  1: it does
                         not wait -- the D2H copies finish on the d2h stream (the caller
                         orders its host reads after that stream), and each bucket's next
                         writer of its gradient-shard storage (its next PACK_RS, in any
                         later step on this ctx) waits for that bucket's D2H instead, so
                         the next step overlaps this step's D2H tail. */
  int32_t reserved;   /* 0 */
} fsdp_host_io;

typedef struct {
  int64_t ns;       /* TIMING: event-measured duration of this op, else -1 */
  int32_t phase;    /* 0 forward, 1 backward */
  int32_t op;       /* FSDP_OP_* */
  int32_t bucket;   /* index in the phase's execution order */
  int32_t stream;   /* 0 compute, 1 comm */
  int64_t start_ns; /* TIMING: start relative to the step's first event (a timeline /
                       Chrome trace), else -1 */
} fsdp_log_entry;

typedef struct {
  fsdp_log_entry* log; /* caller array or NULL */
  int32_t log_capacity;
  int32_t log_len;     /* entries written (sequence length) */
  int64_t step_ns;     /* TIMING: first to last compute-stream event */
  int64_t op_ns[FSDP_N_OPS];    /* TIMING: summed ns per op code */
  int32_t op_count[FSDP_N_OPS]; /* ops per code in this step */
  int32_t kernel_launches;      /* library kernels enqueued by this step */
  int32_t collectives;          /* NCCL collectives enqueued by this step */
} fsdp_step_report;

fsdp_status fsdp_run_schedule(fsdp_ctx* ctx, const fsdp_schedule* s, fsdp_step_report* out);

/* CUDA-graph capture of one step (CUDA graphs instead of a tracing
 * compiler): fsdp_step_graph_create records everything fsdp_run_schedule
 * would enqueue for `s` -- kernels, NCCL collectives, the events between the
 * compute and comm streams -- by stream capture from s->compute (thread-local
 * mode) and instantiates it; fsdp_step_graph_launch replays the whole step
 * as one launch on `stream`.  Every pointer, proxy length and flag is baked
 * in at capture: replay with the same buffers.  s->compute must be a
 * non-default stream; TIMING,
 * DRY_RUN and host I/O are rejected, and FSDP_SCHED_P2P unless its
 * fsdp_p2p_schedule has a device epoch_counter (FSDP_ERR_INVALID_ARG).
 * fsdp_step_graph_info: library kernels / collectives in the captured step. */
typedef struct fsdp_step_graph fsdp_step_graph;
fsdp_status fsdp_step_graph_create(fsdp_ctx* ctx, const fsdp_schedule* s, fsdp_step_graph** out);
fsdp_status fsdp_step_graph_launch(fsdp_step_graph* g, fsdp_stream_t stream);
fsdp_status fsdp_step_graph_info(const fsdp_step_graph* g, int32_t* kernel_launches, int32_t* collectives);
fsdp_status fsdp_step_graph_destroy(fsdp_step_graph* g);

/* ------------------------------------------- cost model and prediction
 * fsdp_comm_time_ns: T(n) = alpha_ns + ceil(n * beta_fs_per_byte / 1e6), the
 *   communication model of P:222 in integer units (what Algorithm 1 uses).
 * fsdp_simulate_schedule: the two-stream timeline of an op sequence (e.g. the
 *   log of fsdp_run_schedule, FSDP_SCHED_DRY_RUN) given per-entry durations
 *   (ns): compute-stream ops run back to back in order; the comm stream is
 *   FIFO and a collective starts when it is at its head and its pack
 *   (PACK_AG / PACK_RS of the same phase and bucket) has finished; a WAIT
 *   blocks the compute stream until its collective has finished (its own
 *   duration is ignored).  Writes the finish time of the compute stream and the
 *   exposed (blocked) time; start/end (nullable, n entries) get each entry's
 *   interval.  Integer ns, deterministic; FSDP_ERR_INVALID_ARG if a collective
 *   or WAIT precedes what it depends on.  Host-only. */
fsdp_status fsdp_comm_time_ns(int64_t nbytes, const fsdp_link* link, int64_t* ns);
fsdp_status fsdp_simulate_schedule(const fsdp_log_entry* seq, int32_t n, const int64_t* dur_ns, int64_t* total_ns,
                                   int64_t* exposed_ns, int64_t* start_ns, int64_t* end_ns);

/* fsdp_simulate_memory: peak memory of the step's FSDP buffers (memory is the
 * paper's other metric, Tables 5 and 6) for an op sequence, as an
 * allocate-on-produce / free-after-last-use allocator would hold them
 * (reading G40), walked in sequence order:
 *   PACK_AG (ph, b): + ag[ph][b]      the flat gathered bucket (N x AG segment)
 *   UNPACK  (ph, b): + full[ph][b]    the full parameters, then - ag[ph][b]
 *   COMPUTE_F b    : - full[0][b]     released after forward use -- except the
 *                                      last forward bucket when backward bucket 0 has no
 *                                      UNPACK (FSDP_SCHED_KEEP_LAST_GATHERED, G42)
 *   COMPUTE_B b    : + grad[b]        the full gradients, then - full[1][b]
 *   PACK_RS b      : + rs[b]          the flat RS input (N x RS segment), then - grad[b]
 *   COPYOUT_RS b   : - rs[b]
 *   AG, RS, WAIT_* : nothing (in-place collectives).
 * The peak is taken after each op's allocation, before its frees; resident
 * shards, gradient shards and activations are outside the curve.  Bytes per
 * bucket in the phase's execution order (arrays of n_fwd / n_bwd entries).
 * Writes the peak and, if `live` is non-NULL, the live bytes after each of
 * the n entries.  FSDP_ERR_INVALID_ARG for a bucket index out of range, a
 * negative size or a live total that goes negative (a free before its
 * allocation).  Host-only. */
typedef struct {
  const int64_t* ag_fwd;   /* n_fwd: N x AG segment bytes */
  const int64_t* full_fwd; /* n_fwd: sum of the members' full parameter bytes */
  const int64_t* ag_bwd;   /* n_bwd */
  const int64_t* full_bwd; /* n_bwd */
  const int64_t* grad_bwd; /* n_bwd: sum of the members' full gradient bytes */
  const int64_t* rs_bwd;   /* n_bwd: N x RS segment bytes */
  int32_t n_fwd;
  int32_t n_bwd;
} fsdp_mem_sizes;
fsdp_status fsdp_simulate_memory(const fsdp_log_entry* seq, int32_t n, const fsdp_mem_sizes* sizes,
                                 int64_t* peak_bytes, int64_t* live);

/* ------------------------------------- peer-memory (fused) collectives
 * The same two collectives as one kernel each over peer memory (NVLink P2P on
 * a multi-GPU node, CUDA IPC mappings; on one GPU, buffers of simulated ranks):
 * every rank pulls what it needs straight from its peers' buffers into its own
 * destination layout -- no staging buffer, no pack, no copy-out, no NCCL.
 *
 *   fsdp_p2p_allgather_bucket: K8 copies the valid rows of every
 *     rank q's shards from peer_segs[q] (rank q's segment-layout shard storage
 *     of this bucket, FSDP_BUCKET_SEGMENT_SHARDS) into this rank's full
 *     parameters.  Wire bytes: (N-1)/N of the gathered bucket, as the AG.
 *   fsdp_p2p_reduce_scatter_bucket: K9 computes this rank's
 *     gradient shards directly: g_shard[t] = sum over q = 0..N-1, in rank order,
 *     of fl32(fp32(grad_q[row r*c + t]) * fl32(1/N)), reading the bf16 (or fp32)
 *     full gradients of every peer: peer_grads[q] is rank q's address of what
 *     this rank binds as full_grads[0]; the members' full_grads must keep the
 *     same offsets from full_grads[0] on every rank (symmetric layout).  Wire
 *     bytes: (N-1)/N of the bucket in the *gradient* dtype (half the fp32 RS for
 *     bf16 gradients); the rank-order fp32 sum is bit-exact against the oracle at
 *     any N.
 * Both are stream-ordered on `stream` and read peer memory without further
 * synchronisation: the caller orders them after the peers' producers (for
 * example with fsdp_p2p_signal / fsdp_p2p_wait, or a host barrier).  world <= 16.
 * Arrays hold `world` device pointers valid in this process. */
fsdp_status fsdp_p2p_allgather_bucket(fsdp_ctx* ctx, fsdp_bucket* b, const void* const* peer_segs,
                                      fsdp_stream_t stream);
fsdp_status fsdp_p2p_reduce_scatter_bucket(fsdp_ctx* ctx, fsdp_bucket* b, const void* const* peer_grads,
                                           fsdp_stream_t stream);

/* ------------------------------------------------ NVLS multicast (K10)
 * NVLink SHARP: the NVSwitch reduces a load issued to a *multicast* address
 * across every GPU of the team (multimem.ld_reduce), so a rank reads only its
 * own reduced chunk -- 1/N of the RS bytes on its NVLink ingress instead of
 * (N-1)/N.  Setup, one team per buffer (a FSDP_NVLS_HANDLE_BYTES handle,
 * exchanged by the caller, e.g. torch.distributed.broadcast_object_list):
 *   rank 0   : fsdp_nvls_create(ctx, bytes, handle, &m)  -- the multicast
 *              object for ctx's world devices, its handle, this GPU added;
 *   others   : fsdp_nvls_import(ctx, handle, bytes, &m)  -- this GPU added;
 *   (host barrier: every rank added)
 *   every rank: fsdp_nvls_bind(m, &uc, &mc, &bytes)  -- this GPU's physical
 *              memory bound, mapped at `uc` (unicast, this GPU only) and at
 *              `mc` (multicast, the team); bytes rounded up to the granularity.
 * Use as RS staging: fsdp_reduce_scatter_bucket(ISSUE | FSDP_NO_COLLECTIVE)
 * packs (K4) into `uc`; after a cross-rank barrier (every rank packed),
 * fsdp_nvls_reduce_scatter_bucket(ctx, b, mc, stream) runs K10: grad_shards =
 * the switch's fp32 sum over ranks of segment `rank` (+ the held shards in
 * accumulation mode); the next pack into the same staging needs another
 * barrier (every rank done reading).  The switch's summation order is its
 * own: results match the oracle within G7's fp32 bound (bit-exact at N <= 2).
 * Handle (fsdp_nvls_handle, FSDP_NVLS_HANDLE_BYTES): create exports a FABRIC
 * handle where the platform has one (IMEX / NVSwitch fabric), else a POSIX
 * file descriptor (type FSDP_NVLS_POSIX_FD: `fd` is valid in the creating
 * process `pid` only -- the caller passes it to each peer, e.g. SCM_RIGHTS over
 * a unix socket as the Python binding does, and writes the RECEIVED fd into
 * the handle before fsdp_nvls_import, which takes ownership of it and closes
 * it).  Errors: FSDP_ERR_UNSUPPORTED without multicast support or where the
 * platform refuses the object (e.g. a one-GPU fabric partition). */
typedef struct fsdp_nvls fsdp_nvls;
enum { FSDP_NVLS_HANDLE_BYTES = 80, FSDP_NVLS_FABRIC = 1, FSDP_NVLS_POSIX_FD = 2 };
typedef struct {
  int32_t type;          /* FSDP_NVLS_FABRIC or FSDP_NVLS_POSIX_FD (0 = a team of one: no handle) */
  int32_t fd;            /* POSIX_FD: the descriptor, valid in the process that holds it */
  int32_t pid;           /* POSIX_FD: the creating process */
  int32_t reserved;
  uint8_t fabric[64];    /* FABRIC: CUmemFabricHandle */
} fsdp_nvls_handle;
fsdp_status fsdp_nvls_create(fsdp_ctx* ctx, int64_t bytes, void* handle_out, fsdp_nvls** out);
fsdp_status fsdp_nvls_import(fsdp_ctx* ctx, const void* handle, int64_t bytes, fsdp_nvls** out);
fsdp_status fsdp_nvls_bind(fsdp_nvls* m, void** uc_ptr, void** mc_ptr, int64_t* bytes);
fsdp_status fsdp_nvls_destroy(fsdp_nvls* m);
fsdp_status fsdp_nvls_reduce_scatter_bucket(fsdp_ctx* ctx, fsdp_bucket* b, const void* mc_staging,
                                            fsdp_stream_t stream);

/* Cross-rank signalling for the peer-memory path (monotonic 64-bit epochs).
 * fsdp_p2p_signal: one thread stores `value` with release semantics at the
 *   system scope into each slots[q] (q < world; NULL entries skipped): slot of
 *   this rank in rank q's flag array, mapped in this process.
 * fsdp_p2p_wait: one warp spins (acquire loads) until flags[q] >= value for
 *   every q < world (flags: this rank's own array), or `timeout_ns` elapses, in
 *   which case it sets *error_flag (device int, nullable) to 1 and returns. */
fsdp_status fsdp_p2p_signal(fsdp_ctx* ctx, void* const* slots, uint64_t value, fsdp_stream_t stream);
fsdp_status fsdp_p2p_wait(fsdp_ctx* ctx, const void* flags, uint64_t value, int64_t timeout_ns,
                          int32_t* error_flag, fsdp_stream_t stream);

/* IPC plumbing for the peer-memory path: a cudaMalloc'd buffer and its
 * 64-byte cudaIpcMemHandle (host memory), to be opened by peer processes. */
fsdp_status fsdp_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle64);
fsdp_status fsdp_ipc_open(const void* handle64, void** dev_ptr);
fsdp_status fsdp_ipc_close(void* dev_ptr);
fsdp_status fsdp_ipc_free(void* dev_ptr);

/* ------------------------------------------ NCCL buffer registration
 * So that the NCCL collectives of the path (8(e)) can run zero-copy on
 * NVSwitch (NVLink SHARP multicast, NCCL's symmetric-memory kernels) instead
 * of staging through NCCL's internal buffers:
 *   fsdp_mem_alloc : ncclMemAlloc -- cuMem-backed device memory NCCL can map
 *                    for multicast; *dev_ptr is at least 4096-B aligned.
 *   fsdp_mem_free  : releases every registration of the ctx that starts at
 *                    dev_ptr, then ncclMemFree.
 *   fsdp_register_buffer: registers [dev_ptr, dev_ptr + bytes) with the ctx's
 *                    communicator:
 *     FSDP_REG_LOCAL     ncclCommRegister (a local call);
 *     FSDP_REG_SYMMETRIC ncclCommWindowRegister(..., NCCL_WIN_COLL_SYMMETRIC):
 *                        a COLLECTIVE call -- every rank registers a buffer of
 *                        the same size, in the same order; dev_ptr from
 *                        fsdp_mem_alloc, 4096-B aligned; collectives on it must
 *                        use the same offsets on every rank (the plan's layout
 *                        guarantees that).
 * Registrations live until fsdp_mem_free of their base pointer or
 * fsdp_ctx_destroy (released before the communicator).  Errors: a ctx with no
 * communicator, NULL / unaligned pointers, bytes < 1 -> FSDP_ERR_INVALID_ARG;
 * NCCL failures -> FSDP_ERR_NCCL (the caller may keep unregistered buffers:
 * registration changes speed, never results). */
enum { FSDP_REG_LOCAL = 0, FSDP_REG_SYMMETRIC = 1 };
fsdp_status fsdp_mem_alloc(fsdp_ctx* ctx, int64_t bytes, void** dev_ptr);
fsdp_status fsdp_mem_free(fsdp_ctx* ctx, void* dev_ptr);
fsdp_status fsdp_register_buffer(fsdp_ctx* ctx, void* dev_ptr, int64_t bytes, int32_t mode);

/* NCCL symmetric windows for the peer-memory path (SURVEY §8(f) NEXT #1,
 * the NCCL 2.28 device API): a buffer registered with FSDP_REG_SYMMETRIC is
 * mapped by NCCL in every rank of the NVLink (LSA) domain, so the K8 / K9
 * peer tables and the K10 multicast staging can come from NCCL instead of
 * CUDA IPC handles and a caller-built multicast object.
 *   fsdp_window_peer_pointers(ctx, base, peer_ptrs[world]): peer_ptrs[q] =
 *       rank q's copy of the window at `base` (ncclGetPeerPointer), valid in
 *       this process; NCCL maps all ranks' windows into one flat range, so
 *       peer_ptrs[rank] is an alias of `base` at another address.  Local (no
 *       communication).
 *       FSDP_ERR_UNSUPPORTED if some rank is outside this rank's NVLink
 *       domain.
 *   fsdp_window_multimem_pointer(ctx, base, &mc): the NVLS multicast address
 *       of the window (ncclGetLsaMultimemPointer of a device communicator
 *       created once per ctx with lsaMultimem; that creation is COLLECTIVE --
 *       the first call must be made by every rank); usable as K10's
 *       mc_staging with `base` as the unicast staging.  FSDP_ERR_UNSUPPORTED
 *       where NCCL gives no multicast mapping (no NVLS).
 * Errors: a ctx without a communicator, `base` not the start of a symmetric
 * window of this ctx -> FSDP_ERR_INVALID_ARG.  (ABI 5) */
fsdp_status fsdp_window_peer_pointers(fsdp_ctx* ctx, const void* base, void** peer_ptrs);
fsdp_status fsdp_window_multimem_pointer(fsdp_ctx* ctx, const void* base, void** mc_ptr);

/* ----------------------------------------------- compute proxy (K7)
 * A measurement device, not a method step: stands in for the layer compute
 * that the paper's reordering overlaps communication with, so that
 * exposed communication is measurable.  `iters` iterations of four
 * independent FMA chains per thread, cut into 16 waves of short CTAs: a grid
 * of 16 x ctas_per_sm CTAs per SM x 256 threads, each CTA holding smem_bytes
 * of dynamic shared memory and running ceil(iters / 16) iterations, so that,
 * like the tiles of a real GEMM, the block scheduler balances it over the SM
 * room a concurrent collective or copy leaves free. */
fsdp_status fsdp_proxy_launch(fsdp_ctx* ctx, int64_t iters, int32_t ctas_per_sm, int32_t smem_bytes,
                              fsdp_stream_t stream);
/* Times fsdp_proxy_launch(iters) on `stream` (median of `reps`) and writes the
 * measured ns; synchronises. */
fsdp_status fsdp_proxy_calibrate(fsdp_ctx* ctx, int64_t iters, int32_t ctas_per_sm, int32_t smem_bytes,
                                 int32_t reps, fsdp_stream_t stream, int64_t* ns_out);

#ifdef __cplusplus
}
#endif
#endif /* FSDP_B200_FSDP_H */
