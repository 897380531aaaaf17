/* SPDX-License-Identifier: Apache-2.0
 *
 * asteria_b200.h — C-ABI of the B200-native Asteria optimizer step.
 *
 * This is the drop-in boundary for the reference's optimizer path
 * (reference: proj/include/asopt/precond.hpp, proj/include/asopt/asyncsched.hpp,
 * proj/src/config.cpp). Every entry point is `extern "C"`, takes plain pointers
 * and sizes, never throws, and returns an asg_status. The message of the last
 * failure on the calling thread is available from asg_last_error().
 *
 * Which reference interface each entry point replaces is cited next to it
 * (path:line relative to the reference's proj/ directory).
 *
 * Device memory convention: parameters (theta) and gradients are caller-owned
 * fp32 device buffers, row-major with an explicit leading dimension. All
 * optimizer state (factors, roots/bases, SOAP moments, shadow snapshots) is
 * owned by an asg_blockset and lives in HBM.
 *
 * Streams are passed as `void*` (a cudaStream_t) so this header does not pull
 * in the CUDA runtime headers. NULL means the blockset's own main stream (a
 * non-blocking stream); to order with the legacy default stream pass
 * cudaStreamLegacy ((void*)0x1), e.g. for torch's default stream (handle 0).
 */
#ifndef ASTERIA_B200_H
#define ASTERIA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASG_API_VERSION 1

/* Status codes: 1:1 with the asopt::Error hierarchy (errors.hpp:10-47) that
 * the optimizer path can raise, plus runtime failures of the GPU layer. */
typedef enum asg_status {
    ASG_OK = 0,
    ASG_ERR_NON_FINITE = 1,          /* NonFiniteError            errors.hpp:16 */
    ASG_ERR_NO_CONVERGENCE = 2,      /* NoConvergenceError        errors.hpp:17 */
    ASG_ERR_NOT_PSD = 3,             /* NotPsdError               errors.hpp:18 */
    ASG_ERR_LAYOUT_MISMATCH = 4,     /* LayoutMismatchError       errors.hpp:19 */
    ASG_ERR_SHAPE_MISMATCH = 5,      /* ShapeMismatchError        errors.hpp:20 */
    ASG_ERR_STALE_UNINITIALIZED = 6, /* StaleUninitializedError   errors.hpp:23 */
    ASG_ERR_WORKER_POOL_DOWN = 7,    /* WorkerPoolDownError       errors.hpp:33 */
    ASG_ERR_CONFIG_INVALID = 8,      /* ConfigInvalidError        errors.hpp:41 */
    ASG_ERR_AUDIT = 9,               /* AuditError                errors.hpp:48 */
    ASG_ERR_MISSING_KEY = 10,        /* MissingKeyError           errors.hpp:27 */
    ASG_ERR_CUDA = 11,               /* CUDA runtime/driver failure            */
    ASG_ERR_OUT_OF_MEMORY = 12,      /* device allocation failed               */
    ASG_ERR_INVALID_ARGUMENT = 13,   /* bad handle / pointer / index           */
    ASG_ERR_UNSUPPORTED = 14,        /* no sm_100a device, or feature absent   */
    ASG_ERR_CAPACITY_EXHAUSTED = 15, /* CapacityExhaustedError    errors.hpp:26 */
    ASG_ERR_IO = 16,                 /* IoError                   errors.hpp:28 */
    ASG_ERR_PINNED_ENTRY = 17,       /* PinnedEntryError          errors.hpp:29 */
    ASG_ERR_DIRTY_NOT_PERSISTED = 18 /* DirtyNotPersistedError    errors.hpp:30 */
} asg_status;

/* Method (precond.hpp:19) extended with KL-Shampoo, which the reference only
 * names as a plug-in point. */
typedef enum asg_method {
    ASG_METHOD_ADAMW = 0,
    ASG_METHOD_SHAMPOO = 1,
    ASG_METHOD_SOAP = 2,
    ASG_METHOD_KL_SHAMPOO = 3
} asg_method;

/* Accumulation (precond.hpp:20). */
typedef enum asg_accumulation { ASG_ACCUM_SUM = 0, ASG_ACCUM_EMA = 1 } asg_accumulation;

/* Arithmetic of the tensor-core GEMMs. 3xTF32 (hi/lo split, three tcgen05
 * kind::tf32 products) is fp32-faithful and is the parity mode. */
typedef enum asg_precision {
    ASG_PREC_3XTF32 = 0,     /* operands stored in HBM as (hi, lo) tf32 pairs */
    ASG_PREC_TF32 = 1,
    ASG_PREC_3XTF32_SMEM = 2, /* the same 3xTF32 products; operands stored as plain fp32 (half the
                                 bytes) and split into (hi, lo) in shared memory after the TMA load */
    ASG_PREC_3XF16 = 3        /* 3xFP16: the step's operands as exact (hi, lo) fp16 pairs with a
                                 per-matrix power-of-two scale (x s = hi + lo to ~2^-22), multiplied by
                                 tcgen05 kind::f16 at twice the tf32 rate; other products as 3XTF32_SMEM */
} asg_precision;

/* Tensor roles (tiers.hpp:35-44) plus the KL-Shampoo inverses and the
 * installed eigenvalues. */
typedef enum asg_role {
    ASG_ROLE_FACTOR_L = 0,
    ASG_ROLE_FACTOR_R = 1,
    ASG_ROLE_INV_L = 2,     /* Shampoo: L^-1/4; KL-Shampoo: L^-1/2 */
    ASG_ROLE_INV_R = 3,
    ASG_ROLE_BASIS_L = 4,   /* SOAP eigenvectors (columns), row-major m x m */
    ASG_ROLE_BASIS_R = 5,
    ASG_ROLE_ROTATED_M = 6,
    ASG_ROLE_ROTATED_V = 7,
    ASG_ROLE_KL_INV_L = 8,  /* KL-Shampoo: L^-1 = INV_L^2 (read-only: derived from the installed root) */
    ASG_ROLE_KL_INV_R = 9,
    ASG_ROLE_EIGVALS_L = 10, /* SOAP installed eigenvalues (ascending) */
    ASG_ROLE_EIGVALS_R = 11
} asg_role;

/* OptimizerConfig (precond.hpp:27-44); JSON keys config.cpp:71-80. */
typedef struct asg_optimizer_config {
    int32_t method;        /* asg_method */
    int32_t accumulation;  /* asg_accumulation */
    double lr;
    double beta1;
    double beta2;
    double eps;
    double weight_decay;
    int64_t precondition_frequency; /* pf */
    double damping;                 /* relative: eps_eff = damping * tr/dim */
    int64_t block_dim_limit;
} asg_optimizer_config;

/* Refresh-install policy of the shadow pipeline. */
typedef enum asg_install_mode {
    /* Reference semantics: a job dispatched at simulated time T with cost C is
     * installable at T + C on the blockset's simulated clock
     * (asyncsched.hpp:7-11, asyncsched.cpp:118-127,268-274). Deterministic. */
    ASG_INSTALL_SIM_CLOCK = 0,
    /* Free-running: a job is installable at StepEnd once its side-stream event
     * has completed. Not bit-reproducible; the bounded-staleness barrier
     * (asyncsched.cpp:191-221) still applies. */
    ASG_INSTALL_EVENT = 1
} asg_install_mode;

/* Arithmetic of the refresh (compute_refresh precond.cpp:129-142).
 *   F64: fp64 eigensolve of the fp32 factor snapshot to the reference's own
 *        stopping rule off(A) <= 1e-12 ||A||_F (densela.hpp:192-203); roots
 *        and SOAP re-projections in fp64. Reference-tight (parity mode).
 *   F32: fp32-level refresh, the fast path. The snapshot is rotated into the
 *        block's previous eigenbasis on the tensor cores (3xTF32:
 *        B = Q^T A Q), a Jacobi eigensolve of B stops once every element obeys
 *        |b_ij| <= 1e-6 * max(sqrt(b_ii b_jj), ||A||_F / sqrt(n)), and the new
 *        basis Q J, the roots V f(lambda) V^T and the SOAP moment
 *        re-projection J^T M J are 3xTF32 tensor-core GEMMs. Accuracy is that
 *        of the fp32 factor it decomposes. */
/*   NEWTON: as F32, except that the Shampoo (L^-1/4) and KL-Shampoo (L^-1/2,
 *        L^-1) roots come from a coupled Newton-Schulz iteration on the
 *        tensor cores (GEMMs only, no eigendecomposition; asg_newton.cu) of
 *        the damped snapshot (A + eps I), eps = damping * tr/n. Same result
 *        as inv_root (densela.hpp:267-282) to fp32 level; SOAP, which needs
 *        the eigenbasis itself, keeps the F32 eigensolve. */
typedef enum asg_refresh_mode { ASG_REFRESH_F64 = 0, ASG_REFRESH_F32 = 1, ASG_REFRESH_NEWTON = 2 } asg_refresh_mode;

/* SchedulerConfig (asyncsched.hpp:50-59); JSON keys config.cpp:81-86. */
typedef struct asg_scheduler_config {
    int64_t staleness_S;
    int64_t pf;
    int32_t pool_size;     /* accepted for schema compatibility; refresh runs on a side stream */
    int32_t drain_budget;  /* staged tier-store transfers installed per ForwardPost (asg_on_hook) */
    double inject_job_delay_steps;
    double inject_job_delay_jitter_steps;
    double step_compute_us;
    double install_cost_us;
    int32_t install_mode;  /* asg_install_mode */
    int32_t refresh_mode;  /* asg_refresh_mode (default F64) */
} asg_scheduler_config;

/* BlockSpec (precond.hpp:47-57). param_index identifies the parameter. */
typedef struct asg_block_spec {
    int64_t param_index;
    int64_t row_begin, row_end;
    int64_t col_begin, col_end;
    int64_t block_dim_limit;
} asg_block_spec;

/* One caller-owned parameter: fp32 device buffers, row-major. */
typedef struct asg_param_desc {
    float* theta;
    const float* grad;
    int64_t rows, cols;
    int64_t ld_theta, ld_grad;
} asg_param_desc;

/* FreshnessRecord (asyncsched.hpp:72-78); -1 encodes "no pending job". */
typedef struct asg_freshness {
    uint64_t installed_version;
    int64_t dispatch_step_of_pending;
    int64_t last_install_step;
    int64_t installed_snapshot_step;
} asg_freshness;

/* PoolStats (asyncsched.hpp:61-70). */
typedef struct asg_pool_stats {
    uint64_t dispatched, completed, installed, coalesced, barrier_waits;
    double wait_total_us;
    int32_t pending, queue_depth;
} asg_pool_stats;

/* PrecondBlock bookkeeping (precond.hpp:63-75). */
typedef struct asg_block_info {
    asg_block_spec spec;
    uint64_t version;
    int64_t last_refresh_step;
    int64_t moment_steps;
    int32_t owner_rank;
    int32_t use_adamw; /* 1-D / degenerate parameter: AdamW fallback (harness.cpp:352) */
} asg_block_info;

/* Schedule trace event kinds (subset of trace.hpp TraceEventKind). */
typedef enum asg_event_kind {
    ASG_EV_DISPATCH = 0,
    ASG_EV_JOB_START = 1,
    ASG_EV_JOB_DONE = 2,
    ASG_EV_INSTALL = 3,
    ASG_EV_BARRIER_WAIT_BEGIN = 4,
    ASG_EV_BARRIER_WAIT_END = 5,
    ASG_EV_PREFETCH = 6, /* tier-store staging of inverse state (trace.hpp:25, asyncsched.cpp:183,261) */
    ASG_EV_DRAIN = 7     /* a staged transfer installed at ForwardPost (asyncsched.cpp:240) */
} asg_event_kind;

typedef struct asg_event {
    int64_t step;
    int32_t kind;   /* asg_event_kind */
    int32_t reserved;
    int64_t block;  /* block index within the blockset */
    uint64_t version;
    double t_us;
} asg_event;

typedef struct asg_blockset asg_blockset;

/* ---- library ----------------------------------------------------------- */
const char* asg_last_error(void);
int asg_api_version(void);
/* 1 if a device with compute capability 10.0 is visible, else 0. */
int asg_device_supported(int device);

/* ---- configuration (precond.cpp:34-62, config.cpp:121-149) -------------- */
int asg_optimizer_defaults(int32_t method, asg_optimizer_config* out);      /* OptimizerConfig::defaults_for precond.cpp:44-62 */
int asg_optimizer_validate(const asg_optimizer_config* cfg);                /* OptimizerConfig::validate     precond.cpp:34-42 */
int asg_scheduler_defaults(asg_scheduler_config* out);                      /* SchedulerConfig{}             asyncsched.hpp:50-59 */
/* Parses the "optimizer" and "async" sections of a RunConfig JSON document;
 * other sections are ignored, as read_if ignores unknown keys (config.cpp:12-15).
 * Method defaults apply before field overrides (config.cpp:126-127);
 * async.pf defaults to optimizer.precondition_frequency (config.cpp:140) and
 * must equal it (config.cpp:42-43). Method strings: "AdamW", "Shampoo",
 * "SOAP", "KL-Shampoo". An optional "gpu" section may set "precision"
 * ("3xtf32"|"tf32"), "install_mode" ("sim_clock"|"event") and "refresh"
 * ("f64"|"f32"|"newton"). */
int asg_config_from_json(const char* json, asg_optimizer_config* opt,
                         asg_scheduler_config* sched, int32_t* precision);

/* ---- blocking (precond.cpp:69-82) --------------------------------------- */
/* Writes up to `capacity` specs; *count receives the total. */
int asg_partition_param(int64_t param_index, int64_t rows, int64_t cols, int64_t limit,
                        asg_block_spec* out, int64_t capacity, int64_t* count);

/* ---- blockset lifecycle ------------------------------------------------- */
/* Partitions every parameter with cfg->block_dim_limit, creates a
 * PrecondBlock per block (PrecondBlock::create precond.cpp:84-110) with all
 * state resident on `device`, and assigns each block one owner rank by LPT
 * over (world, rank). 1-D parameters (rows==1 or cols==1) use AdamW
 * (harness.cpp:352). `seed` keys the scheduler's jitter stream
 * (asyncsched.cpp:248). */
int asg_blockset_create(int device, const asg_optimizer_config* opt,
                        const asg_scheduler_config* sched, const asg_param_desc* params,
                        int64_t n_params, int32_t precision, int32_t rank, int32_t world,
                        uint64_t seed, asg_blockset** out);
int asg_blockset_destroy(asg_blockset* bs);
/* Rebinds theta/grad device pointers (same shapes). */
int asg_blockset_bind_params(asg_blockset* bs, const asg_param_desc* params, int64_t n_params);
int asg_blockset_num_blocks(const asg_blockset* bs, int64_t* n);
int asg_blockset_block_info(const asg_blockset* bs, int64_t idx, asg_block_info* out);
/* Bytes of optimizer state resident in HBM (every device allocation of the
 * blockset except the refresh workspace). */
int asg_blockset_state_bytes(const asg_blockset* bs, uint64_t* bytes);
/* Bytes of the refresh / install workspace (chunked; independent of the
 * block count above one chunk). */
int asg_blockset_workspace_bytes(const asg_blockset* bs, uint64_t* bytes);
/* The blockset's main stream (cudaStream_t) for callers that want to order
 * their own work with it. */
int asg_blockset_stream(const asg_blockset* bs, void** stream);

/* ---- the optimizer step (harness.cpp:439-475 per-block call order) ------ */
/* Global gradient squared norm over every parameter (feeds clip_scale,
 * harness.cpp:219-223,435) and a non-finite flag. Synchronizes the stream. */
int asg_grad_sqnorm(asg_blockset* bs, void* stream, double* sqnorm, int32_t* nonfinite);
/* accumulate_factors (precond.cpp:173-189) for every owned block on
 * clip_scale * grad. KL-Shampoo uses the installed inverses. */
int asg_accumulate(asg_blockset* bs, double clip_scale, void* stream);
/* ShadowScheduler::maybe_dispatch (asyncsched.cpp:108-142) for every owned
 * block: snapshot (snapshot_factors precond.cpp:112-117) and launch the
 * refresh (compute_refresh precond.cpp:129-142) on the low-priority side
 * stream. */
int asg_maybe_dispatch(asg_blockset* bs, int64_t step, int64_t* n_dispatched);
/* ShadowScheduler::staleness_barrier (asyncsched.cpp:191-221). */
int asg_staleness_barrier(asg_blockset* bs, int64_t step, double* waited_us);
/* Cold-start rule (harness.cpp:455-466) + precondition_{shampoo,soap}
 * (precond.cpp:191-223) + apply_update (precond.cpp:244-251), fused, for
 * every owned block; AdamW (precond.cpp:229-242) for 1-D parameters. */
int asg_precondition_apply(asg_blockset* bs, int64_t step, double clip_scale, double lr_scale,
                           void* stream);
/* on_hook(StepEnd) (asyncsched.cpp:268-286): installs ready refreshes. */
int asg_step_end(asg_blockset* bs, int64_t step);
/* accumulate -> maybe_dispatch -> staleness_barrier -> precondition/apply ->
 * StepEnd, for one step. */
int asg_step(asg_blockset* bs, int64_t step, double clip_scale, double lr_scale, void* stream);
/* Advances the simulated clock (SimClock::advance asyncsched.hpp:33-36). */
int asg_clock_advance(asg_blockset* bs, double us);
int asg_get_freshness(const asg_blockset* bs, int64_t idx, asg_freshness* out);
int asg_get_stats(const asg_blockset* bs, asg_pool_stats* out);
/* Copies up to `capacity` schedule events; *count receives the total. */
int asg_get_events(const asg_blockset* bs, asg_event* out, int64_t capacity, int64_t* count);
int asg_synchronize(asg_blockset* bs);

/* ---- per-block entry points (parity tests; host fp64 in/out) ------------ */
/* These mirror the per-block functions of precond.hpp for one block. */
int asg_block_read(asg_blockset* bs, int64_t idx, int32_t role, double* out, int64_t count);
int asg_block_write(asg_blockset* bs, int64_t idx, int32_t role, const double* in, int64_t count);
int asg_block_set_counters(asg_blockset* bs, int64_t idx, uint64_t version,
                           int64_t last_refresh_step, int64_t moment_steps);
/* accumulate_factors(block, g, cfg) precond.cpp:173-189 */
int asg_block_accumulate_f64(asg_blockset* bs, int64_t idx, const double* g, int64_t ld);
/* refresh_inverse = install_refresh(compute_refresh(snapshot_factors(b)), step)
 * precond.cpp:166-171, synchronous. */
int asg_block_refresh_f64(asg_blockset* bs, int64_t idx, int64_t step);
/* precondition_shampoo precond.cpp:191-198 (also KL-Shampoo's L^-1/2 G R^-1/2) */
int asg_block_precondition_f64(asg_blockset* bs, int64_t idx, const double* g, int64_t ld,
                               double* out);
/* soap_scaled_step precond.cpp:208-223 (updates rotated moments) */
int asg_block_soap_step_f64(asg_blockset* bs, int64_t idx, const double* g, int64_t ld,
                            double* out);

/* ---- the split refresh (precond.hpp:77-98) ------------------------------
 * snapshot_factors (precond.cpp:112-117): device copies of a block's L and R;
 * its checksum is the reference's snapshot_checksum (precond.cpp:114-115,
 * FNV-1a bytes.hpp:14-22) over the fp32 factor bytes, for isolation audits.
 * compute_refresh (precond.cpp:129-142) is pure over the snapshot (the block's
 * own factors and installed state are untouched; synchronous). install_refresh
 * (precond.cpp:144-164) consumes the result: roots swapped in (Shampoo /
 * KL-Shampoo) or, for SOAP, rot = Q_new^T Q_old applied to the moments and
 * the bases swapped; version += 1, last_refresh_step = step. The block must
 * have no scheduled (maybe_dispatch) refresh in flight. */
typedef struct asg_snapshot asg_snapshot;
typedef struct asg_refresh_result asg_refresh_result;
int asg_snapshot_factors(asg_blockset* bs, int64_t idx, asg_snapshot** out);
int asg_snapshot_checksum(const asg_snapshot* snap, uint64_t* checksum);
int asg_snapshot_destroy(asg_snapshot* snap);
int asg_compute_refresh(asg_blockset* bs, const asg_snapshot* snap, asg_refresh_result** out);
int asg_install_refresh(asg_blockset* bs, int64_t idx, asg_refresh_result* result, int64_t step);
int asg_refresh_result_destroy(asg_refresh_result* result);
/* replicated_state / load_replicated_state (precond.cpp:253-279): flat
 * [L side m*m | R side n*n] of the inverse roots (Shampoo, KL-Shampoo) or the
 * eigenbases (SOAP), host fp64. */
int asg_block_replicated_state(asg_blockset* bs, int64_t idx, double* out, int64_t count);
int asg_block_load_replicated_state(asg_blockset* bs, int64_t idx, const double* in, int64_t count);
/* pack_spd / unpack_spd (densela.hpp:124-142): lower triangle packed row-major
 * ((0,0), (1,0), (1,1), (2,0), ...), n(n+1)/2 entries per matrix; fp32 device
 * buffers, batched. */
int asg_pack_spd_f32(const float* A, int64_t batch, int64_t n, float* packed, void* stream);
int asg_unpack_spd_f32(const float* packed, int64_t batch, int64_t n, float* A, void* stream);

/* adamw_step (precond.cpp:229-242) and apply_update (precond.cpp:244-251) with
 * host matrices (the step fuses both into its kernels; these are the
 * per-call entry points). AdamState: fp32 moments in HBM. adamw_step returns
 * the bias-corrected direction and throws NonFinite on a non-finite gradient
 * before touching the state; apply_update: theta -= lr*lr_scale*(u + wd*theta)
 * (fp64), NonFinite on a non-finite update before touching theta. */
typedef struct asg_adam_state asg_adam_state;
int asg_adam_state_create(int64_t rows, int64_t cols, asg_adam_state** out);
int asg_adam_state_destroy(asg_adam_state* st);
int asg_adamw_step_f64(asg_adam_state* st, const double* g, const asg_optimizer_config* cfg, double* out);
int asg_apply_update_f64(double* theta, const double* update, int64_t rows, int64_t cols,
                         const asg_optimizer_config* cfg, double lr_scale);

/* ---- multi-GPU: ownership sharding + parameter all-gather ---------------- */
/* Host-only ownership plan (no device needed): partitions every parameter with
 * opt->block_dim_limit (precond.cpp:69-82) and assigns each unit (block, or a
 * whole 1-D AdamW parameter) to one of `world` ranks by LPT on its per-step
 * cost. Units are enumerated exactly as asg_blockset_create does; owner[i]
 * receives the rank of unit i (capacity >= *count). */
int asg_plan_owners(const asg_optimizer_config* opt, const int64_t* rows, const int64_t* cols,
                    int64_t n_params, int32_t world, int32_t* owner, int64_t capacity, int64_t* count);
/* Elements per rank segment of the owner-major exchange buffers (the largest
 * shard); asg_unpack_gathered with this stride uses precomputed offsets. */
int asg_gather_stride(const asg_blockset* bs, int64_t* stride);
/* Data-parallel gradients -> owners ("next" row F1; harness.cpp:417-436): packs
 * every unit's gradient slice owner-major (rank r's units at r * stride, zero
 * padding) into `sendbuf` [world * stride] for a reduce-scatter (SUM) ... */
int asg_pack_grads(asg_blockset* bs, float* sendbuf, void* stream);
/* ... and writes this rank's reduced segment `recvbuf` [stride], times `scale`
 * (1/world for the reference's average, simnet allreduce_avg), into its owned
 * gradient slices. */
int asg_unpack_reduced_grads(asg_blockset* bs, const float* recvbuf, float scale, void* stream);
/* Squared norm over this rank's owned gradient slices (sum over ranks = the
 * global clip norm, harness.cpp:219-223); synchronizes the stream. */
int asg_grad_sqnorm_owned(asg_blockset* bs, void* stream, double* sqnorm, int32_t* nonfinite);
/* Elements of theta owned by `rank` (owner-major layout). */
int asg_shard_elems(const asg_blockset* bs, int32_t rank, int64_t* elems);
/* Packs this rank's owned block slices of theta into `sendbuf` (device). */
int asg_pack_owned(asg_blockset* bs, float* sendbuf, void* stream);
/* Scatters an all-gathered owner-major buffer (ranks concatenated, each
 * padded to `stride_elems`) back into every parameter. */
int asg_unpack_gathered(asg_blockset* bs, const float* recvbuf, int64_t stride_elems, void* stream);

/* ---- bucketed parameter all-gather over NCCL --------
 * Every shape's units are split into `buckets_per_shape` runs per rank; bucket
 * (shape, c) holds run c of every rank (1-D AdamW parameters: one bucket). The
 * plan depends only on the ownership plan, so all ranks hold the same list.
 * Exchange buffer of a bucket: [world][stride] fp32, rank r's updated slices
 * at r * stride (asg_bucket_stride). */
int asg_set_allgather_buckets(asg_blockset* bs, int32_t buckets_per_shape);
int asg_bucket_count(const asg_blockset* bs, int64_t* count);
int asg_bucket_stride(const asg_blockset* bs, int64_t bucket, int64_t* stride);
/* Packs this rank's updated slices of bucket `bucket` into sendbuf [stride]. */
int asg_bucket_pack(asg_blockset* bs, int64_t bucket, float* sendbuf, void* stream);
/* Scatters an all-gathered bucket buffer [world][stride] into every parameter. */
int asg_bucket_unpack(asg_blockset* bs, int64_t bucket, const float* recvbuf, void* stream);
/* NCCL is loaded at run time (libnccl.so.2). The unique id is 128 bytes
 * (NCCL_UNIQUE_ID_BYTES); rank 0 creates it, the caller distributes it. The
 * communicator is a ncclComm_t passed as void*, created on the current
 * device. */
int asg_nccl_unique_id(uint8_t* out);
int asg_nccl_comm_init(int32_t world, int32_t rank, const uint8_t* id, void** comm);
int asg_nccl_comm_destroy(void* comm);
/* After asg_step: all-gathers every bucket over `comm` (ncclAllGather) on
 * `stream` (ordered after the step) and scatters into every parameter. */
int asg_allgather_params(asg_blockset* bs, void* comm, void* stream);
/* Fused variant: with a communicator set (NULL unsets), asg_step /
 * asg_precondition_apply update the blocks bucket by bucket and all-gather
 * bucket b on a high-priority communication stream while the main stream
 * updates bucket b+1; the step ends (on the main stream) after the last
 * bucket's scatter. */
int asg_set_allgather_comm(asg_blockset* bs, void* comm, int32_t buckets_per_shape);

/* ---- profiling ---------------------------------------------------------- */
typedef struct asg_kernel_stats {
    uint64_t launches;       /* kernels this library launched (process-wide counter delta) */
    uint64_t gemm_launches;  /* tcgen05 GEMM launches recorded while profiling */
    double gemm_alg_flops;   /* algorithmic flops of those launches (SYRK: n^2 k, GEMM: 2 m n k) */
    double gemm_ms;          /* sum of their CUDA-event durations on the launching stream */
} asg_kernel_stats;
/* HBM-bound kernels of the step, timed while profiling (CUDA events on their
 * launching stream), with their algorithmic bytes: the gradient prep
 * (gather + clip scale + tf32 split + transpose; 4 B read + 16 B written per
 * element), the clip norm (4 B/elt, harness.cpp:219-223) and the multi-tensor
 * AdamW (28 B/elt, precond.cpp:229-251). */
typedef enum asg_hbm_kind { ASG_HBM_PREP = 0, ASG_HBM_SQNORM = 1, ASG_HBM_ADAMW = 2, ASG_HBM_KINDS = 3 } asg_hbm_kind;
typedef struct asg_hbm_stats {
    uint64_t launches[ASG_HBM_KINDS];
    double bytes[ASG_HBM_KINDS];
    double ms[ASG_HBM_KINDS];
} asg_hbm_stats;
/* Synchronizes the device, returns the HBM-kernel stats since the last reset. */
int asg_get_hbm_stats(asg_blockset* bs, asg_hbm_stats* out, int32_t reset);
/* Process-wide count of kernel launches issued by this library (graph
 * replays count the kernels of one pass through the graph; sweeps repeated by
 * a device-driven WHILE loop are not counted again). */
int asg_launch_count(uint64_t* count);
/* While enabled, every GEMM launch is bracketed by CUDA events on its stream. */
int asg_profile_enable(asg_blockset* bs, int32_t enable);
/* Synchronizes, returns the stats accumulated since the last reset. */
int asg_get_kernel_stats(asg_blockset* bs, asg_kernel_stats* out, int32_t reset);


/* ---- tiered store of optimizer state (F3; tierstore.hpp, tierstore.cpp) ---
 * Keyed tensors ("block_id/role") across three tiers, with the reference's
 * semantics: byte-accurate residency gauges, least-recently-touched eviction
 * one tier down, pinning, explicit flush/reclaim, an append-only cold file in
 * the reference's bit-exact ASTRCOLD format (tierstore.hpp:8-13), and
 * asynchronous prefetch by a transfer worker whose completed copies are
 * installed only by drain_ready (never blocking on incomplete ones).
 * B200 mapping: Hot = device memory (HBM) of `hot_device`, Host = pinned host
 * memory, Cold = the file. Host<->Hot moves are DMA copies on the store's own
 * copy stream; a prefetch to Hot is staged by the worker thread (file read ->
 * pinned -> cudaMemcpyAsync into a stream-ordered device allocation) so the
 * training thread never waits for the link. hot_device = -1 keeps the Hot
 * tier in host memory (bookkeeping-only hosts without a GPU). */
typedef enum asg_tier { ASG_TIER_HOT = 0, ASG_TIER_HOST = 1, ASG_TIER_COLD = 2 } asg_tier;

typedef struct asg_store_config {           /* StoreConfig tierstore.hpp:33-39 */
    uint64_t hot_capacity_bytes;            /* default 1 GiB */
    uint64_t host_capacity_bytes;           /* default 1 GiB */
    const char* cold_path;                  /* required */
    double transfer_bandwidth_bytes_per_sec; /* injected link model; 0 = unthrottled */
    uint64_t transfer_latency_us;
    int32_t hot_device;                     /* CUDA device of the Hot tier; -1: host memory */
} asg_store_config;

typedef struct asg_entry_view {             /* EntryView tierstore.hpp:61-69 */
    int32_t tier;
    uint64_t bytes;
    int32_t dirty, pinned;
    int64_t last_touch_step;
    int32_t staged_pending, staged_ready;
} asg_entry_view;

typedef struct asg_residency {              /* ResidencyGauges tierstore.hpp:41-45 */
    uint64_t hot_bytes, host_bytes, cold_bytes;
} asg_residency;

typedef struct asg_io_counters {            /* IoCounters tierstore.hpp:47-59 */
    uint64_t file_writes, file_reads, write_skips, page_ins, evictions, prefetch_requests, transfers_started,
        transfers_coalesced, transfers_completed, transfers_dropped, drains_installed;
} asg_io_counters;

typedef struct asg_tierstore asg_tierstore;

/* Fills the reference's defaults (tierstore.hpp:33-39; cold_path NULL, hot_device -1). */
int asg_store_config_defaults(asg_store_config* out);
/* TierStore::TierStore tierstore.cpp:24-43: truncates/creates the cold file and writes its header. */
int asg_tierstore_create(const asg_store_config* cfg, asg_tierstore** out);
int asg_tierstore_destroy(asg_tierstore* st);
/* Keys are (block_id, role): role is an asg_role (TensorRole tiers.hpp:35-44). */
/* put tierstore.cpp:169-211 (bytes: host memory) */
int asg_tier_put(asg_tierstore* st, const char* block_id, int32_t role, const void* bytes, uint64_t size, int32_t tier,
                 asg_entry_view* out);
/* put from device memory (the Hot-tier source of a blockset's state: no host round trip for Hot puts) */
int asg_tier_put_device(asg_tierstore* st, const char* block_id, int32_t role, const void* dev_bytes, uint64_t size,
                        int32_t tier, asg_entry_view* out);
/* get tierstore.cpp:213-229: copies the payload to host `out` (capacity `cap`;
 * *size receives the payload size even when cap is too small -> ShapeMismatch);
 * a Cold entry is paged in to Host. */
int asg_tier_get(asg_tierstore* st, const char* block_id, int32_t role, void* out, uint64_t cap, uint64_t* size,
                 int32_t* tier);
/* Device address of a Hot entry's payload (valid until the entry moves). */
int asg_tier_device_ptr(asg_tierstore* st, const char* block_id, int32_t role, void** dev_ptr);
int asg_tier_demote(asg_tierstore* st, const char* block_id, int32_t role, int32_t to);   /* :231-234 */
int asg_tier_promote(asg_tierstore* st, const char* block_id, int32_t role, int32_t to);  /* :236-257 */
int asg_tier_reclaim(asg_tierstore* st, const char* block_id, int32_t role, uint64_t* freed); /* :259-273 */
int asg_tier_flush(asg_tierstore* st, const char* block_id, int32_t role);                 /* :275-282 */
int asg_tier_pin(asg_tierstore* st, const char* block_id, int32_t role);
int asg_tier_unpin(asg_tierstore* st, const char* block_id, int32_t role);
/* prefetch tierstore.cpp:294-308: returns at once; duplicates coalesce onto one ticket */
int asg_tier_prefetch(asg_tierstore* st, const char* block_id, int32_t role, int32_t to, uint64_t* ticket);
/* drain_ready tierstore.cpp:404-420 */
int asg_tier_drain_ready(asg_tierstore* st, int32_t max_items, int32_t* installed);
int asg_tier_advance_step(asg_tierstore* st, int64_t step);
int asg_tier_contains(asg_tierstore* st, const char* block_id, int32_t role, int32_t* out);
int asg_tier_inspect(asg_tierstore* st, const char* block_id, int32_t role, asg_entry_view* out);
int asg_tier_gauges(asg_tierstore* st, asg_residency* out);
int asg_tier_counters(asg_tierstore* st, asg_io_counters* out);
/* audit tierstore.cpp:437-456: ASG_ERR_AUDIT on any mismatch */
int asg_tier_audit(asg_tierstore* st);

/* The scheduler side of the store (ShadowScheduler with a TierStore,
 * asyncsched.hpp:117-119): once attached, every scheduler install writes the
 * block's refreshed inverse state (INV_L/R; SOAP: BASIS_L/R) to the Host tier
 * and prefetches it toward Hot (asyncsched.cpp:164-184); the store is not
 * owned. NULL detaches. */
int asg_blockset_attach_store(asg_blockset* bs, asg_tierstore* store);
/* HookEvent kinds (asyncsched.hpp): ForwardPost drains at most drain_budget staged
 * transfers enqueued before `step`; BackwardPre prefetches Cold inverse state
 * to Host; StepEnd is asg_step_end (asyncsched.cpp:223-286). */
typedef enum asg_hook { ASG_HOOK_FORWARD_POST = 0, ASG_HOOK_BACKWARD_PRE = 1, ASG_HOOK_STEP_END = 2 } asg_hook;
int asg_on_hook(asg_blockset* bs, int32_t kind, int64_t step);

/* Benchmark input: overwrites the gradient slice of every unit
 * this rank owns with N(0, 1/cols(param)) i.i.d. values from Philox4x32-10
 * keyed (seed, step, unit) -- one launch on `stream` (NULL: the main stream).
 * Not part of the optimizer step; the caller's gradient buffers are written. */
int asg_synth_gradients(asg_blockset* bs, uint64_t seed, int64_t step, void* stream);

/* ---- diagnostics: the tensor-core GEMM on its own ----------------------- */
/* C[b] = alpha * A[b] * B[b]^T + beta * C[b] for b < batch, fp32 device
 * slabs: A is [batch][M][K], B is [batch][N][K], C is [batch][M][N]
 * (row-major). M, N multiples of 128, K multiple of 32. Runs the same
 * tcgen05 kernel the optimizer step uses. */
int asg_gemm_tn(const float* A, const float* B, float* C, int64_t batch, int64_t M, int64_t N,
                int64_t K, float alpha, float beta, int32_t precision, void* stream);
/* Batched symmetric eigendecomposition (the refresh kernel): values
 * ascending, vectors as columns, fp64 device buffers [batch][n][n]. */
int asg_sym_eig_batched(const double* A, double* values, double* vectors, int64_t batch, int64_t n,
                        void* stream);
/* The F32 refresh's tensor-core block Jacobi on its own: fp32 device buffers
 * A [batch][n][n] (symmetric), vectors [batch][n][n] (columns), fp64 values
 * [batch][n] ascending; n > 64. Same stopping rule as ASG_REFRESH_F32.
 * Works in chunks on a per-device scratch arena that persists between calls
 * (calls on one device serialise on it); synchronizes the stream. */
int asg_sym_eig_batched_f32(const float* A, double* values, float* vectors, int64_t batch, int64_t n,
                            void* stream);
/* The NEWTON refresh's inverse root on its own (inv_root densela.hpp:267-282
 * with relative_damping precond.cpp:121-125): out[b] = (A[b] + eps_b I)^(-1/p),
 * eps_b = damping * tr(A[b]) / n, p in {2, 4}, by coupled Newton-Schulz
 * iterations on the tensor cores. fp32 device buffers [batch][n][n], n <= 4096;
 * precision: asg_precision of the iterates and products (ASG_PREC_3XF16: scaled
 * fp16 pairs at spectral-bound scales; 3XTF32 / 3XTF32_SMEM: tf32 pairs; TF32).
 * Chunked on the same scratch arena as asg_sym_eig_batched_f32; synchronizes
 * the stream. */
int asg_inv_root_batched_f32(const float* A, float* out, int64_t batch, int64_t n, int32_t p, double damping,
                             int32_t precision, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* ASTERIA_B200_H */
