/*
 * gsot.h — C ABI of the B200 group-sparse OT dual solver (libgsot.so).
 *
 * Drop-in boundary for the hot path of the reference library `groupot`
 * (/root/reference/proj/include/groupot). Every entry point names the
 * reference interface it replaces. Plain pointers and sizes only; all
 * pointers are HOST memory unless the name ends in `_device`.
 *
 *  reference (C++, Eigen)                          this ABI
 *  ----------------------------------------------  -------------------------
 *  ProblemInstance + validate_instance             gsot_create / gsot_create_device
 *    core.hpp:47-55, :117-139
 *  RegParams(gamma, mu)         core.hpp:59-75     gsot_create, gsot_set_params
 *  params_from_rho              core.hpp:148-151   gsot_params_from_rho
 *  ObjectiveFn + GradientFn closures               gsot_eval (one fused call)
 *    solver.hpp:101-120 / :161-210, lbfgs.hpp:32-33
 *  dual_objective               dual.hpp:38-52     gsot_eval (objective out)
 *  dual_gradient + ColumnGradFn dual.hpp:54-100    gsot_eval (grad out)
 *  FastGradDispatcher::init     screening.hpp:220  gsot_init_snapshot
 *  FastGradDispatcher::refresh  screening.hpp:231  gsot_refresh
 *  take_snapshot                screening.hpp:24   gsot_refresh / gsot_snapshot_norms
 *  build_active_set             screening.hpp:147  gsot_refresh / gsot_active_set
 *  GradStats::PerCall           screening.hpp:181  gsot_call_stats
 *  recover_plan                 dual.hpp:116-128   gsot_plan_columns (column-streamed)
 *  plan nonzero blocks          dual.hpp:139-169   gsot_block_mask
 *  plan_diagnostics(recover_plan) dual.hpp:130-169 gsot_plan_diagnostics
 *  primal_objective(recover_plan) core.hpp:153-180  gsot_primal_objective
 *  solve / solve_baseline /     solver.hpp:92-293  gsot_solve
 *    solve_fast / audit_solve
 *  SolverOptions, Solution      solver.hpp:25-42   gsot_solver_options, gsot_solve_result
 *
 * Error convention: every function returns a gsot_status. The reference's
 * exception classes (errors.hpp) map one-to-one onto status codes; the
 * message and the exception's fields (NegativeCost::row/col/value,
 * MarginalNotNormalized::which/index) are available from the calling thread
 * through gsot_last_error() / gsot_last_error_detail(). Line-search failure
 * is NOT an error (lbfgs.hpp:29, solver.hpp:41): it is a result flag.
 *
 * Threading: one context owns one CUDA stream and is not reentrant (the
 * reference dispatcher is stateful and single-threaded, screening.hpp:206).
 * Calls are synchronous with respect to the host buffers they take.
 *
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point returns GSOT_ERR_CUDA.
 */
#ifndef GSOT_H
#define GSOT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GSOT_API __attribute__((visibility("default")))
#else
#define GSOT_API
#endif

typedef enum gsot_status {
  GSOT_OK = 0,
  GSOT_ERR_DIMENSION_MISMATCH = 1,      /* errors.hpp:14-18 DimensionMismatch */
  GSOT_ERR_NEGATIVE_COST = 2,           /* errors.hpp:20-31 NegativeCost */
  GSOT_ERR_MARGINAL_NOT_NORMALIZED = 3, /* errors.hpp:33-41 MarginalNotNormalized */
  GSOT_ERR_PARTITION_MISMATCH = 4,      /* errors.hpp:43-47 PartitionMismatch */
  GSOT_ERR_INVALID_ARGUMENT = 5,        /* errors.hpp:9-12 Error (RegParams, core.hpp:61-66) */
  GSOT_ERR_RHO_OUT_OF_RANGE = 6,        /* errors.hpp:49-56 RhoOutOfRange (detail.value = rho) */
  GSOT_ERR_AUDIT_VIOLATION = 7,         /* errors.hpp:85-89 AuditViolation */
  GSOT_ERR_CUDA = 8,                    /* no device / CUDA runtime failure */
  GSOT_ERR_OUT_OF_MEMORY = 9,
  GSOT_ERR_STATE = 10 /* call order violated (e.g. screened eval before a snapshot) */
} gsot_status;

typedef struct gsot_ctx gsot_ctx;

/* Fields of the last error raised on this thread (errors.hpp field layout). */
typedef struct gsot_error_detail {
  int32_t status;
  int64_t row, col; /* NegativeCost */
  double value;     /* NegativeCost */
  char which;       /* MarginalNotNormalized: 'a' or 'b' */
  int64_t index;    /* MarginalNotNormalized: first offending index, -1 = sum */
} gsot_error_detail;

GSOT_API const char* gsot_last_error(void);
GSOT_API int gsot_last_error_detail(gsot_error_detail* out);
GSOT_API const char* gsot_version(void);

/* core.hpp:148-151: gamma_eff = gamma*(1-rho), mu_eff = rho/(1-rho). */
GSOT_API int gsot_params_from_rho(double gamma, double rho, double* gamma_eff, double* mu_eff);

/* ProblemInstance + RegParams + validate_instance (core.hpp:117-139).
 * cost: m x n column-major (the reference's Eigen::MatrixXd layout), host
 * memory; a: m, b: n; group_sizes: L contiguous row blocks (GroupPartition,
 * core.hpp:17-43). Validation order and first-offender semantics follow the
 * reference (GroupPartition ctor, RegParams ctor, then cost j-major scan,
 * marginal a, marginal b, partition cover). The cost is copied to HBM in
 * the group-padded layout. */
GSOT_API int gsot_create(const double* cost, int64_t m, int64_t n, const int32_t* group_sizes,
                         int32_t L, const double* a, const double* b, double gamma, double mu,
                         gsot_ctx** out);
/* Same, with `d_cost` a DEVICE pointer (m x n column-major). */
GSOT_API int gsot_create_device(const double* d_cost, int64_t m, int64_t n,
                                const int32_t* group_sizes, int32_t L, const double* a,
                                const double* b, double gamma, double mu, gsot_ctx** out);
/* Release a context. Contexts made by gsot_create / gsot_create_device park
 * their device state (buffers, stream, captured graphs) in a small
 * process-wide cache; a later create of the same shape and partition on the
 * same device reuses it and only uploads the new data. GSOT_CTX_CACHE=0 in the
 * environment frees immediately instead. */
/* A column shard of a larger instance (multi-GPU column sharding, DESIGN.md
 * §8): cost is the m x n_shard column block (column-major), b_shard the
 * shard's entries of b, a the row marginal or zeros. Validated like
 * gsot_create except that the marginals are checked entrywise only (their
 * sums are the full instance's). With a = 0, gsot_eval's grad[0, m) is minus
 * the shard's plan row sums and its objective b_shard.beta_shard - psi_shard:
 * the terms a sharded driver all-reduces. */
GSOT_API int gsot_create_shard(const double* cost, int64_t m, int64_t n_shard,
                               const int32_t* group_sizes, int32_t L, const double* a,
                               const double* b_shard, double gamma, double mu, gsot_ctx** out);
/* The same with the column block already in device memory (column-major). */
GSOT_API int gsot_create_shard_device(const double* d_cost, int64_t m, int64_t n_shard,
                                      const int32_t* group_sizes, int32_t L, const double* a,
                                      const double* b_shard, double gamma, double mu,
                                      gsot_ctx** out);
GSOT_API void gsot_destroy(gsot_ctx* ctx);
/* Free every parked context's device state now (the cache of gsot_destroy).
 * Returns the number of contexts freed. A create that runs out of device
 * memory drains the cache and retries once by itself. */
GSOT_API int64_t gsot_cache_clear(void);
/* Replace (gamma, mu) keeping the resident cost (RegParams ctor checks). */
GSOT_API int gsot_set_params(gsot_ctx* ctx, double gamma, double mu);
/* Problem shape: m, n, L and the device bytes held by the context. */
GSOT_API int gsot_shape(const gsot_ctx* ctx, int64_t* m, int64_t* n, int32_t* L,
                        int64_t* device_bytes);

/* ---- Stage 1: fused evaluation (ObjectiveFn + GradientFn) ---------------- */

enum {
  GSOT_EVAL_DENSE = 0,
  GSOT_EVAL_SCREENED = 1,
  /* | GSOT_EVAL_EXACT: cross-block sums in the reference's own order
   * (sequential; verification mode) */
  GSOT_EVAL_EXACT = 2
};

/* GradStats::PerCall (screening.hpp:181-186). */
typedef struct gsot_call_stats {
  int64_t in_active;
  int64_t skipped;
  int64_t unskipped;
  int64_t upper_bounds;
} gsot_call_stats;

/* One fused pass at x = [alpha (m); beta (n)]: objective (dual.hpp:38-52)
 * and gradient [grad_alpha; grad_beta] (dual.hpp:85-100, solver.hpp:114-116
 * order). DENSE = solve_baseline's provider (every block computed; stats
 * booked as {0,0,L*n,0}, solver.hpp:117-119). SCREENED = FastGradDispatcher
 * against the current snapshot / active set (Algorithm 2); the screened
 * objective skips exactly the blocks whose psi is provably 0, so it equals
 * the dense objective. Any of objective / grad / stats may be NULL. */
GSOT_API int gsot_eval(gsot_ctx* ctx, const double* x, int mode, double* objective, double* grad,
                       gsot_call_stats* stats);
/* Device-pointer variant (x and grad are device pointers of length m+n). */
GSOT_API int gsot_eval_device(gsot_ctx* ctx, const double* d_x, int mode, double* objective,
                              double* d_grad, gsot_call_stats* stats);

/* The reference's sequential floating-point sum ((s0 + t[0]) + t[1]) + ...
 * (every reduction of the reference accumulates left to right, e.g.
 * regularizer.hpp:47-51), computed in parallel on the device and bit for bit
 * by the exact-order engine. terms: host, n doubles. */
GSOT_API int gsot_sequential_sum(gsot_ctx* ctx, const double* terms, int64_t n, double s0,
                                 double* out);
/* FastGradDispatcher's upper_bound_offset (screening.hpp:206-215, the
 * fault-injection knob audit_solve exposes, solver.hpp:266-270) for later
 * SCREENED gsot_eval calls on this context; 0.0 (the default) is the safe
 * screen. */
GSOT_API int gsot_set_upper_bound_offset(gsot_ctx* ctx, double offset);
/* FastGradDispatcher::init (screening.hpp:220-227): snapshot at x, empty
 * active set. */
GSOT_API int gsot_init_snapshot(gsot_ctx* ctx, const double* x);
/* FastGradDispatcher::refresh (screening.hpp:231-235): when use_active_set,
 * rebuild the active set from lower bounds against the CURRENT snapshot at
 * x, then retake the snapshot at x. */
GSOT_API int gsot_refresh(gsot_ctx* ctx, const double* x, int use_active_set);
/* Download the snapshot norms z~, k~, o~ as L x n column-major (index
 * l + j*L, the reference SnapshotStore layout). Any pointer may be NULL. */
GSOT_API int gsot_snapshot_norms(gsot_ctx* ctx, double* z, double* k, double* o);
/* Download the active set as L x n column-major uint8 (ActiveSet::member)
 * and its count. member may be NULL. */
GSOT_API int gsot_active_set(gsot_ctx* ctx, uint8_t* member, int64_t* count);
/* Nonzero-block map at x: out[l + j*L] = 1 iff z(l,j) > tau
 * (regularizer.hpp:67, i.e. the plan block is nonzero). */
GSOT_API int gsot_block_mask(gsot_ctx* ctx, const double* x, uint8_t* nonzero);
/* recover_plan (dual.hpp:116-128) for columns [j0, j1): out is
 * m x (j1-j0) column-major. Entries are bitwise the reference's grad_block
 * values. */
GSOT_API int gsot_plan_columns(gsot_ctx* ctx, const double* x, int64_t j0, int64_t j1,
                               double* out);
/* PlanDiagnostics (dual.hpp:130-135) of the plan at x. */
typedef struct gsot_plan_diag {
  double marginal_res_a; /* |T 1 - a|_inf */
  double marginal_res_b; /* |T' 1 - b|_inf */
  double group_sparsity; /* fraction of (group, column) blocks that are all 0.0 */
  double mass;           /* sum of all plan entries */
} gsot_plan_diag;
/* plan_diagnostics(recover_plan(x), inst) (dual.hpp:116-128, :139-169)
 * computed on the device without storing the plan: group_sparsity is exact
 * (the same all-zero test on bitwise plan entries); the residuals and mass
 * come from device row / column sums (fixed order, not the reference's
 * summation order: reported, not asserted, as in the reference). */
GSOT_API int gsot_plan_diagnostics(gsot_ctx* ctx, const double* x, gsot_plan_diag* out);
/* primal_objective(recover_plan(x), inst, p) (core.hpp:153-180): <T, C> plus
 * gamma (|T_j|^2 / 2 + mu sum_l |T_{l,j}|) over the columns, on the device
 * without storing the plan (per-block sums, then columns in group order:
 * not the reference's summation order; within ~1e-12 relative). With the
 * dual objective it gives the duality gap. */
GSOT_API int gsot_primal_objective(gsot_ctx* ctx, const double* x, double* out);

/* ---- Stage 2: the whole solve -------------------------------------------- */

enum {
  GSOT_MODE_BASELINE = 0,            /* SolverMode::baseline */
  GSOT_MODE_FAST = 1,                /* SolverMode::fast */
  GSOT_MODE_FAST_NO_LOWER_BOUND = 2, /* SolverMode::fast_no_lower_bound */
  GSOT_MODE_AUDIT = 3                /* SolverMode::audit (audit_solve) */
};

/* SolverOptions (solver.hpp:25-31) + audit_solve's upper_bound_offset. */
typedef struct gsot_solver_options {
  int32_t snapshot_interval; /* 10 */
  double grad_tol;           /* 1e-6 */
  int32_t max_outer_loops;   /* 200 */
  int32_t lbfgs_memory;      /* 10 */
  int32_t mode;              /* GSOT_MODE_FAST */
  double upper_bound_offset; /* 0.0; fault injection (solver.hpp:266-270) */
  int32_t flags;             /* GSOT_SOLVE_EXACT: reference-order sums and dots */
} gsot_solver_options;

enum {
  GSOT_SOLVE_EXACT = 1,
  /* with GSOT_MODE_AUDIT: audit a fast_no_lower_bound solve (no active set),
   * i.e. audit_solve of a SolverOptions whose mode is fast_no_lower_bound
   * (solver.hpp:271) */
  GSOT_SOLVE_NO_ACTIVE_SET = 2
};

/* Solution (solver.hpp:33-42) minus the dense state/plan (returned through
 * x_out and gsot_plan_columns), GradStats totals (screening.hpp:173-180)
 * and AuditReport (solver.hpp:46-51). */
typedef struct gsot_solve_result {
  double objective;
  int32_t iterations;
  int32_t chunks;
  int32_t converged;
  int32_t line_search_failed;
  int64_t blocks_in_active_set;
  int64_t blocks_skipped;
  int64_t blocks_unskipped;
  int64_t upper_bounds_evaluated;
  int64_t outer_loops;
  int64_t grad_calls;
  double wall_seconds; /* the maximize span, as Solution::wall_time (solver.hpp:243-246) */
  int64_t audit_skip_checks;
  int64_t audit_active_checks;
  int64_t audit_column_compares;
  int64_t audit_gradient_calls;
  /* work of the screened evaluations: blocks computed (|W| = active set +
   * unskipped) and (group, 32-column) tasks launched, summed over calls */
  int64_t eval_blocks;
  int64_t eval_tasks;
} gsot_solve_result;

GSOT_API void gsot_default_solver_options(gsot_solver_options* o);
/* solve (solver.hpp:284-293) from x0 = 0 on the resident instance. x_out
 * (m+n, may be NULL) receives [alpha; beta]. history (may be NULL) receives
 * up to history_cap rows of 4 int64 (GradStats::history). The objective is
 * finish_solution's dense re-evaluation at the final state. */
GSOT_API int gsot_solve(gsot_ctx* ctx, const gsot_solver_options* opts, double* x_out,
                        gsot_solve_result* result, int64_t* history, int64_t history_cap);

/* ---- Multi-GPU: the column-sharded solve on the device ----
 *
 * The reference solves on one host (solver.hpp:284-293); its only parallel
 * decomposition is by column. Rank p of P builds a shard
 * context (gsot_create_shard[_device]) over its column block J_p with
 * a = the row marginal on rank 0 and zeros on every other rank, attaches a
 * communicator, and calls gsot_solve: the same device-resident solve (CUDA
 * graphs, compact L-BFGS) with, per device sequence, ONE sum all-reduce of
 * the gradient head (m doubles: a - sum_p rowsum_p) and a 16-double tail
 * (a.alpha, b.beta, psi, g.d, the step's g.d and d.d, the GradStats
 * counters), plus one of (memory+1)*5 doubles inside every direction update
 * (the L-BFGS dots; the replicated alpha part counted once). Every rank then
 * takes the same host decisions. x_out receives the rank's [alpha; beta_p].
 * Modes: GSOT_MODE_BASELINE / FAST / FAST_NO_LOWER_BOUND; exact-order and
 * audit solves are single-context only (GSOT_ERR_INVALID_ARGUMENT). */
enum { GSOT_REDUCE_SUM = 0, GSOT_REDUCE_MAX = 1 };
/* Host transport: called synchronously with `count` doubles in host memory,
 * reduces them in place over the ranks (identical result on every rank);
 * returns 0 on success. */
typedef int (*gsot_allreduce_fn)(double* buf, int64_t count, int32_t op, void* user);
/* A fresh NCCL unique id (128 bytes) for gsot_comm_attach_nccl (rank 0 makes
 * it, the caller broadcasts it). NCCL is loaded at run time (libnccl.so.2,
 * the process's own copy when one is loaded). */
GSOT_API int gsot_comm_unique_id(unsigned char id[128]);
/* Attach an NCCL communicator over the world's GPUs (one rank per GPU,
 * collective over the ranks): the all-reduces run on the context's stream
 * inside the solver's CUDA graphs. */
GSOT_API int gsot_comm_attach_nccl(gsot_ctx* ctx, const unsigned char id[128], int32_t world,
                                   int32_t rank);
/* Attach a host transport (testing and hosts without NCCL): the solver runs
 * its sequences eagerly and synchronises around every all-reduce. */
GSOT_API int gsot_comm_attach_host(gsot_ctx* ctx, int32_t world, int32_t rank,
                                   gsot_allreduce_fn fn, void* user);
/* Detach (and destroy) the communicator: the context solves alone again. */
GSOT_API int gsot_comm_detach(gsot_ctx* ctx);

/* ---- Inputs: synthetic instances (SURVEY.md §8(d) recipe) ----------------- */

/* Per-config sizes: cfg in 1..5. Returns m, n, L, d. */
GSOT_API int gsot_config_shape(int32_t cfg, int64_t* m, int64_t* n, int32_t* L, int64_t* d);
/* Host features + marginals for config cfg with seed: src (m x d row-major,
 * rows sorted by class), tgt (n x d row-major, shuffled), group sizes (L),
 * a (m), b (n). Pinned RNG = reference Rng (data_io.hpp:32-62). */
GSOT_API int gsot_config_features(int32_t cfg, uint64_t seed, double* src, double* tgt,
                                  int32_t* sizes, double* a, double* b);
/* cost_matrix (data_io.hpp:101-123) on device: k-sequential fp64 without
 * FMA, then optional C /= max(C) (data_io.hpp:162-165). src/tgt host,
 * row-major; d_cost device m x n column-major (caller-allocated). */
GSOT_API int gsot_cost_matrix_device(const double* src, int64_t m, const double* tgt, int64_t n,
                                     int64_t d, int normalize, double* d_cost);
/* make_instance (data_io.hpp:157-181) on the device: the cost of source
 * features src (m x d row-major, rows grouped by class: group_sizes, the
 * partition_from_labels of the sorted labels, data_io.hpp:127-152) and target
 * features tgt (n x d row-major) is computed straight into HBM
 * (cost_matrix, data_io.hpp:101-123, bitwise), divided by its maximum when
 * normalize (and the maximum is > 0), and validated like gsot_create
 * (validate_instance, core.hpp:117-139). a, b: the marginals make_instance
 * chose (uniform, or the normalised sample weights). The cost never visits
 * the host. */
GSOT_API int gsot_create_features(const double* src, int64_t m, const double* tgt, int64_t n,
                                  int64_t d, const int32_t* group_sizes, int32_t L,
                                  const double* a, const double* b, int normalize, double gamma,
                                  double mu, gsot_ctx** out);
/* Build a context for config cfg directly on device (the cost never visits
 * the host). */
GSOT_API int gsot_create_config(int32_t cfg, uint64_t seed, double gamma, double mu,
                                gsot_ctx** out);

/* ---- Measurement ---------------------------------------------------------- */

/* Per-kernel-class device time (CUDA events on the context stream, event
 * nodes inside the solver's graphs) and algorithmic bytes since the last
 * reset. kind: 0 eval(fused blocks), 1 snapshot, 2 bounds, 3 active set,
 * 4 finalize, 5 lbfgs vector ops, 6 delta norms, 7 misc; read-only kind 8:
 * the eval launches that read at least half the dense bytes (near-dense);
 * read-only kind 9: the eval launches with bytes = the cost bytes they
 * fetched (whole 8-column quarters of each task read), to set beside kind 0.
 * enable: 0 off, negative every class, positive a bit mask (1 << kind) of
 * the classes 0-7. */
GSOT_API int gsot_profile_enable(gsot_ctx* ctx, int enable);
GSOT_API int gsot_profile_read(gsot_ctx* ctx, int kind, double* ms, double* bytes,
                               int64_t* launches);
GSOT_API int gsot_profile_reset(gsot_ctx* ctx);
/* Select the CUDA device used by contexts created afterwards on this host
 * thread (one process per GPU: LOCAL_RANK). */
GSOT_API int gsot_set_device(int32_t device);
/* CUDA-event timer on the context stream: op 0 records the start event,
 * op 1 records the stop event, synchronizes and returns the elapsed ms. */
GSOT_API int gsot_timer(gsot_ctx* ctx, int op, double* ms);
/* Number of kernels this library launched on the context (all kinds). */
GSOT_API int64_t gsot_kernel_launches(const gsot_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* GSOT_H */
