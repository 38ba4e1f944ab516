/*
 * gsot_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * Plain-C restatement of the reference `groupot` hot path
 * (/root/reference/proj/include/groupot/{regularizer,dual,screening,lbfgs,
 * solver,core,data_io}.hpp), kept line-for-line in order of floating-point
 * operations so that it is bitwise equal to the reference compiled against the
 * sequential Eigen shim (oracle/_ref). Pinned by tests/test_oracle_pin.py
 * against oracle/_ref and against tests/golden/ fixtures generated from the
 * real reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the timed CPU
 * baseline. The product path (paper_2303_07597_b200/) never calls it.
 *
 * Layout conventions follow the reference: cost is column-major m x n
 * (block (l,j) = g_l contiguous doubles at offset off_l + j*m); snapshot
 * matrices and the active set are |L| x n column-major (index l + j*L).
 */
#ifndef GSOT_ORACLE_H
#define GSOT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* regularizer.hpp:23-91 */
double go_pos_part_norm(const double* f, int n);
double go_neg_part_norm(const double* f, int n);
double go_vec_norm(const double* f, int n);
double go_sum_entries(const double* v, int n);
void go_residual_block(const double* alpha, double beta_j, const double* cost, int n, double* out);
double go_grad_block(const double* f, int n, double gamma, double tau, double* out);
double go_psi_block(const double* f, int n, double gamma, double mu, double tau);

typedef struct {
  const double* cost; /* m x n column-major */
  int64_t m, n;
  int32_t L;
  const int32_t* sizes;   /* L */
  const int32_t* offsets; /* L+1, caller-provided prefix sums */
  const double* a;        /* m */
  const double* b;        /* n */
  double gamma, mu;
} go_problem;

/* core.hpp:117-139. Returns 0 ok, else a gsot_status-compatible code and
 * fills *row,*col (NegativeCost) or *which,*index (MarginalNotNormalized). */
int go_validate(const go_problem* p, int64_t* row, int64_t* col, char* which, int64_t* index);
double go_compensated_sum(const double* v, int64_t n); /* core.hpp:85-98 */

/* dual.hpp:38-52 and :85-100 with baseline_column_grad (:59-77) */
double go_dual_objective(const go_problem* p, const double* alpha, const double* beta);
void go_dual_gradient(const go_problem* p, const double* alpha, const double* beta, double* ga,
                      double* gb);
void go_recover_plan(const go_problem* p, const double* alpha, const double* beta, double* plan);
/* recover_plan restricted to columns [j0, j1) into out (m x (j1-j0)). */
void go_plan_columns(const go_problem* p, const double* alpha, const double* beta, int64_t j0,
                     int64_t j1, double* out);

/* dual.hpp:139-169 plan_diagnostics of an m x n column-major plan:
 * out = {marginal_res_a, marginal_res_b, group_sparsity, mass}. */
void go_plan_diagnostics(const go_problem* p, const double* plan, double* out);

/* screening.hpp:24-50 take_snapshot: z,k,o are L x n column-major. */
void go_take_snapshot(const go_problem* p, const double* alpha, const double* beta, double* z,
                      double* k, double* o);
/* screening.hpp:63-83: per-group pos/full/neg norms of alpha - alpha_snap,
 * sqrt(g), and dbeta = beta - beta_snap. */
void go_delta_norms(const go_problem* p, const double* alpha, const double* beta,
                    const double* alpha_snap, const double* beta_snap, double* dpos,
                    double* dfull, double* dneg, double* sqrt_g, double* dbeta);
/* screening.hpp:147-166; member is L x n column-major uint8. Returns count. */
int64_t go_build_active_set(const go_problem* p, const double* alpha_snap,
                            const double* beta_snap, const double* k_snap, const double* o_snap,
                            const double* alpha, const double* beta, uint8_t* member);
/* FastGradDispatcher gradient call (screening.hpp:239-287 + dual.hpp:85-100).
 * counters[4] = in_active, skipped, unskipped, upper_bounds. member may be
 * NULL (fast-no-lb). path (optional, L x n col-major) receives 0 active,
 * 1 skipped, 2 computed-after-bound. */
void go_fast_gradient(const go_problem* p, const double* alpha_snap, const double* beta_snap,
                      const double* z_snap, const uint8_t* member, double ub_offset,
                      const double* alpha, const double* beta, double* ga, double* gb,
                      int64_t counters[4], uint8_t* path);

/* lbfgs.hpp:11-30 */
typedef struct {
  int chunk_iters, max_chunks, memory;
  double grad_tol, wolfe_c1, wolfe_c2;
  int max_bracket, max_zoom;
} go_maximize_options;
void go_default_maximize_options(go_maximize_options* o);

/* solver.hpp:13-42. mode: 0 baseline, 1 fast, 2 fast-no-lb, 3 audit. */
typedef struct {
  int snapshot_interval;
  double grad_tol;
  int max_outer_loops;
  int lbfgs_memory;
  int mode;
} go_solver_options;

typedef struct {
  double objective;
  int iterations;
  int chunks;
  int converged;
  int line_search_failed;
  int64_t blocks_in_active_set, blocks_skipped, blocks_unskipped, upper_bounds_evaluated;
  int64_t outer_loops, grad_calls;
  double wall_seconds; /* maximize span, solver.hpp:243-246 */
  /* audit report (solver.hpp:46-51) */
  int64_t audit_skip_checks, audit_active_checks, audit_column_compares, audit_gradient_calls;
} go_solve_result;

/* solve (solver.hpp:284-293). x_out: m+n final state. history (optional):
 * grad_calls x 4 int64 (in_active, skipped, unskipped, upper_bounds),
 * capacity history_cap rows. plan (optional): m x n. Returns 0 or an error
 * code (validation, or 7 = AuditViolation). trace_x (optional): accepted
 * iterates are appended as rows of length m+n up to trace_cap rows
 * (row 0 = x0). */
int go_solve(const go_problem* p, const go_solver_options* o, double ub_offset, double* x_out,
             go_solve_result* res, int64_t* history, int64_t history_cap, double* plan,
             double* trace_x, int64_t trace_cap, int64_t* trace_rows);

/* Generic maximize over callbacks (for the L-BFGS unit tests). */
typedef double (*go_objective_fn)(void* ctx, const double* x);
typedef void (*go_gradient_fn)(void* ctx, const double* x, double* g);
typedef void (*go_hook_fn)(void* ctx, int chunk, const double* x);
typedef struct {
  double objective;
  int iterations, chunks, converged, line_search_failed;
} go_maximize_result;
void go_maximize(go_objective_fn f, go_gradient_fn g, go_hook_fn hook, void* ctx, const double* x0,
                 int64_t dim, const go_maximize_options* o, double* x_out, double* grad_out,
                 go_maximize_result* r);

/* data_io.hpp:32-62 Rng, and the instance recipe of SURVEY.md §8(d). */
typedef struct {
  uint64_t mt[312];
  int mti;
  int has_spare;
  double spare;
} go_rng;
void go_rng_seed(go_rng* r, uint64_t seed);
uint64_t go_rng_next(go_rng* r);
double go_rng_uniform01(go_rng* r);
double go_rng_normal(go_rng* r);
uint64_t go_rng_index(go_rng* r, uint64_t bound);

/* data_io.hpp:101-123 cost_matrix (k-sequential, no FMA), column-major. */
void go_cost_matrix(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                    double* cost);
/* same, with j-range [j0,j1) only and nthreads host threads (bench setup). */
void go_cost_matrix_par(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                        double* cost, int nthreads);

/* Synthetic instance recipe of the five BASELINE.json configs (SURVEY.md
 * §8(d), pinned in DESIGN.md §6): shape query and host features, the same
 * draw order as the product's generator (paper_2303_07597_b200/csrc/
 * gsot_data.cu). src m x d and tgt n x d row-major. */
int go_config_shape(int cfg, int64_t* m, int64_t* n, int32_t* L, int64_t* d);
int go_config_features(int cfg, uint64_t seed, double* src, double* tgt, int32_t* sizes,
                       double* a, double* b);

#ifdef __cplusplus
}
#endif
#endif
