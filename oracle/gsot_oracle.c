/*
 * gsot_oracle.c — CPU ORACLE (test infrastructure only; see gsot_oracle.h).
 *
 * Restates the reference algorithm in plain C, preserving the order of every
 * floating-point operation (compile with -ffp-contract=off, as the reference's
 * proj/CMakeLists.txt:15-17 does). Each function cites the reference
 * file:line it follows; paths are relative to
 * /root/reference/proj/include/groupot/.
 */
#define _POSIX_C_SOURCE 200809L
#include "gsot_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- block math
 * regularizer.hpp:23-91. Sequential loops, one rounding per operation. */

double go_pos_part_norm(const double* f, int n) { /* regularizer.hpp:23-30 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = f[i] > 0.0 ? f[i] : 0.0;
    acc += v * v;
  }
  return sqrt(acc);
}

double go_neg_part_norm(const double* f, int n) { /* regularizer.hpp:32-39 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = f[i] < 0.0 ? f[i] : 0.0;
    acc += v * v;
  }
  return sqrt(acc);
}

double go_vec_norm(const double* f, int n) { /* regularizer.hpp:41-45 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += f[i] * f[i];
  return sqrt(acc);
}

double go_sum_entries(const double* v, int n) { /* regularizer.hpp:47-51 */
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += v[i];
  return acc;
}

void go_residual_block(const double* alpha, double beta_j, const double* cost, int n,
                       double* out) { /* regularizer.hpp:55-58 */
  for (int i = 0; i < n; ++i) out[i] = alpha[i] + beta_j - cost[i];
}

double go_grad_block(const double* f, int n, double gamma, double tau,
                     double* out) { /* regularizer.hpp:64-74 */
  const double z = go_pos_part_norm(f, n);
  if (z <= tau) {
    for (int i = 0; i < n; ++i) out[i] = 0.0;
    return z;
  }
  const double scale = (1.0 - tau / z) / gamma;
  for (int i = 0; i < n; ++i) out[i] = f[i] > 0.0 ? scale * f[i] : 0.0;
  return z;
}

double go_psi_block(const double* f, int n, double gamma, double mu,
                    double tau) { /* regularizer.hpp:78-91 */
  const double z = go_pos_part_norm(f, n);
  if (z <= tau) return 0.0;
  const double scale = (1.0 - tau / z) / gamma;
  double dot = 0.0;
  double sq = 0.0;
  for (int i = 0; i < n; ++i) {
    const double g = f[i] > 0.0 ? scale * f[i] : 0.0;
    dot += f[i] * g;
    sq += g * g;
  }
  return dot - gamma * (0.5 * sq + mu * sqrt(sq));
}

static double tau_of(const go_problem* p) { return p->mu * p->gamma; } /* core.hpp:70 */

static double seq_dot(const double* a, const double* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

/* ---------------------------------------------------------------- validation */

double go_compensated_sum(const double* v, int64_t n) { /* core.hpp:85-98 */
  double sum = 0.0, comp = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = v[i];
    const double t = sum + x;
    if (fabs(sum) >= fabs(x))
      comp += (sum - t) + x;
    else
      comp += (x - t) + sum;
    sum = t;
  }
  return sum + comp;
}

/* status codes match include/gsot.h */
enum { ST_OK = 0, ST_DIM = 1, ST_NEGCOST = 2, ST_MARGINAL = 3, ST_PARTITION = 4, ST_PARAM = 5,
       ST_AUDIT = 7 };

static int check_marginal(const double* v, int64_t n, char which, char* w, int64_t* index) {
  /* core.hpp:100-112 */
  for (int64_t i = 0; i < n; ++i) {
    if (!(v[i] >= 0.0) || !isfinite(v[i])) {
      if (w) *w = which;
      if (index) *index = i;
      return ST_MARGINAL;
    }
  }
  const double sum = go_compensated_sum(v, n);
  if (fabs(sum - 1.0) > 1e-12) {
    if (w) *w = which;
    if (index) *index = -1;
    return ST_MARGINAL;
  }
  return ST_OK;
}

int go_validate(const go_problem* p, int64_t* row, int64_t* col, char* which,
                int64_t* index) { /* core.hpp:117-139 (+ GroupPartition ctor :19-30, RegParams :61-66) */
  if (p->L < 1) return ST_PARTITION;
  for (int l = 0; l < p->L; ++l)
    if (p->sizes[l] < 1) return ST_PARTITION;
  if (!(p->gamma > 0.0) || !isfinite(p->gamma)) return ST_PARAM;
  if (!(p->mu > 0.0) || !isfinite(p->mu)) return ST_PARAM;
  for (int64_t j = 0; j < p->n; ++j) {
    for (int64_t i = 0; i < p->m; ++i) {
      const double c = p->cost[i + j * p->m];
      if (!(c >= 0.0) || !isfinite(c)) {
        if (row) *row = i;
        if (col) *col = j;
        return ST_NEGCOST;
      }
    }
  }
  int st = check_marginal(p->a, p->m, 'a', which, index);
  if (st) return st;
  st = check_marginal(p->b, p->n, 'b', which, index);
  if (st) return st;
  if (p->offsets[p->L] != p->m) return ST_PARTITION;
  return ST_OK;
}

/* ---------------------------------------------------------------- dual */

double go_dual_objective(const go_problem* p, const double* alpha,
                         const double* beta) { /* dual.hpp:38-52 */
  const double tau = tau_of(p);
  double psi_sum = 0.0;
  double* f = (double*)malloc(sizeof(double) * (size_t)p->m);
  for (int64_t j = 0; j < p->n; ++j) {
    go_residual_block(alpha, beta[j], p->cost + j * p->m, (int)p->m, f);
    for (int l = 0; l < p->L; ++l)
      psi_sum += go_psi_block(f + p->offsets[l], p->sizes[l], p->gamma, p->mu, tau);
  }
  free(f);
  return seq_dot(alpha, p->a, p->m) + seq_dot(beta, p->b, p->n) - psi_sum;
}

static void baseline_column(const go_problem* p, const double* alpha, const double* beta,
                            int64_t j, double* gcol, double* fblock) { /* dual.hpp:59-77 */
  const double* cj = p->cost + j * p->m;
  const double bj = beta[j];
  const double tau = tau_of(p);
  for (int l = 0; l < p->L; ++l) {
    const int off = p->offsets[l];
    const int g = p->sizes[l];
    go_residual_block(alpha + off, bj, cj + off, g, fblock);
    go_grad_block(fblock, g, p->gamma, tau, gcol + off);
  }
}

static void assemble_column(const go_problem* p, int64_t j, const double* gcol, double* ga,
                            double* gb) { /* dual.hpp:94-98 */
  for (int64_t i = 0; i < p->m; ++i) ga[i] -= gcol[i];
  gb[j] = p->b[j] - go_sum_entries(gcol, (int)p->m);
}

void go_dual_gradient(const go_problem* p, const double* alpha, const double* beta, double* ga,
                      double* gb) { /* dual.hpp:85-100 with the baseline provider */
  double* gcol = (double*)malloc(sizeof(double) * (size_t)p->m);
  double* fb = (double*)malloc(sizeof(double) * (size_t)p->m);
  memcpy(ga, p->a, sizeof(double) * (size_t)p->m);
  for (int64_t j = 0; j < p->n; ++j) {
    baseline_column(p, alpha, beta, j, gcol, fb);
    assemble_column(p, j, gcol, ga, gb);
  }
  free(gcol);
  free(fb);
}

void go_plan_columns(const go_problem* p, const double* alpha, const double* beta, int64_t j0,
                     int64_t j1, double* out) { /* dual.hpp:116-128 restricted to [j0,j1) */
  double* fb = (double*)malloc(sizeof(double) * (size_t)p->m);
  for (int64_t j = j0; j < j1; ++j) baseline_column(p, alpha, beta, j, out + (j - j0) * p->m, fb);
  free(fb);
}

void go_recover_plan(const go_problem* p, const double* alpha, const double* beta, double* plan) {
  go_plan_columns(p, alpha, beta, 0, p->n, plan);
}

void go_plan_diagnostics(const go_problem* p, const double* plan,
                         double* out) { /* dual.hpp:139-169 */
  const int64_t m = p->m, n = p->n;
  /* rowwise().sum(): row i summed over j in order (sequential Eigen reduction) */
  double ra = 0.0, rb = 0.0, mass = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s += plan[i + j * m];
    const double d = fabs(s - p->a[i]);
    ra = (i == 0 || d > ra) ? d : ra; /* cwiseAbs().maxCoeff() */
  }
  for (int64_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += plan[i + j * m];
    const double d = fabs(s - p->b[j]);
    rb = (j == 0 || d > rb) ? d : rb;
  }
  for (int64_t e = 0; e < m * n; ++e) mass += plan[e]; /* t.plan.sum(), storage order */
  long zero_blocks = 0;
  for (int64_t j = 0; j < n; ++j)
    for (int l = 0; l < p->L; ++l) {
      int all_zero = 1;
      for (int64_t i = p->offsets[l]; i < p->offsets[l] + p->sizes[l]; ++i)
        if (plan[i + j * m] != 0.0) {
          all_zero = 0;
          break;
        }
      zero_blocks += all_zero;
    }
  out[0] = ra;
  out[1] = rb;
  out[2] = (double)zero_blocks / ((double)p->L * (double)n);
  out[3] = mass;
}

/* ---------------------------------------------------------------- screening */

void go_take_snapshot(const go_problem* p, const double* alpha, const double* beta, double* z,
                      double* k, double* o) { /* screening.hpp:24-50 */
  double* f = (double*)malloc(sizeof(double) * (size_t)p->m);
  for (int64_t j = 0; j < p->n; ++j) {
    go_residual_block(alpha, beta[j], p->cost + j * p->m, (int)p->m, f);
    for (int l = 0; l < p->L; ++l) {
      const double* fl = f + p->offsets[l];
      const int g = p->sizes[l];
      z[l + j * p->L] = go_pos_part_norm(fl, g);
      k[l + j * p->L] = go_vec_norm(fl, g);
      o[l + j * p->L] = go_neg_part_norm(fl, g);
    }
  }
  free(f);
}

void go_delta_norms(const go_problem* p, const double* alpha, const double* beta,
                    const double* alpha_snap, const double* beta_snap, double* dpos,
                    double* dfull, double* dneg, double* sqrt_g,
                    double* dbeta) { /* screening.hpp:63-83 */
  double* da = (double*)malloc(sizeof(double) * (size_t)p->m);
  for (int64_t i = 0; i < p->m; ++i) da[i] = alpha[i] - alpha_snap[i];
  for (int l = 0; l < p->L; ++l) {
    const double* dl = da + p->offsets[l];
    const int g = p->sizes[l];
    dpos[l] = go_pos_part_norm(dl, g);
    dfull[l] = go_vec_norm(dl, g);
    dneg[l] = go_neg_part_norm(dl, g);
    sqrt_g[l] = sqrt((double)g);
  }
  for (int64_t j = 0; j < p->n; ++j) dbeta[j] = beta[j] - beta_snap[j];
  free(da);
}

static double upper_bound(double zs, double dpos, double sqrt_g,
                          double db) { /* screening.hpp:88-93 */
  const double db_pos = db > 0.0 ? db : 0.0;
  return zs + dpos + sqrt_g * db_pos;
}

static double lower_bound(double ks, double os, double dfull, double dneg, double sqrt_g,
                          double db) { /* screening.hpp:99-105 */
  const double db_neg = db < 0.0 ? -db : 0.0;
  return ks - dfull - sqrt_g * fabs(db) - os - dneg - sqrt_g * db_neg;
}

typedef struct {
  double *dpos, *dfull, *dneg, *sqrt_g, *dbeta;
} deltas_t;

static void deltas_alloc(deltas_t* d, const go_problem* p) {
  d->dpos = (double*)malloc(sizeof(double) * (size_t)p->L);
  d->dfull = (double*)malloc(sizeof(double) * (size_t)p->L);
  d->dneg = (double*)malloc(sizeof(double) * (size_t)p->L);
  d->sqrt_g = (double*)malloc(sizeof(double) * (size_t)p->L);
  d->dbeta = (double*)malloc(sizeof(double) * (size_t)p->n);
}
static void deltas_free(deltas_t* d) {
  free(d->dpos);
  free(d->dfull);
  free(d->dneg);
  free(d->sqrt_g);
  free(d->dbeta);
}

int64_t go_build_active_set(const go_problem* p, const double* alpha_snap,
                            const double* beta_snap, const double* k_snap, const double* o_snap,
                            const double* alpha, const double* beta,
                            uint8_t* member) { /* screening.hpp:147-166 */
  deltas_t d;
  deltas_alloc(&d, p);
  go_delta_norms(p, alpha, beta, alpha_snap, beta_snap, d.dpos, d.dfull, d.dneg, d.sqrt_g,
                 d.dbeta);
  const double tau = tau_of(p);
  int64_t count = 0;
  for (int64_t j = 0; j < p->n; ++j) {
    for (int l = 0; l < p->L; ++l) {
      const int64_t idx = l + j * p->L;
      const double lb = lower_bound(k_snap[idx], o_snap[idx], d.dfull[l], d.dneg[l], d.sqrt_g[l],
                                    d.dbeta[j]);
      member[idx] = lb > tau ? 1 : 0;
      if (lb > tau) ++count;
    }
  }
  deltas_free(&d);
  return count;
}

/* FastGradDispatcher::begin_call/column/end_call (screening.hpp:239-287) feeding
 * dual_gradient (dual.hpp:85-100). */
typedef struct {
  const go_problem* p;
  const double *alpha_snap, *beta_snap, *z_snap;
  const uint8_t* member;
  double ub_offset;
  deltas_t d;
  double* fblock;
  int64_t call[4];
} dispatcher_t;

static void dispatch_column(dispatcher_t* ds, const double* alpha, const double* beta, int64_t j,
                            double* gcol, uint8_t* path) { /* screening.hpp:246-276 */
  const go_problem* p = ds->p;
  const double* cj = p->cost + j * p->m;
  const double bj = beta[j];
  const double tau = tau_of(p);
  for (int l = 0; l < p->L; ++l) {
    const int off = p->offsets[l];
    const int g = p->sizes[l];
    double* out = gcol + off;
    const int64_t idx = l + j * p->L;
    if (ds->member && ds->member[idx]) {
      go_residual_block(alpha + off, bj, cj + off, g, ds->fblock);
      go_grad_block(ds->fblock, g, p->gamma, tau, out);
      ++ds->call[0];
      if (path) path[idx] = 0;
      continue;
    }
    const double zbar = upper_bound(ds->z_snap[idx], ds->d.dpos[l], ds->d.sqrt_g[l],
                                    ds->d.dbeta[j]) +
                        ds->ub_offset;
    ++ds->call[3];
    if (zbar <= tau) {
      for (int i = 0; i < g; ++i) out[i] = 0.0;
      ++ds->call[1];
      if (path) path[idx] = 1;
    } else {
      go_residual_block(alpha + off, bj, cj + off, g, ds->fblock);
      go_grad_block(ds->fblock, g, p->gamma, tau, out);
      ++ds->call[2];
      if (path) path[idx] = 2;
    }
  }
}

void go_fast_gradient(const go_problem* p, const double* alpha_snap, const double* beta_snap,
                      const double* z_snap, const uint8_t* member, double ub_offset,
                      const double* alpha, const double* beta, double* ga, double* gb,
                      int64_t counters[4], uint8_t* path) {
  dispatcher_t ds;
  memset(&ds, 0, sizeof ds);
  ds.p = p;
  ds.alpha_snap = alpha_snap;
  ds.beta_snap = beta_snap;
  ds.z_snap = z_snap;
  ds.member = member;
  ds.ub_offset = ub_offset;
  deltas_alloc(&ds.d, p);
  go_delta_norms(p, alpha, beta, alpha_snap, beta_snap, ds.d.dpos, ds.d.dfull, ds.d.dneg,
                 ds.d.sqrt_g, ds.d.dbeta);
  ds.fblock = (double*)malloc(sizeof(double) * (size_t)p->m);
  double* gcol = (double*)malloc(sizeof(double) * (size_t)p->m);
  memcpy(ga, p->a, sizeof(double) * (size_t)p->m);
  for (int64_t j = 0; j < p->n; ++j) {
    dispatch_column(&ds, alpha, beta, j, gcol, path);
    assemble_column(p, j, gcol, ga, gb);
  }
  for (int c = 0; c < 4; ++c) counters[c] = ds.call[c];
  free(gcol);
  free(ds.fblock);
  deltas_free(&ds.d);
}

/* ---------------------------------------------------------------- L-BFGS
 * lbfgs.hpp:61-274, ascent form. Vector arithmetic is elementwise with one
 * rounding per operation (Eigen under -ffp-contract=off); reductions are
 * sequential (the oracle/_ref Eigen shim). */

void go_default_maximize_options(go_maximize_options* o) { /* lbfgs.hpp:11-20 */
  o->chunk_iters = 10;
  o->max_chunks = 200;
  o->memory = 10;
  o->grad_tol = 1e-6;
  o->wolfe_c1 = 1e-4;
  o->wolfe_c2 = 0.9;
  o->max_bracket = 40;
  o->max_zoom = 12;
}

typedef struct { /* lbfgs.hpp:40-46 */
  double t, value, slope;
  double *x, *grad; /* valid iff has_vec */
  int has_vec;
} lspoint_t;

static void ls_copy(lspoint_t* dst, const lspoint_t* src, int64_t dim) {
  dst->t = src->t;
  dst->value = src->value;
  dst->slope = src->slope;
  dst->has_vec = src->has_vec;
  if (src->has_vec) {
    memcpy(dst->x, src->x, sizeof(double) * (size_t)dim);
    memcpy(dst->grad, src->grad, sizeof(double) * (size_t)dim);
  }
}

static double norm_inf(const double* v, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) m = fmax(m, fabs(v[i]));
  return m;
}

typedef void (*accept_fn)(void* ctx, int iteration, const double* x);

static void maximize_impl(go_objective_fn objective, go_gradient_fn gradient, go_hook_fn hook,
                          accept_fn on_accept, void* ctx, const double* x0, int64_t dim,
                          const go_maximize_options* opts, double* x_out, double* grad_out,
                          go_maximize_result* res) {
  const size_t vb = sizeof(double) * (size_t)dim;
  double* x = x_out;
  double* gx = grad_out;
  memcpy(x, x0, vb);
  gradient(ctx, x, gx); /* lbfgs.hpp:70-71 */
  double fx = objective(ctx, x);
  res->iterations = 0;
  res->chunks = 0;
  res->converged = 0;
  res->line_search_failed = 0;

  const int mem = opts->memory;
  double** s_hist = (double**)calloc((size_t)mem + 1, sizeof(double*));
  double** y_hist = (double**)calloc((size_t)mem + 1, sizeof(double*));
  double* rho_hist = (double*)calloc((size_t)mem + 1, sizeof(double));
  double* two_loop_a = (double*)calloc((size_t)mem + 1, sizeof(double));
  int k_hist = 0;
  double* d = (double*)malloc(vb);
  double* q = (double*)malloc(vb);
  lspoint_t trial, lo, prev;
  trial.x = (double*)malloc(vb);
  trial.grad = (double*)malloc(vb);
  lo.x = (double*)malloc(vb);
  lo.grad = (double*)malloc(vb);
  prev.x = (double*)malloc(vb);
  prev.grad = (double*)malloc(vb);
  trial.has_vec = lo.has_vec = prev.has_vec = 0;
  int stalled = 0, zero_gradient = 0;

#define EVAL_AT(tt)                                               \
  do {                                                            \
    trial.t = (tt);                                               \
    for (int64_t e = 0; e < dim; ++e) trial.x[e] = x[e] + trial.t * d[e]; \
    trial.value = objective(ctx, trial.x);                        \
    gradient(ctx, trial.x, trial.grad);                           \
    trial.slope = seq_dot(trial.grad, d, dim);                    \
    trial.has_vec = 1;                                            \
  } while (0)

  for (int chunk = 0; chunk < opts->max_chunks && !stalled && !zero_gradient; ++chunk) {
    ++res->chunks;
    for (int it = 0; it < opts->chunk_iters; ++it) {
      int accepted = 0;
      for (int attempt = 0; attempt < 2 && !accepted; ++attempt) { /* lbfgs.hpp:99 */
        if (attempt == 1) {
          if (k_hist == 0) break;
          for (int i = 0; i < k_hist; ++i) {
            free(s_hist[i]);
            free(y_hist[i]);
          }
          k_hist = 0;
        }
        memcpy(q, gx, vb); /* two-loop, lbfgs.hpp:109-124 */
        const int k = k_hist;
        for (int i = 0; i < k; ++i) two_loop_a[i] = 0.0;
        for (int i = k; i-- > 0;) {
          two_loop_a[i] = rho_hist[i] * seq_dot(s_hist[i], q, dim);
          for (int64_t e = 0; e < dim; ++e) q[e] -= two_loop_a[i] * y_hist[i][e];
        }
        if (k > 0) {
          const double yy = seq_dot(y_hist[k - 1], y_hist[k - 1], dim);
          if (yy > 0.0) {
            const double sc = seq_dot(s_hist[k - 1], y_hist[k - 1], dim) / yy;
            for (int64_t e = 0; e < dim; ++e) q[e] *= sc;
          }
        }
        for (int i = 0; i < k; ++i) {
          const double b = rho_hist[i] * seq_dot(y_hist[i], q, dim);
          for (int64_t e = 0; e < dim; ++e) q[e] += (two_loop_a[i] - b) * s_hist[i][e];
        }
        memcpy(d, q, vb);

        double dir_slope = seq_dot(gx, d, dim); /* lbfgs.hpp:126-137 */
        if (!(dir_slope > 0.0)) {
          for (int i = 0; i < k_hist; ++i) {
            free(s_hist[i]);
            free(y_hist[i]);
          }
          k_hist = 0;
          memcpy(d, gx, vb);
          dir_slope = seq_dot(gx, gx, dim);
          if (dir_slope == 0.0) {
            zero_gradient = 1;
            break;
          }
        }

        const double f0 = fx; /* lbfgs.hpp:141-148 */
        const double armijo = opts->wolfe_c1 * dir_slope;
#define SUFFICIENT(P) ((P).value >= f0 + armijo * (P).t)
#define CURVATURE_OK(P) (fabs((P).slope) <= opts->wolfe_c2 * dir_slope)

        double t_init = 1.0; /* lbfgs.hpp:150-154 */
        if (res->iterations == 0) {
          const double dnorm = sqrt(seq_dot(d, d, dim));
          if (dnorm > 0.0) t_init = 1.0 / dnorm;
        }

        int have_bracket = 0;
        lo.t = 0.0;
        lo.value = f0;
        lo.slope = dir_slope;
        lo.has_vec = 0;
        double hi_t = 0.0;

        double t = t_init; /* bracketing, lbfgs.hpp:165-187 */
        ls_copy(&prev, &lo, dim);
        for (int i = 0; i < opts->max_bracket; ++i) {
          EVAL_AT(t);
          if (!SUFFICIENT(trial) || (i > 0 && trial.value <= prev.value)) {
            ls_copy(&lo, &prev, dim);
            hi_t = trial.t;
            have_bracket = 1;
            break;
          }
          if (CURVATURE_OK(trial)) {
            accepted = 1;
            break;
          }
          if (trial.slope <= 0.0) {
            ls_copy(&lo, &trial, dim);
            hi_t = prev.t;
            have_bracket = 1;
            break;
          }
          ls_copy(&prev, &trial, dim);
          t *= 2.0;
        }

        if (!accepted && have_bracket) { /* zoom, lbfgs.hpp:189-231 */
          double hi_value = NAN;
          for (int i = 0; i < opts->max_zoom; ++i) {
            double cand = 0.5 * (lo.t + hi_t);
            if (isfinite(hi_value)) {
              const double dt = hi_t - lo.t;
              const double denom = 2.0 * (lo.value + lo.slope * dt - hi_value);
              if (denom != 0.0) {
                const double interp = lo.t + lo.slope * dt * dt / denom;
                const double lo_guard = lo.t + 0.1 * dt;
                const double hi_guard = hi_t - 0.1 * dt;
                const double lim_min = lo_guard < hi_guard ? lo_guard : hi_guard;
                const double lim_max = lo_guard < hi_guard ? hi_guard : lo_guard;
                if (interp >= lim_min && interp <= lim_max) cand = interp;
              }
            }
            if (cand == lo.t || cand == hi_t) break;
            EVAL_AT(cand);
            if (!SUFFICIENT(trial) || trial.value <= lo.value) {
              hi_t = cand;
              hi_value = trial.value;
              continue;
            }
            if (CURVATURE_OK(trial)) {
              accepted = 1;
              break;
            }
            if (trial.slope * (hi_t - lo.t) <= 0.0) {
              hi_t = lo.t;
              hi_value = lo.value;
            }
            ls_copy(&lo, &trial, dim);
          }
          if (!accepted && lo.t > 0.0) {
            ls_copy(&trial, &lo, dim);
            accepted = 1;
          }
        }
        if (!accepted && !have_bracket && prev.t > 0.0) {
          ls_copy(&trial, &prev, dim);
          accepted = 1;
        }
#undef SUFFICIENT
#undef CURVATURE_OK
      }
      if (zero_gradient) break;
      if (!accepted) {
        stalled = 1;
        break;
      }

      /* curvature pair, lbfgs.hpp:243-255 */
      double* s = (double*)malloc(vb);
      double* y = (double*)malloc(vb);
      for (int64_t e = 0; e < dim; ++e) s[e] = trial.x[e] - x[e];
      for (int64_t e = 0; e < dim; ++e) y[e] = gx[e] - trial.grad[e];
      const double sy = seq_dot(s, y, dim);
      if (sy > 1e-10 * sqrt(seq_dot(s, s, dim)) * sqrt(seq_dot(y, y, dim))) {
        if (k_hist == mem) {
          free(s_hist[0]);
          free(y_hist[0]);
          memmove(s_hist, s_hist + 1, sizeof(double*) * (size_t)(mem - 1));
          memmove(y_hist, y_hist + 1, sizeof(double*) * (size_t)(mem - 1));
          memmove(rho_hist, rho_hist + 1, sizeof(double) * (size_t)(mem - 1));
          --k_hist;
        }
        s_hist[k_hist] = s;
        y_hist[k_hist] = y;
        rho_hist[k_hist] = 1.0 / sy;
        ++k_hist;
      } else {
        free(s);
        free(y);
      }
      memcpy(x, trial.x, vb);
      memcpy(gx, trial.grad, vb);
      fx = trial.value;
      ++res->iterations;
      if (on_accept) on_accept(ctx, res->iterations, x);
    }

    if (stalled) break;
    if (hook) hook(ctx, res->chunks - 1, x);
    if (norm_inf(gx, dim) <= opts->grad_tol) {
      res->converged = 1;
      break;
    }
  }
#undef EVAL_AT
  if (!res->converged) res->converged = norm_inf(gx, dim) <= opts->grad_tol;
  res->line_search_failed = stalled && !res->converged;
  res->objective = fx;
  for (int i = 0; i < k_hist; ++i) {
    free(s_hist[i]);
    free(y_hist[i]);
  }
  free(s_hist);
  free(y_hist);
  free(rho_hist);
  free(two_loop_a);
  free(d);
  free(q);
  free(trial.x);
  free(trial.grad);
  free(lo.x);
  free(lo.grad);
  free(prev.x);
  free(prev.grad);
}

void go_maximize(go_objective_fn f, go_gradient_fn g, go_hook_fn hook, void* ctx, const double* x0,
                 int64_t dim, const go_maximize_options* o, double* x_out, double* grad_out,
                 go_maximize_result* r) {
  maximize_impl(f, g, hook, NULL, ctx, x0, dim, o, x_out, grad_out, r);
}

/* ---------------------------------------------------------------- solver
 * solver.hpp:92-293 */

typedef struct {
  const go_problem* p;
  int mode; /* 0 baseline, 1 fast, 2 fast-no-lb, 3 audit(fast) , 4 audit(no-lb) */
  int use_active_set;
  int audit;
  double ub_offset;
  /* snapshot */
  double *alpha_snap, *beta_snap, *z, *k, *o;
  uint8_t* member;
  /* stats */
  go_solve_result* res;
  int64_t* history;
  int64_t history_cap;
  double *ga, *gb, *gcol, *refcol, *fblock;
  uint8_t* path;
  int violated;
  /* trace */
  double* trace_x;
  int64_t trace_cap, *trace_rows;
} solve_ctx_t;

static double solve_objective(void* vctx, const double* x) { /* solver.hpp:101-104, :161-164 */
  solve_ctx_t* c = (solve_ctx_t*)vctx;
  return go_dual_objective(c->p, x, x + c->p->m);
}

static void push_history(solve_ctx_t* c, const int64_t call[4]) {
  const int64_t row = c->res->grad_calls;
  if (c->history && row < c->history_cap)
    for (int q = 0; q < 4; ++q) c->history[row * 4 + q] = call[q];
  c->res->blocks_in_active_set += call[0];
  c->res->blocks_skipped += call[1];
  c->res->blocks_unskipped += call[2];
  c->res->upper_bounds_evaluated += call[3];
  ++c->res->grad_calls;
}

static void solve_gradient(void* vctx, const double* x, double* out) {
  solve_ctx_t* c = (solve_ctx_t*)vctx;
  const go_problem* p = c->p;
  const double* alpha = x;
  const double* beta = x + p->m;
  if (c->mode == 0) { /* solver.hpp:105-120 */
    go_dual_gradient(p, alpha, beta, out, out + p->m);
    const int64_t call[4] = {0, 0, (int64_t)p->L * p->n, 0};
    push_history(c, call);
    return;
  }
  /* solver.hpp:166-210 */
  int64_t call[4];
  if (c->violated) return;
  go_fast_gradient(p, c->alpha_snap, c->beta_snap, c->z, c->use_active_set ? c->member : NULL,
                   c->ub_offset, alpha, beta, out, out + p->m, call, c->audit ? c->path : NULL);
  if (c->audit) {
    /* re-derive each screened column and compare with the plain provider */
    dispatcher_t ds;
    memset(&ds, 0, sizeof ds);
    ds.p = p;
    ds.alpha_snap = c->alpha_snap;
    ds.beta_snap = c->beta_snap;
    ds.z_snap = c->z;
    ds.member = c->use_active_set ? c->member : NULL;
    ds.ub_offset = c->ub_offset;
    deltas_alloc(&ds.d, p);
    go_delta_norms(p, alpha, beta, c->alpha_snap, c->beta_snap, ds.d.dpos, ds.d.dfull, ds.d.dneg,
                   ds.d.sqrt_g, ds.d.dbeta);
    ds.fblock = c->fblock;
    for (int64_t j = 0; j < p->n && !c->violated; ++j) {
      dispatch_column(&ds, alpha, beta, j, c->gcol, c->path);
      baseline_column(p, alpha, beta, j, c->refcol, c->fblock);
      if (memcmp(c->gcol, c->refcol, sizeof(double) * (size_t)p->m) != 0) c->violated = 1;
      ++c->res->audit_column_compares;
      for (int l = 0; l < p->L && !c->violated; ++l) {
        if (c->path[l + j * p->L] != 1) continue;
        ++c->res->audit_skip_checks;
        for (int i = p->offsets[l]; i < p->offsets[l + 1]; ++i)
          if (c->refcol[i] != 0.0) c->violated = 1;
      }
    }
    deltas_free(&ds.d);
    ++c->res->audit_gradient_calls;
  }
  push_history(c, call);
}

static void solve_hook(void* vctx, int chunk, const double* x) { /* solver.hpp:212-241 */
  solve_ctx_t* c = (solve_ctx_t*)vctx;
  const go_problem* p = c->p;
  (void)chunk;
  if (c->mode == 0) return;
  const double* alpha = x;
  const double* beta = x + p->m;
  if (c->use_active_set) /* screening.hpp:231-235 */
    go_build_active_set(p, c->alpha_snap, c->beta_snap, c->k, c->o, alpha, beta, c->member);
  go_take_snapshot(p, alpha, beta, c->z, c->k, c->o);
  memcpy(c->alpha_snap, alpha, sizeof(double) * (size_t)p->m);
  memcpy(c->beta_snap, beta, sizeof(double) * (size_t)p->n);
  if (c->audit && c->use_active_set) {
    double* f = (double*)malloc(sizeof(double) * (size_t)p->m);
    const double tau = tau_of(p);
    for (int64_t j = 0; j < p->n; ++j) {
      int have = 0;
      for (int l = 0; l < p->L; ++l) {
        if (!c->member[l + j * p->L]) continue;
        if (!have) {
          go_residual_block(alpha, beta[j], p->cost + j * p->m, (int)p->m, f);
          have = 1;
        }
        ++c->res->audit_active_checks;
        const double z = go_pos_part_norm(f + p->offsets[l], p->sizes[l]);
        if (!(z > tau)) c->violated = 1;
      }
    }
    free(f);
  }
}

static void solve_accept(void* vctx, int iteration, const double* x) {
  solve_ctx_t* c = (solve_ctx_t*)vctx;
  (void)iteration;
  if (!c->trace_x || !c->trace_rows || *c->trace_rows >= c->trace_cap) return;
  const int64_t dim = c->p->m + c->p->n;
  memcpy(c->trace_x + (*c->trace_rows) * dim, x, sizeof(double) * (size_t)dim);
  ++*c->trace_rows;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int go_solve(const go_problem* p, const go_solver_options* o, double ub_offset, double* x_out,
             go_solve_result* res, int64_t* history, int64_t history_cap, double* plan,
             double* trace_x, int64_t trace_cap, int64_t* trace_rows) {
  memset(res, 0, sizeof *res);
  int st = go_validate(p, NULL, NULL, NULL, NULL); /* solver.hpp:94, :136 */
  if (st) return st;
  const int64_t m = p->m, n = p->n, L = p->L;
  solve_ctx_t c;
  memset(&c, 0, sizeof c);
  c.p = p;
  c.res = res;
  c.history = history;
  c.history_cap = history_cap;
  c.ub_offset = ub_offset;
  int mode = o->mode;
  if (mode == 3) { /* audit: solver.hpp:268-281 (audit of a fast solve) */
    c.audit = 1;
    c.use_active_set = 1;
    c.mode = 1;
  } else if (mode == 4) { /* audit with fast-no-lb */
    c.audit = 1;
    c.use_active_set = 0;
    c.mode = 2;
  } else {
    c.mode = mode;
    c.use_active_set = (mode == 1);
  }
  c.trace_x = trace_x;
  c.trace_cap = trace_cap;
  c.trace_rows = trace_rows;
  if (c.mode != 0) {
    c.alpha_snap = (double*)calloc((size_t)m, sizeof(double));
    c.beta_snap = (double*)calloc((size_t)n, sizeof(double));
    c.z = (double*)malloc(sizeof(double) * (size_t)(L * n));
    c.k = (double*)malloc(sizeof(double) * (size_t)(L * n));
    c.o = (double*)malloc(sizeof(double) * (size_t)(L * n));
    c.member = (uint8_t*)calloc((size_t)(L * n), 1);
    go_take_snapshot(p, c.alpha_snap, c.beta_snap, c.z, c.k, c.o); /* init, screening.hpp:220-227 */
    c.gcol = (double*)malloc(sizeof(double) * (size_t)m);
    c.refcol = (double*)malloc(sizeof(double) * (size_t)m);
    c.fblock = (double*)malloc(sizeof(double) * (size_t)m);
    c.path = (uint8_t*)calloc((size_t)(L * n), 1);
  }
  go_maximize_options mo; /* solver.hpp:63-70 */
  go_default_maximize_options(&mo);
  mo.chunk_iters = o->snapshot_interval;
  mo.max_chunks = o->max_outer_loops;
  mo.memory = o->lbfgs_memory;
  mo.grad_tol = o->grad_tol;
  double* x0 = (double*)calloc((size_t)(m + n), sizeof(double));
  double* g = (double*)malloc(sizeof(double) * (size_t)(m + n));
  go_maximize_result mr;
  const double t0 = now_s();
  if (trace_x && trace_rows) { /* row 0 = x0, then every accepted iterate */
    *trace_rows = 0;
    if (trace_cap > 0) {
      memcpy(trace_x, x0, sizeof(double) * (size_t)(m + n));
      *trace_rows = 1;
    }
  }
  maximize_impl(solve_objective, solve_gradient, c.mode != 0 ? solve_hook : NULL,
                trace_x ? solve_accept : NULL, &c, x0, m + n, &mo, x_out, g, &mr);
  const double t1 = now_s();
  res->wall_seconds = t1 - t0;
  res->iterations = mr.iterations;
  res->chunks = mr.chunks;
  res->converged = mr.converged;
  res->line_search_failed = mr.line_search_failed;
  res->outer_loops = mr.chunks;
  /* finish_solution, solver.hpp:72-87 */
  res->objective = go_dual_objective(p, x_out, x_out + m);
  if (plan) go_recover_plan(p, x_out, x_out + m, plan);
  free(x0);
  free(g);
  free(c.alpha_snap);
  free(c.beta_snap);
  free(c.z);
  free(c.k);
  free(c.o);
  free(c.member);
  free(c.gcol);
  free(c.refcol);
  free(c.fblock);
  free(c.path);
  return c.violated ? ST_AUDIT : ST_OK;
}

/* ---------------------------------------------------------------- data
 * data_io.hpp:32-62: std::mt19937_64 (restated from its published
 * definition), uniforms (x >> 11) * 2^-53, Box-Muller normals with a cached
 * spare, index = engine() % bound. */

#define MT_N 312
#define MT_M 156
void go_rng_seed(go_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->mti = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

uint64_t go_rng_next(go_rng* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL,
                        MA = 0xB5026F5AA96619E9ULL;
  if (r->mti >= MT_N) {
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
      const uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    }
    for (; i < MT_N - 1; ++i) {
      const uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    }
    const uint64_t x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MA : 0ULL);
    r->mti = 0;
  }
  uint64_t y = r->mt[r->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

double go_rng_uniform01(go_rng* r) { return (double)(go_rng_next(r) >> 11) * 0x1.0p-53; }

double go_rng_normal(go_rng* r) { /* data_io.hpp:40-53 */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = go_rng_uniform01(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  const double u2 = go_rng_uniform01(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rr * sin(angle);
  r->has_spare = 1;
  return rr * cos(angle);
}

uint64_t go_rng_index(go_rng* r, uint64_t bound) { return go_rng_next(r) % bound; }

void go_cost_matrix(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                    double* cost) { /* data_io.hpp:101-123; src m x d, tgt n x d row-major here */
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t k = 0; k < d; ++k) {
        const double diff = src[i * d + k] - tgt[j * d + k];
        acc += diff * diff;
      }
      cost[i + j * m] = acc;
    }
  }
}

typedef struct {
  const double *src, *tgt;
  int64_t m, n, d, j0, j1;
  double* cost;
} cm_job_t;

static void* cm_worker(void* v) {
  cm_job_t* jb = (cm_job_t*)v;
  for (int64_t j = jb->j0; j < jb->j1; ++j) {
    for (int64_t i = 0; i < jb->m; ++i) {
      double acc = 0.0;
      for (int64_t k = 0; k < jb->d; ++k) {
        const double diff = jb->src[i * jb->d + k] - jb->tgt[j * jb->d + k];
        acc += diff * diff;
      }
      jb->cost[i + j * jb->m] = acc;
    }
  }
  return NULL;
}

void go_cost_matrix_par(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                        double* cost, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  cm_job_t* jobs = (cm_job_t*)malloc(sizeof(cm_job_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].src = src;
    jobs[t].tgt = tgt;
    jobs[t].m = m;
    jobs[t].n = n;
    jobs[t].d = d;
    jobs[t].j0 = n * t / nthreads;
    jobs[t].j1 = n * (t + 1) / nthreads;
    jobs[t].cost = cost;
    pthread_create(&th[t], NULL, cm_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

/* ---------------------------------------------------------------- configs */

typedef struct {
  int64_t m, n;
  int32_t L;
  int64_t d;
  double sigma;
  int transform, zipf, dirichlet;
} cfg_spec_t;

static int cfg_spec(int cfg, cfg_spec_t* s) {
  static const cfg_spec_t T[5] = {{1000, 1000, 10, 64, 1.0, 1, 0, 0},
                                  {10000, 10000, 100, 128, 1.0, 0, 0, 0},
                                  {50000, 20000, 1000, 256, 1.0, 2, 0, 0},
                                  {40000, 30000, 500, 128, 1.0, 0, 1, 1},
                                  {100000, 50000, 200, 512, 1.5, 0, 0, 0}};
  if (cfg < 1 || cfg > 5) return ST_PARAM;
  *s = T[cfg - 1];
  return ST_OK;
}

int go_config_shape(int cfg, int64_t* m, int64_t* n, int32_t* L, int64_t* d) {
  cfg_spec_t s;
  if (cfg_spec(cfg, &s)) return ST_PARAM;
  if (m) *m = s.m;
  if (n) *n = s.n;
  if (L) *L = s.L;
  if (d) *d = s.d;
  return ST_OK;
}

static int64_t zipf_total(double c, int32_t L, int32_t* out) {
  int64_t tot = 0;
  for (int k = 1; k <= L; ++k) {
    double v = round(c * pow((double)k, -1.1));
    v = fmin(4000.0, fmax(2.0, v));
    if (out) out[k - 1] = (int32_t)v;
    tot += (int64_t)v;
  }
  return tot;
}

int go_config_features(int cfg, uint64_t seed, double* src, double* tgt, int32_t* sizes,
                       double* a, double* b) {
  cfg_spec_t s;
  if (cfg_spec(cfg, &s)) return ST_PARAM;
  const int64_t m = s.m, n = s.n, d = s.d;
  const int32_t L = s.L;
  if (s.zipf) {
    double lo = 1.0, hi = 1e7;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (zipf_total(mid, L, NULL) >= m)
        hi = mid;
      else
        lo = mid;
    }
    const int64_t tot = zipf_total(hi, L, sizes);
    sizes[1] -= (int32_t)(tot - m);
  } else {
    for (int32_t l = 0; l < L; ++l) sizes[l] = (int32_t)(m / L);
  }
  go_rng rng;
  go_rng_seed(&rng, seed);
  double* means = (double*)malloc(sizeof(double) * (size_t)(L * d));
  for (int64_t e = 0; e < L * d; ++e) means[e] = 2.0 * go_rng_normal(&rng);
  int64_t row = 0;
  for (int32_t l = 0; l < L; ++l)
    for (int32_t r = 0; r < sizes[l]; ++r, ++row)
      for (int64_t k = 0; k < d; ++k)
        src[row * d + k] = means[l * d + k] + s.sigma * go_rng_normal(&rng);
  const int64_t per = n / L;
  for (int64_t t = 0; t < n; ++t)
    for (int64_t k = 0; k < d; ++k)
      tgt[t * d + k] = means[(t / per) * d + k] + s.sigma * go_rng_normal(&rng);
  if (s.transform) {
    double* G = (double*)malloc(sizeof(double) * (size_t)(d * d));
    double* A = (double*)malloc(sizeof(double) * (size_t)(d * d));
    double* shift = (double*)malloc(sizeof(double) * (size_t)d);
    double* y = (double*)malloc(sizeof(double) * (size_t)d);
    for (int64_t e = 0; e < d * d; ++e) G[e] = go_rng_normal(&rng);
    for (int64_t r = 0; r < d; ++r) shift[r] = 0.5;
    if (s.transform == 1) { /* modified Gram-Schmidt, positive R diagonal */
      memcpy(A, G, sizeof(double) * (size_t)(d * d));
      for (int64_t c = 0; c < d; ++c) {
        for (int64_t p = 0; p < c; ++p) {
          double dot = 0.0;
          for (int64_t r = 0; r < d; ++r) dot += A[r * d + p] * A[r * d + c];
          for (int64_t r = 0; r < d; ++r) A[r * d + c] -= dot * A[r * d + p];
        }
        double nrm = 0.0;
        for (int64_t r = 0; r < d; ++r) nrm += A[r * d + c] * A[r * d + c];
        nrm = sqrt(nrm);
        for (int64_t r = 0; r < d; ++r) A[r * d + c] /= nrm;
      }
    } else {
      const double sc = 0.1 / sqrt((double)d);
      for (int64_t r = 0; r < d; ++r)
        for (int64_t c = 0; c < d; ++c) A[r * d + c] = (r == c ? 1.0 : 0.0) + sc * G[r * d + c];
      for (int64_t r = 0; r < d; ++r) shift[r] = go_rng_normal(&rng);
    }
    for (int64_t t = 0; t < n; ++t) {
      for (int64_t r = 0; r < d; ++r) {
        double acc = 0.0;
        for (int64_t c = 0; c < d; ++c) acc += A[r * d + c] * tgt[t * d + c];
        y[r] = acc + shift[r];
      }
      memcpy(tgt + t * d, y, sizeof(double) * (size_t)d);
    }
    free(G);
    free(A);
    free(shift);
    free(y);
  }
  for (int64_t i = n - 1; i > 0; --i) { /* data_io.hpp:93-96 */
    const int64_t j = (int64_t)go_rng_index(&rng, (uint64_t)i + 1);
    if (i != j)
      for (int64_t k = 0; k < d; ++k) {
        const double t = tgt[i * d + k];
        tgt[i * d + k] = tgt[j * d + k];
        tgt[j * d + k] = t;
      }
  }
  if (s.dirichlet) {
    double* e = (double*)malloc(sizeof(double) * (size_t)m);
    for (int64_t i = 0; i < m; ++i) {
      double u = go_rng_uniform01(&rng);
      if (u <= 0.0) u = 0x1.0p-53;
      e[i] = -log(u);
    }
    const double sum = go_compensated_sum(e, m);
    for (int64_t i = 0; i < m; ++i) a[i] = e[i] / sum;
    free(e);
  } else {
    for (int64_t i = 0; i < m; ++i) a[i] = 1.0 / (double)m;
  }
  for (int64_t j = 0; j < n; ++j) b[j] = 1.0 / (double)n;
  free(means);
  return ST_OK;
}
