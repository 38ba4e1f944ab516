// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (oracle/).
//
// Exposes the UNMODIFIED reference library (/root/reference/proj/include/
// groupot, compiled against oracle/shim/Eigen) through a small C ABI so that
// tests can (1) pin the C restatement oracle/gsot_oracle.c against the real
// reference and (2) generate tests/golden/ fixtures, and so that
// `bench.py --impl reference` can time the reference's own solver on the
// GPU box's host cores. Built into oracle/_ref/ by oracle/Makefile; never
// linked into the product.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "groupot/data_io.hpp"
#include "groupot/solver.hpp"

using namespace groupot;

namespace {

thread_local std::string g_err;

ProblemInstance make(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                     const double* a, const double* b) {
  Eigen::MatrixXd c(m, n);
  std::memcpy(c.data(), cost, sizeof(double) * static_cast<size_t>(m * n));
  Eigen::VectorXd av(m), bv(n);
  std::memcpy(av.data(), a, sizeof(double) * static_cast<size_t>(m));
  std::memcpy(bv.data(), b, sizeof(double) * static_cast<size_t>(n));
  return ProblemInstance{std::move(c), std::move(av), std::move(bv),
                         GroupPartition(std::vector<int>(sizes, sizes + L))};
}

DualState state(const double* alpha, const double* beta, int64_t m, int64_t n) {
  DualState s{Eigen::VectorXd(m), Eigen::VectorXd(n)};
  std::memcpy(s.alpha.data(), alpha, sizeof(double) * static_cast<size_t>(m));
  std::memcpy(s.beta.data(), beta, sizeof(double) * static_cast<size_t>(n));
  return s;
}

// Status codes of include/gsot.h.
int map_exception() {
  try {
    throw;
  } catch (const NegativeCost& e) {
    g_err = e.what();
    return 2;
  } catch (const MarginalNotNormalized& e) {
    g_err = e.what();
    return 3;
  } catch (const PartitionMismatch& e) {
    g_err = e.what();
    return 4;
  } catch (const DimensionMismatch& e) {
    g_err = e.what();
    return 1;
  } catch (const RhoOutOfRange& e) {
    g_err = e.what();
    return 6;
  } catch (const AuditViolation& e) {
    g_err = e.what();
    return 7;
  } catch (const Error& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                 const double* a, const double* b, double gamma, double mu, int64_t* row,
                 int64_t* col, char* which, int64_t* index) {
  try {
    RegParams p(gamma, mu);
    (void)p;
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    validate_instance(inst);
    return 0;
  } catch (const NegativeCost& e) {
    if (row) *row = e.row;
    if (col) *col = e.col;
    g_err = e.what();
    return 2;
  } catch (const MarginalNotNormalized& e) {
    if (which) *which = e.which;
    if (index) *index = e.index;
    g_err = e.what();
    return 3;
  } catch (...) {
    return map_exception();
  }
}

int ref_eval(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
             const double* a, const double* b, double gamma, double mu, const double* alpha,
             const double* beta, double* objective, double* ga, double* gb) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    RegParams p(gamma, mu);
    DualState s = state(alpha, beta, m, n);
    *objective = dual_objective(s, inst, p);
    Eigen::VectorXd gav, gbv;
    dual_gradient(s, inst, p, gav, gbv);
    std::memcpy(ga, gav.data(), sizeof(double) * static_cast<size_t>(m));
    std::memcpy(gb, gbv.data(), sizeof(double) * static_cast<size_t>(n));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// plan_diagnostics(recover_plan(x)) (dual.hpp:116-169); out = {res_a, res_b,
// group_sparsity, mass}. plan_in (optional) replaces the recovered plan.
int ref_plan_diagnostics(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                         const double* a, const double* b, const double* plan_in, double* out) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    TransportPlan t;
    t.plan.resize(m, n);
    std::memcpy(t.plan.data(), plan_in, sizeof(double) * static_cast<size_t>(m * n));
    const PlanDiagnostics d = plan_diagnostics(t, inst);
    out[0] = d.marginal_res_a;
    out[1] = d.marginal_res_b;
    out[2] = d.group_sparsity;
    out[3] = d.mass;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// primal_objective(plan, inst, p) (core.hpp:167-180) of a given m x n plan.
int ref_primal_objective(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                         const double* a, const double* b, double gamma, double mu,
                         const double* plan_in, double* out) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    TransportPlan t;
    t.plan.resize(m, n);
    std::memcpy(t.plan.data(), plan_in, sizeof(double) * static_cast<size_t>(m * n));
    *out = primal_objective(t, inst, RegParams(gamma, mu));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_plan(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
             const double* a, const double* b, double gamma, double mu, const double* alpha,
             const double* beta, double* plan) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    RegParams p(gamma, mu);
    TransportPlan t = recover_plan(state(alpha, beta, m, n), inst, p);
    std::memcpy(plan, t.plan.data(), sizeof(double) * static_cast<size_t>(m * n));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_snapshot(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                 const double* a, const double* b, const double* alpha, const double* beta,
                 double* z, double* k, double* o) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    SnapshotStore snap = take_snapshot(state(alpha, beta, m, n), inst);
    const size_t bytes = sizeof(double) * static_cast<size_t>(L * n);
    std::memcpy(z, snap.z_snap.data(), bytes);
    std::memcpy(k, snap.k_snap.data(), bytes);
    std::memcpy(o, snap.o_snap.data(), bytes);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// build_active_set(snapshot at (alpha_s, beta_s), state (alpha, beta)).
int ref_active_set(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                   const double* a, const double* b, double gamma, double mu,
                   const double* alpha_s, const double* beta_s, const double* alpha,
                   const double* beta, uint8_t* member, int64_t* count) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    RegParams p(gamma, mu);
    SnapshotStore snap = take_snapshot(state(alpha_s, beta_s, m, n), inst);
    ActiveSet as = build_active_set(snap, state(alpha, beta, m, n), p, inst.groups);
    std::memcpy(member, as.member.data(), as.member.size());
    *count = as.count;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// One FastGradDispatcher gradient call: snapshot at (alpha_s, beta_s); the
// active set built against the snapshot at (alpha_a, beta_a) first when
// use_active_set (refresh order of screening.hpp:231-235: active set from
// the OLD snapshot, then a new snapshot), i.e. this reproduces the
// dispatcher state after `init(x_a)` then `refresh(x_s)`:
//   active = build_active_set(snap(x_a), x_s); snap = take_snapshot(x_s).
// Then gradient at (alpha, beta). counters: in_active, skipped, unskipped,
// upper_bounds.
int ref_fast_gradient(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                      const double* a, const double* b, double gamma, double mu,
                      const double* alpha_a, const double* beta_a, const double* alpha_s,
                      const double* beta_s, int use_active_set, double ub_offset,
                      const double* alpha, const double* beta, double* ga, double* gb,
                      int64_t* counters, uint8_t* member_out) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    RegParams p(gamma, mu);
    GradStats stats;
    FastGradDispatcher disp(inst, p, stats, use_active_set != 0, ub_offset);
    disp.init(state(alpha_a, beta_a, m, n));
    disp.refresh(state(alpha_s, beta_s, m, n), 1);
    if (member_out)
      std::memcpy(member_out, disp.active_set().member.data(), disp.active_set().member.size());
    DualState s = state(alpha, beta, m, n);
    disp.begin_call(s);
    Eigen::VectorXd gav, gbv;
    dual_gradient(
        s, inst, p, [&](int j, Eigen::VectorXd& gcol) { disp.column(j, gcol); }, gav, gbv);
    disp.end_call();
    std::memcpy(ga, gav.data(), sizeof(double) * static_cast<size_t>(m));
    std::memcpy(gb, gbv.data(), sizeof(double) * static_cast<size_t>(n));
    const auto& h = stats.history.back();
    counters[0] = h.in_active;
    counters[1] = h.skipped;
    counters[2] = h.unskipped;
    counters[3] = h.upper_bounds;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Timing sample of the reference hot path (bench.py: the reference arm and
// cpu_baseline). The instance is built once (its copy is not timed); then,
// timed with steady_clock as solver.hpp:243-246 times maximize:
//   times[2] += FastGradDispatcher init(x_a) + refresh(x_s): two take_snapshot
//               passes and one build_active_set (screening.hpp:220-235);
//   times[0] += dual_objective(x)                      (dual.hpp:38-52, dense
//               in every mode, solver.hpp:161-164);
//   times[1] += dual_gradient(x) through the dispatcher (screening.hpp:239-287).
// repeated `reps` times. counters: the last gradient call's GradStats row.
int ref_time_eval(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
                  const double* a, const double* b, double gamma, double mu,
                  const double* alpha_a, const double* beta_a, const double* alpha_s,
                  const double* beta_s, const double* alpha, const double* beta, int reps,
                  double* times, int64_t* counters, double* objective) {
  try {
    using clock = std::chrono::steady_clock;
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    RegParams p(gamma, mu);
    DualState sa = state(alpha_a, beta_a, m, n), ss = state(alpha_s, beta_s, m, n),
              s = state(alpha, beta, m, n);
    times[0] = times[1] = times[2] = 0.0;
    for (int r = 0; r < reps; ++r) {
      GradStats stats;
      FastGradDispatcher disp(inst, p, stats, true, 0.0);
      auto t0 = clock::now();
      disp.init(sa);
      disp.refresh(ss, 1);
      auto t1 = clock::now();
      *objective = dual_objective(s, inst, p);
      auto t2 = clock::now();
      disp.begin_call(s);
      Eigen::VectorXd gav, gbv;
      dual_gradient(
          s, inst, p, [&](int j, Eigen::VectorXd& gcol) { disp.column(j, gcol); }, gav, gbv);
      disp.end_call();
      auto t3 = clock::now();
      times[2] += std::chrono::duration<double>(t1 - t0).count();
      times[0] += std::chrono::duration<double>(t2 - t1).count();
      times[1] += std::chrono::duration<double>(t3 - t2).count();
      const auto& h = stats.history.back();
      counters[0] = h.in_active;
      counters[1] = h.skipped;
      counters[2] = h.unskipped;
      counters[3] = h.upper_bounds;
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// load_csv (data_io.hpp:270-352): shape query, then the data. Errors map to
// status codes: 11 ParseError (detail line/col), 12 MissingLabelColumn,
// 13 InconsistentDimension (detail line), 5 other Error; msg via
// ref_last_error.
int ref_load_csv(const char* src_path, const char* tgt_path, int64_t* shape /* m, n, d, sw, tw */,
                 int64_t* detail /* line, column */, double* src_feat, int32_t* labels,
                 double* src_w, double* tgt_feat, double* tgt_w) {
  try {
    auto [src, tgt] = load_csv(src_path, tgt_path);
    shape[0] = src.features.rows();
    shape[1] = tgt.features.rows();
    shape[2] = src.features.cols();
    shape[3] = src.weights.size();
    shape[4] = tgt.weights.size();
    if (src_feat)
      for (Eigen::Index i = 0; i < src.features.rows(); ++i)
        for (Eigen::Index k = 0; k < src.features.cols(); ++k)
          src_feat[i * src.features.cols() + k] = src.features(i, k);
    if (labels)
      for (size_t i = 0; i < src.labels.size(); ++i) labels[i] = src.labels[i];
    if (src_w)
      for (Eigen::Index i = 0; i < src.weights.size(); ++i) src_w[i] = src.weights[i];
    if (tgt_feat)
      for (Eigen::Index i = 0; i < tgt.features.rows(); ++i)
        for (Eigen::Index k = 0; k < tgt.features.cols(); ++k)
          tgt_feat[i * tgt.features.cols() + k] = tgt.features(i, k);
    if (tgt_w)
      for (Eigen::Index i = 0; i < tgt.weights.size(); ++i) tgt_w[i] = tgt.weights[i];
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    detail[0] = e.line;
    detail[1] = e.column;
    return 11;
  } catch (const MissingLabelColumn& e) {
    g_err = e.what();
    return 12;
  } catch (const InconsistentDimension& e) {
    g_err = e.what();
    detail[0] = e.line;
    return 13;
  } catch (...) {
    return map_exception();
  }
}

// make_instance (data_io.hpp:157-181) from the two CSV files: cost (m x n
// column-major), a, b, group sizes (L, up to m entries).
int ref_make_instance(const char* src_path, const char* tgt_path, int normalize, int use_weights,
                      double* cost, double* a, double* b, int32_t* sizes, int32_t* L) {
  try {
    auto [src, tgt] = load_csv(src_path, tgt_path);
    ProblemInstance inst = make_instance(src, tgt, normalize != 0, use_weights != 0);
    std::memcpy(cost, inst.cost.data(), sizeof(double) * inst.cost.size());
    std::memcpy(a, inst.a.data(), sizeof(double) * inst.a.size());
    std::memcpy(b, inst.b.data(), sizeof(double) * inst.b.size());
    *L = inst.groups.num_groups();
    for (int l = 0; l < *L; ++l) sizes[l] = inst.groups.size(l);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// partition_from_labels (data_io.hpp:127-152): sizes into out (up to n).
int ref_partition_from_labels(const int32_t* labels, int64_t n, int32_t* out, int32_t* L) {
  try {
    GroupPartition g = partition_from_labels(std::vector<int>(labels, labels + n));
    *L = g.num_groups();
    for (int l = 0; l < *L; ++l) out[l] = g.size(l);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// solve(): mode 0 baseline, 1 fast, 2 fast-no-lb, 3 audit, 4 audit of fast-no-lb. out_scalars:
// [objective, wall_seconds]; out_ints: [iterations, converged,
// line_search_failed, outer_loops, grad_calls, in_active, skipped,
// unskipped, upper_bounds]. history: grad_calls x 4 (cap rows). plan
// optional (m x n col-major).
int ref_solve(const double* cost, int64_t m, int64_t n, const int32_t* sizes, int32_t L,
              const double* a, const double* b, double gamma, double mu, int mode,
              int snapshot_interval, double grad_tol, int max_outer_loops, int lbfgs_memory,
              double ub_offset, double* x_out, double* out_scalars, int64_t* out_ints,
              int64_t* history, int64_t history_cap, double* plan) {
  try {
    ProblemInstance inst = make(cost, m, n, sizes, L, a, b);
    RegParams p(gamma, mu);
    SolverOptions o;
    o.snapshot_interval = snapshot_interval;
    o.grad_tol = grad_tol;
    o.max_outer_loops = max_outer_loops;
    o.lbfgs_memory = lbfgs_memory;
    // mode 4: audit_solve of a fast_no_lower_bound SolverOptions (solver.hpp:271)
    o.mode = mode == 0                ? SolverMode::baseline
             : mode == 1              ? SolverMode::fast
             : mode == 2 || mode == 4 ? SolverMode::fast_no_lower_bound
                                      : SolverMode::audit;
    Solution sol = mode >= 3 ? audit_solve(inst, p, o, ub_offset).first : solve(inst, p, o);
    std::memcpy(x_out, sol.state.alpha.data(), sizeof(double) * static_cast<size_t>(m));
    std::memcpy(x_out + m, sol.state.beta.data(), sizeof(double) * static_cast<size_t>(n));
    out_scalars[0] = sol.objective;
    out_scalars[1] = std::chrono::duration<double>(sol.wall_time).count();
    out_ints[0] = sol.iterations;
    out_ints[1] = sol.converged;
    out_ints[2] = sol.line_search_failed;
    out_ints[3] = sol.stats.outer_loops;
    out_ints[4] = sol.stats.grad_calls;
    out_ints[5] = sol.stats.blocks_in_active_set;
    out_ints[6] = sol.stats.blocks_skipped;
    out_ints[7] = sol.stats.blocks_unskipped;
    out_ints[8] = sol.stats.upper_bounds_evaluated;
    if (history) {
      const int64_t rows = std::min<int64_t>(history_cap, static_cast<int64_t>(sol.stats.history.size()));
      for (int64_t r = 0; r < rows; ++r) {
        const auto& h = sol.stats.history[static_cast<size_t>(r)];
        history[r * 4 + 0] = h.in_active;
        history[r * 4 + 1] = h.skipped;
        history[r * 4 + 2] = h.unskipped;
        history[r * 4 + 3] = h.upper_bounds;
      }
    }
    if (plan) std::memcpy(plan, sol.plan.plan.data(), sizeof(double) * static_cast<size_t>(m * n));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Reference Rng stream (data_io.hpp:32-62): kind 0 raw engine(), 1 uniform01,
// 2 normal, 3 index(bound).
void ref_rng_stream(uint64_t seed, int kind, uint64_t bound, int64_t count, double* out_d,
                    uint64_t* out_u) {
  Rng rng(seed);
  for (int64_t i = 0; i < count; ++i) {
    switch (kind) {
      case 1: out_d[i] = rng.uniform01(); break;
      case 2: out_d[i] = rng.normal(); break;
      case 3: out_u[i] = rng.index(bound); break;
      default: {
        // Rng hides its engine; a fresh std::mt19937_64 with the same seed is
        // the documented engine (data_io.hpp:59).
        static thread_local std::mt19937_64* eng = nullptr;
        if (i == 0) {
          delete eng;
          eng = new std::mt19937_64(seed);
        }
        out_u[i] = (*eng)();
      }
    }
  }
}

// The paper's d=2 generator + make_instance (data_io.hpp:67-98, :157-181),
// normalize_cost as requested. Outputs cost (m x n col-major, m = n =
// classes*per_class), a, b, sizes (classes).
int ref_gen_synthetic(int num_classes, int per_class, uint64_t seed, int normalize, double* cost,
                      double* a, double* b, int32_t* sizes, double* src_feat, double* tgt_feat) {
  try {
    auto [src, tgt] = gen_synthetic(num_classes, per_class, seed);
    ProblemInstance inst = make_instance(src, tgt, normalize != 0);
    const int64_t m = inst.m(), n = inst.n();
    std::memcpy(cost, inst.cost.data(), sizeof(double) * static_cast<size_t>(m * n));
    std::memcpy(a, inst.a.data(), sizeof(double) * static_cast<size_t>(m));
    std::memcpy(b, inst.b.data(), sizeof(double) * static_cast<size_t>(n));
    for (int l = 0; l < inst.groups.num_groups(); ++l) sizes[l] = inst.groups.size(l);
    if (src_feat)
      for (int64_t i = 0; i < m; ++i)
        for (int k = 0; k < 2; ++k) src_feat[i * 2 + k] = src.features(i, k);
    if (tgt_feat)
      for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 2; ++k) tgt_feat[i * 2 + k] = tgt.features(i, k);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Reference cost_matrix on row-major feature arrays (data_io.hpp:101-123).
void ref_cost_matrix(const double* src, int64_t m, const double* tgt, int64_t n, int64_t d,
                     double* cost) {
  LabeledSamples s;
  UnlabeledSamples t;
  s.features.resize(m, d);
  t.features.resize(n, d);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = 0; k < d; ++k) s.features(i, k) = src[i * d + k];
  for (int64_t j = 0; j < n; ++j)
    for (int64_t k = 0; k < d; ++k) t.features(j, k) = tgt[j * d + k];
  Eigen::MatrixXd c = cost_matrix(s, t);
  std::memcpy(cost, c.data(), sizeof(double) * static_cast<size_t>(m * n));
}

}  // extern "C"
