// groupot_b200.hpp — drop-in adapter: the reference `groupot` C++ API on
// top of the B200 C ABI (gsot.h).
//
// Include AFTER the reference headers ("groupot/solver.hpp"). It adds the
// namespace groupot::b200 with the same entry points and types as the
// reference's solver.hpp / dual.hpp / screening.hpp, backed by libgsot.so:
//
//   reference                                  drop-in
//   groupot::solve(inst, p, opts)              groupot::b200::solve(inst, p, opts)
//   groupot::solve_baseline / solve_fast       groupot::b200::solve_baseline / solve_fast
//   groupot::audit_solve(inst, p, opts, off)   groupot::b200::audit_solve(...)
//   groupot::dual_objective(s, inst, p)        groupot::b200::Device::objective(s)
//   groupot::dual_gradient(s, inst, p, ga, gb) groupot::b200::Device::gradient(s, ga, gb)
//   groupot::recover_plan(s, inst, p)          groupot::b200::Device::plan(s)
//   ObjectiveFn / GradientFn closures          groupot::b200::Device::callbacks()
//   FastGradDispatcher + run_screened wiring   groupot::b200::Device::screened_callbacks()
//   plan_diagnostics(recover_plan(s), inst)    groupot::b200::Device::plan_diagnostics(s)
//   groupot::run_grid(inst, grid, nc, pc, sink) groupot::b200::run_grid(...) (one warm
//                                              device context for the whole grid;
//                                              uses "groupot/bench.hpp" when on the path)
//
// Inputs are read straight from the Eigen storage (column-major cost, as
// ProblemInstance holds it, solver.hpp:47-55); status codes are rethrown as
// the reference's exception classes (errors.hpp) with their fields.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "gsot.h"
#if __has_include("groupot/bench.hpp")
#include "groupot/bench.hpp"    // BenchRecord, GridSpec (run_grid)
#include "groupot/data_io.hpp"  // LabeledSamples, UnlabeledSamples, partition_from_labels
#define GSOT_B200_HAVE_BENCH 1
#else
#define GSOT_B200_HAVE_BENCH 0
#endif

namespace groupot {
namespace b200 {

// Status -> the reference's exception types (errors.hpp:9-89).
inline void check(int st) {
  if (st == GSOT_OK) return;
  gsot_error_detail d;
  gsot_last_error_detail(&d);
  std::string msg = gsot_last_error();
  auto strip = [&](const char* prefix) {
    const std::string p(prefix);
    if (msg.compare(0, p.size(), p) == 0) msg = msg.substr(p.size());
  };
  switch (st) {
    case GSOT_ERR_DIMENSION_MISMATCH: strip("dimension mismatch: "); throw DimensionMismatch(msg);
    case GSOT_ERR_NEGATIVE_COST: throw NegativeCost(d.row, d.col, d.value);
    case GSOT_ERR_MARGINAL_NOT_NORMALIZED:
      strip(std::string("marginal ").append(1, d.which).append(": ").c_str());
      throw MarginalNotNormalized(d.which, d.index, msg);
    case GSOT_ERR_PARTITION_MISMATCH: strip("group partition: "); throw PartitionMismatch(msg);
    case GSOT_ERR_RHO_OUT_OF_RANGE: throw RhoOutOfRange(d.value);
    case GSOT_ERR_AUDIT_VIOLATION: strip("audit violation: "); throw AuditViolation(msg);
    default: throw Error(msg);
  }
}

// The resident instance on the GPU (one gsot_ctx).
class Device {
 public:
  Device(const ProblemInstance& inst, const RegParams& p) : m_(inst.m()), n_(inst.n()) {
    std::vector<int32_t> sizes(inst.groups.sizes().begin(), inst.groups.sizes().end());
    if (inst.a.size() != m_ || inst.b.size() != n_) {
      // validate_instance order (core.hpp:117-131): the cost scan comes
      // first; gsot_create cannot take mismatched marginals, so it runs here.
      for (Eigen::Index j = 0; j < n_; ++j)
        for (Eigen::Index i = 0; i < m_; ++i) {
          const double c = inst.cost(i, j);
          if (!(c >= 0.0) || !std::isfinite(c)) throw NegativeCost(i, j, c);
        }
      if (inst.a.size() != m_)
        throw DimensionMismatch("marginal a has length " + std::to_string(inst.a.size()) +
                                ", cost has " + std::to_string(m_) + " rows");
      throw DimensionMismatch("marginal b has length " + std::to_string(inst.b.size()) +
                              ", cost has " + std::to_string(n_) + " columns");
    }
    check(gsot_create(inst.cost.data(), m_, n_, sizes.data(), static_cast<int32_t>(sizes.size()),
                      inst.a.data(), inst.b.data(), p.gamma(), p.mu(), &ctx_));
  }
  // make_instance (data_io.hpp:157-181) straight into HBM: the cost of the
  // samples (cost_matrix, data_io.hpp:101-123) is computed on the device,
  // divided by its maximum when normalize_cost, with make_instance's
  // marginals (uniform, or the normalised sample weights when use_weights)
  // and partition_from_labels; validated like validate_instance. The
  // m x n cost never exists on the host (gsot_create_features).
  Device(const LabeledSamples& src, const UnlabeledSamples& tgt, bool normalize_cost,
         bool use_weights, const RegParams& p)
      : m_(src.features.rows()), n_(tgt.features.rows()) {
    const Eigen::Index d = src.features.cols();
    if (tgt.features.cols() != d)
      throw InconsistentDimension(1, "target has " + std::to_string(tgt.features.cols()) +
                                         " features, source has " + std::to_string(d));
    const GroupPartition groups = partition_from_labels(src.labels);
    std::vector<int32_t> sizes(groups.sizes().begin(), groups.sizes().end());
    Eigen::VectorXd a, b;
    if (use_weights && src.weights.size() == m_)
      a = src.weights / src.weights.sum();
    else
      a = Eigen::VectorXd::Constant(m_, 1.0 / static_cast<double>(m_));
    if (use_weights && tgt.weights.size() == n_)
      b = tgt.weights / tgt.weights.sum();
    else
      b = Eigen::VectorXd::Constant(n_, 1.0 / static_cast<double>(n_));
    std::vector<double> sf(static_cast<size_t>(m_ * d)), tf(static_cast<size_t>(n_ * d));
    for (Eigen::Index i = 0; i < m_; ++i)  // row-major features
      for (Eigen::Index k = 0; k < d; ++k) sf[static_cast<size_t>(i * d + k)] = src.features(i, k);
    for (Eigen::Index j = 0; j < n_; ++j)
      for (Eigen::Index k = 0; k < d; ++k) tf[static_cast<size_t>(j * d + k)] = tgt.features(j, k);
    check(gsot_create_features(sf.data(), m_, tf.data(), n_, d, sizes.data(),
                               static_cast<int32_t>(sizes.size()), a.data(), b.data(),
                               normalize_cost ? 1 : 0, p.gamma(), p.mu(), &ctx_));
  }
  ~Device() { gsot_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  gsot_ctx* handle() const { return ctx_; }
  Eigen::Index m() const { return m_; }
  Eigen::Index n() const { return n_; }

  // dual_objective (dual.hpp:38-52)
  double objective(const DualState& s) {
    double obj = 0.0;
    pack(s);
    check(gsot_eval(ctx_, x_.data(), GSOT_EVAL_DENSE, &obj, nullptr, nullptr));
    return obj;
  }
  // dual_gradient (dual.hpp:85-100)
  void gradient(const DualState& s, Eigen::VectorXd& ga, Eigen::VectorXd& gb) {
    pack(s);
    g_.resize(static_cast<size_t>(m_ + n_));
    check(gsot_eval(ctx_, x_.data(), GSOT_EVAL_DENSE, nullptr, g_.data(), nullptr));
    ga.resize(m_);
    gb.resize(n_);
    std::memcpy(ga.data(), g_.data(), sizeof(double) * static_cast<size_t>(m_));
    std::memcpy(gb.data(), g_.data() + m_, sizeof(double) * static_cast<size_t>(n_));
  }
  // recover_plan (dual.hpp:116-128)
  TransportPlan plan(const DualState& s) {
    pack(s);
    TransportPlan t;
    t.plan.resize(m_, n_);
    check(gsot_plan_columns(ctx_, x_.data(), 0, n_, t.plan.data()));
    return t;
  }
  // plan_diagnostics(recover_plan(s), inst) (dual.hpp:116-169) without the
  // m x n plan: the all-zero block fraction exactly, residuals / mass from
  // device row and column sums
  PlanDiagnostics plan_diagnostics(const DualState& s) {
    pack(s);
    gsot_plan_diag d;
    check(gsot_plan_diagnostics(ctx_, x_.data(), &d));
    PlanDiagnostics r;
    r.marginal_res_a = d.marginal_res_a;
    r.marginal_res_b = d.marginal_res_b;
    r.group_sparsity = d.group_sparsity;
    r.mass = d.mass;
    return r;
  }
  // build_active_set(take_snapshot(s, inst), s, p, groups).count
  // (screening.hpp:24-50, :147-166): the active set at the snapshot point
  long long active_set_size(const DualState& s) {
    pack(s);
    check(gsot_init_snapshot(ctx_, x_.data()));
    check(gsot_refresh(ctx_, x_.data(), 1));
    int64_t count = 0;
    check(gsot_active_set(ctx_, nullptr, &count));
    return static_cast<long long>(count);
  }
  // new RegParams on the resident instance (no re-upload, no re-validation of C)
  void set_params(const RegParams& p) { check(gsot_set_params(ctx_, p.gamma(), p.mu())); }

  // The screened plug-in level (FastGradDispatcher, screening.hpp:206-315, as
  // run_screened wires it, solver.hpp:133-250): init the snapshot at x0, then
  // ObjectiveFn / GradientFn that evaluate with block skipping (and the active
  // set), and the ChunkHook that refreshes. The reference's own maximize
  // driven by these is solve_fast; `stats` collects GradStats (per call
  // history included). exact: reference-order sums (GSOT_EVAL_EXACT).
  struct Screened {
    ObjectiveFn objective;
    GradientFn gradient;
    ChunkHook hook;
    std::shared_ptr<GradStats> stats;
  };
  Screened screened_callbacks(const Eigen::VectorXd& x0, bool use_active_set, bool exact = false) {
    check(gsot_init_snapshot(ctx_, x0.data()));
    auto st = std::make_shared<GradStats>();
    const int mode = GSOT_EVAL_SCREENED | (exact ? GSOT_EVAL_EXACT : 0);
    auto eval = [this, st, mode](const Eigen::VectorXd& x) {
      const size_t dim = static_cast<size_t>(m_ + n_);
      if (have_scache_ && scache_x_.size() == dim &&
          std::memcmp(scache_x_.data(), x.data(), sizeof(double) * dim) == 0)
        return;
      scache_x_.assign(x.data(), x.data() + dim);
      sg_.resize(dim);
      gsot_call_stats cs;
      check(gsot_eval(ctx_, scache_x_.data(), mode, &scache_obj_, sg_.data(), &cs));
      have_scache_ = true;
      st->blocks_in_active_set += cs.in_active;  // screening.hpp:280-287
      st->blocks_skipped += cs.skipped;
      st->blocks_unskipped += cs.unskipped;
      st->upper_bounds_evaluated += cs.upper_bounds;
      ++st->grad_calls;
      st->history.push_back({cs.in_active, cs.skipped, cs.unskipped, cs.upper_bounds});
    };
    Screened r;
    r.stats = st;
    r.objective = [eval, this](const Eigen::VectorXd& x) {
      eval(x);
      return scache_obj_;
    };
    r.gradient = [eval, this](const Eigen::VectorXd& x, Eigen::VectorXd& out) {
      eval(x);
      out.resize(m_ + n_);
      std::memcpy(out.data(), sg_.data(), sizeof(double) * static_cast<size_t>(m_ + n_));
    };
    r.hook = [this, st, use_active_set](int, const Eigen::VectorXd& x) {
      check(gsot_refresh(ctx_, x.data(), use_active_set ? 1 : 0));  // screening.hpp:231-235
      ++st->outer_loops;
      have_scache_ = false;  // a new snapshot: the next call screens afresh
    };
    return r;
  }

  // ObjectiveFn / GradientFn for the reference's maximize (lbfgs.hpp:32-33):
  // one fused device evaluation serves both calls at the same x.
  std::pair<ObjectiveFn, GradientFn> callbacks() {
    ObjectiveFn f = [this](const Eigen::VectorXd& x) {
      eval_cached(x);
      return cache_obj_;
    };
    GradientFn g = [this](const Eigen::VectorXd& x, Eigen::VectorXd& out) {
      eval_cached(x);
      out.resize(m_ + n_);
      std::memcpy(out.data(), g_.data(), sizeof(double) * static_cast<size_t>(m_ + n_));
    };
    return {f, g};
  }

 private:
  void pack(const DualState& s) {
    if (s.alpha.size() != m_ || s.beta.size() != n_)
      throw DimensionMismatch("dual state does not match the instance");
    x_.resize(static_cast<size_t>(m_ + n_));
    std::memcpy(x_.data(), s.alpha.data(), sizeof(double) * static_cast<size_t>(m_));
    std::memcpy(x_.data() + m_, s.beta.data(), sizeof(double) * static_cast<size_t>(n_));
  }
  void eval_cached(const Eigen::VectorXd& x) {
    const size_t dim = static_cast<size_t>(m_ + n_);
    if (have_cache_ && cache_x_.size() == dim &&
        std::memcmp(cache_x_.data(), x.data(), sizeof(double) * dim) == 0)
      return;
    cache_x_.assign(x.data(), x.data() + dim);
    g_.resize(dim);
    check(gsot_eval(ctx_, cache_x_.data(), GSOT_EVAL_DENSE, &cache_obj_, g_.data(), nullptr));
    have_cache_ = true;
  }

  gsot_ctx* ctx_ = nullptr;
  Eigen::Index m_, n_;
  std::vector<double> x_, g_, cache_x_;
  double cache_obj_ = 0.0;
  bool have_cache_ = false;
  std::vector<double> sg_, scache_x_;  // screened callbacks' evaluation cache
  double scache_obj_ = 0.0;
  bool have_scache_ = false;
};

// Exact-order solves (bitwise the reference's trajectory; verification mode).
inline bool& exact_order() {
  static bool on = false;
  return on;
}

namespace detail {

inline int mode_code(SolverMode mode) {
  switch (mode) {
    case SolverMode::baseline: return GSOT_MODE_BASELINE;
    case SolverMode::fast: return GSOT_MODE_FAST;
    case SolverMode::fast_no_lower_bound: return GSOT_MODE_FAST_NO_LOWER_BOUND;
    case SolverMode::audit: return GSOT_MODE_AUDIT;
  }
  throw Error("unknown solver mode");
}

// One solve on a resident instance (solver.hpp:92-293 through gsot_solve);
// with_plan: recover the m x n plan into Solution::plan (finish_solution).
inline Solution run_on(Device& dev, const SolverOptions& opts,
                       int mode, double ub_offset, AuditReport* report, bool with_plan) {
  gsot_solver_options o;
  gsot_default_solver_options(&o);
  o.snapshot_interval = opts.snapshot_interval;
  o.grad_tol = opts.grad_tol;
  o.max_outer_loops = opts.max_outer_loops;
  o.lbfgs_memory = opts.lbfgs_memory;
  o.mode = mode;
  o.upper_bound_offset = ub_offset;
  o.flags = (exact_order() ? GSOT_SOLVE_EXACT : 0) |
            (mode == GSOT_MODE_AUDIT && opts.mode == SolverMode::fast_no_lower_bound
                 ? GSOT_SOLVE_NO_ACTIVE_SET
                 : 0);
  const Eigen::Index m = dev.m(), n = dev.n();
  std::vector<double> x(static_cast<size_t>(m + n));
  // worst case per accepted iteration: two attempts of max_bracket (40) +
  // max_zoom (12) evaluations (lbfgs.hpp:11-30), plus the initial call
  const int64_t cap =
      static_cast<int64_t>(opts.snapshot_interval) * opts.max_outer_loops * 2 * (40 + 12) + 16;
  std::vector<int64_t> hist(static_cast<size_t>(cap) * 4);
  gsot_solve_result r;
  check(gsot_solve(dev.handle(), &o, x.data(), &r, hist.data(), cap));
  Solution sol;  // solver.hpp:33-42, finish_solution (:72-87)
  sol.state.alpha.resize(m);
  sol.state.beta.resize(n);
  std::memcpy(sol.state.alpha.data(), x.data(), sizeof(double) * static_cast<size_t>(m));
  std::memcpy(sol.state.beta.data(), x.data() + m, sizeof(double) * static_cast<size_t>(n));
  sol.objective = r.objective;
  if (with_plan) sol.plan = dev.plan(sol.state);
  sol.stats.blocks_in_active_set = r.blocks_in_active_set;
  sol.stats.blocks_skipped = r.blocks_skipped;
  sol.stats.blocks_unskipped = r.blocks_unskipped;
  sol.stats.upper_bounds_evaluated = r.upper_bounds_evaluated;
  sol.stats.outer_loops = r.outer_loops;
  sol.stats.grad_calls = r.grad_calls;
  const int64_t rows = std::min<int64_t>(r.grad_calls, cap);
  for (int64_t i = 0; i < rows; ++i)
    sol.stats.history.push_back({hist[i * 4], hist[i * 4 + 1], hist[i * 4 + 2], hist[i * 4 + 3]});
  sol.iterations = r.iterations;
  sol.wall_time = std::chrono::nanoseconds(static_cast<int64_t>(r.wall_seconds * 1e9));
  sol.converged = r.converged != 0;
  sol.line_search_failed = r.line_search_failed != 0;
  if (report) {
    report->skip_checks = r.audit_skip_checks;
    report->active_checks = r.audit_active_checks;
    report->column_compares = r.audit_column_compares;
    report->gradient_calls = r.audit_gradient_calls;
  }
  return sol;
}

inline Solution run(const ProblemInstance& inst, const RegParams& p, const SolverOptions& opts,
                    int mode, double ub_offset, AuditReport* report) {
  Device dev(inst, p);
  return run_on(dev, opts, mode, ub_offset, report, true);
}

}  // namespace detail

// solver.hpp:92-127
inline Solution solve_baseline(const ProblemInstance& inst, const RegParams& p,
                               const SolverOptions& opts = {}) {
  return detail::run(inst, p, opts, GSOT_MODE_BASELINE, 0.0, nullptr);
}
// solver.hpp:254-258
inline Solution solve_fast(const ProblemInstance& inst, const RegParams& p,
                           const SolverOptions& opts = {}) {
  const int mode = opts.mode == SolverMode::fast_no_lower_bound ? GSOT_MODE_FAST_NO_LOWER_BOUND
                                                                : GSOT_MODE_FAST;
  return detail::run(inst, p, opts, mode, 0.0, nullptr);
}
// solver.hpp:268-281
inline std::pair<Solution, AuditReport> audit_solve(const ProblemInstance& inst,
                                                    const RegParams& p,
                                                    const SolverOptions& opts = {},
                                                    double upper_bound_offset = 0.0) {
  AuditReport report;
  if (opts.mode == SolverMode::baseline) return {b200::solve_baseline(inst, p, opts), report};
  Solution sol = detail::run(inst, p, opts, GSOT_MODE_AUDIT, upper_bound_offset, &report);
  return {std::move(sol), report};
}
// solver.hpp:284-293
inline Solution solve(const ProblemInstance& inst, const RegParams& p,
                      const SolverOptions& opts = {}) {
  switch (opts.mode) {
    case SolverMode::baseline: return b200::solve_baseline(inst, p, opts);
    case SolverMode::fast:
    case SolverMode::fast_no_lower_bound: return b200::solve_fast(inst, p, opts);
    case SolverMode::audit: return b200::audit_solve(inst, p, opts).first;
  }
  throw Error("unknown solver mode");
}

// solve (solver.hpp:284-293) on a resident device instance (e.g. built from
// CSV samples with the Device(LabeledSamples, UnlabeledSamples, ...)
// constructor): baseline, fast and fast_no_lower_bound; with_plan recovers
// the m x n plan on the host.
inline Solution solve(Device& dev, const SolverOptions& opts = {}, bool with_plan = false) {
  int mode = GSOT_MODE_FAST;
  switch (opts.mode) {
    case SolverMode::baseline: mode = GSOT_MODE_BASELINE; break;
    case SolverMode::fast: mode = GSOT_MODE_FAST; break;
    case SolverMode::fast_no_lower_bound: mode = GSOT_MODE_FAST_NO_LOWER_BOUND; break;
    case SolverMode::audit: mode = GSOT_MODE_AUDIT; break;
  }
  return detail::run_on(dev, opts, mode, 0.0, nullptr, with_plan);
}

// run_grid (bench.hpp:137-180): the (gamma, rho, mode) grid in the reference's
// deterministic order, on ONE device context: the cost is uploaded and
// validated once, each (gamma, rho) only swaps the parameters. Records carry
// the reference's fields (make_record, bench.hpp:99-126) with the plan
// diagnostics computed on the device; active_set_size_final is the fresh
// active-set build at the solution for non-baseline modes (bench.hpp:168-175).
// The sink receives each Solution without its m x n plan unless with_plans.
#if GSOT_B200_HAVE_BENCH
inline std::vector<BenchRecord> run_grid(
    const ProblemInstance& inst, const GridSpec& grid, int num_classes, int per_class,
    const std::function<void(const BenchRecord&, const Solution&)>& sink = nullptr,
    bool with_plans = false) {
  std::vector<BenchRecord> rows;
  std::unique_ptr<Device> dev;
  for (const double gamma : grid.gammas) {
    for (const double rho : grid.rhos) {
      const RegParams p = params_from_rho(gamma, rho);  // core.hpp:148-151 (throws alike)
      if (!dev)
        dev = std::make_unique<Device>(inst, p);
      else
        dev->set_params(p);
      for (const SolverMode mode : grid.modes) {
        SolverOptions opts = grid.base;
        opts.mode = mode;
        Solution sol = detail::run_on(*dev, opts, detail::mode_code(mode), 0.0, nullptr,
                                      with_plans);
        BenchRecord r;
        r.mode = to_string(mode);
        r.num_classes = num_classes;
        r.per_class = per_class;
        r.m = static_cast<long>(inst.m());
        r.n = static_cast<long>(inst.n());
        r.gamma = gamma;
        r.rho = rho;
        r.iterations = sol.iterations;
        r.outer_loops = static_cast<long>(sol.stats.outer_loops);
        r.wall_ms = std::chrono::duration<double, std::milli>(sol.wall_time).count();
        r.objective = sol.objective;
        r.blocks_computed = sol.stats.blocks_in_active_set + sol.stats.blocks_unskipped;
        r.blocks_skipped = sol.stats.blocks_skipped;
        r.upper_bounds_evaluated = sol.stats.upper_bounds_evaluated;
        const PlanDiagnostics diag = dev->plan_diagnostics(sol.state);
        r.group_sparsity = diag.group_sparsity;
        r.marginal_res_a = diag.marginal_res_a;
        r.marginal_res_b = diag.marginal_res_b;
        r.converged = sol.converged;
        if (mode != SolverMode::baseline) r.active_set_size_final = dev->active_set_size(sol.state);
        if (sink) sink(r, sol);
        rows.push_back(std::move(r));
      }
    }
  }
  return rows;
}
#endif

}  // namespace b200
}  // namespace groupot
