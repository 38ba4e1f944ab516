// dropin_check.cpp — TEST INFRASTRUCTURE: the reference C++ API, unchanged,
// next to the drop-in groupot::b200 adapter (include/groupot_b200.hpp) on
// the same ProblemInstance. Built by oracle/Makefile into oracle/_ref/ (it
// needs the reference headers, present in the build container only) and run
// on the GPU box by tests/test_gpu_dropin.py. Prints one JSON object.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>

#include "groupot/bench.hpp"
#include "groupot/data_io.hpp"
#include "groupot/solver.hpp"
#include "groupot_b200.hpp"

using namespace groupot;

static double max_abs_diff(const Eigen::MatrixXd& a, const Eigen::MatrixXd& b) {
  double m = 0.0;
  for (Eigen::Index j = 0; j < a.cols(); ++j)
    for (Eigen::Index i = 0; i < a.rows(); ++i) m = std::max(m, std::abs(a(i, j) - b(i, j)));
  return m;
}

int main() {
  // the reference's own generator and instance builder (data_io.hpp:67-98, :157-181)
  auto [src, tgt] = gen_synthetic(4, 25, 7);
  ProblemInstance inst = make_instance(src, tgt, true);
  const RegParams p(1.0, 0.1);
  std::printf("{");
  // evaluation through the adapter vs the reference
  DualState s{Eigen::VectorXd::Constant(inst.m(), 0.02), Eigen::VectorXd::Constant(inst.n(), 0.01)};
  b200::Device dev(inst, p);
  const double obj_ref = dual_objective(s, inst, p);
  const double obj_dev = dev.objective(s);
  Eigen::VectorXd ga, gb, ga2, gb2;
  dual_gradient(s, inst, p, ga, gb);
  dev.gradient(s, ga2, gb2);
  double gerr = 0.0;
  for (Eigen::Index i = 0; i < ga.size(); ++i) gerr = std::max(gerr, std::abs(ga[i] - ga2[i]));
  for (Eigen::Index j = 0; j < gb.size(); ++j) gerr = std::max(gerr, std::abs(gb[j] - gb2[j]));
  const double plan_err = max_abs_diff(recover_plan(s, inst, p).plan, dev.plan(s).plan);
  std::printf("\"obj_rel\": %.3e, \"grad_abs\": %.3e, \"plan_eval_abs\": %.3e",
              std::abs(obj_dev - obj_ref) / std::abs(obj_ref), gerr, plan_err);
  // the reference's own maximize() driving device evaluations
  {
    auto [f, g] = dev.callbacks();
    MaximizeOptions mo;
    mo.max_chunks = 3;
    mo.grad_tol = 1e-12;
    const MaximizeResult rd = maximize(f, g, Eigen::VectorXd::Zero(inst.m() + inst.n()), mo);
    SolverOptions so;
    so.max_outer_loops = 3;
    so.grad_tol = 1e-12;
    so.mode = SolverMode::baseline;
    const Solution rr = groupot::solve(inst, p, so);
    double xd = 0.0;
    for (Eigen::Index i = 0; i < inst.m(); ++i) xd = std::max(xd, std::abs(rd.x[i] - rr.state.alpha[i]));
    std::printf(", \"maximize_iters\": [%d, %d], \"maximize_x_abs\": %.3e", rd.iterations,
                rr.iterations, xd);
  }
  // solve() in every mode: reference vs drop-in
  const SolverMode modes[] = {SolverMode::baseline, SolverMode::fast,
                              SolverMode::fast_no_lower_bound, SolverMode::audit};
  for (SolverMode mode : modes) {
    SolverOptions o;
    o.mode = mode;
    o.max_outer_loops = 30;
    const Solution r = groupot::solve(inst, p, o);
    const Solution d = b200::solve(inst, p, o);
    std::printf(", \"%s\": {\"iters\": [%d, %d], \"converged\": [%d, %d], \"obj_rel\": %.3e, "
                "\"plan_abs\": %.3e, \"grad_calls\": [%ld, %ld]}",
                to_string(mode), r.iterations, d.iterations, (int)r.converged, (int)d.converged,
                std::abs(d.objective - r.objective) / std::abs(r.objective),
                max_abs_diff(r.plan.plan, d.plan.plan), (long)r.stats.grad_calls,
                (long)d.stats.grad_calls);
  }
  // the reference's own maximize driving the device's screened callbacks
  // (FastGradDispatcher level) == the reference's solve_fast, exact order
  {
    SolverOptions so;
    so.max_outer_loops = 5;
    so.grad_tol = 1e-12;
    const Solution rf = groupot::solve_fast(inst, p, so);
    auto cb = dev.screened_callbacks(Eigen::VectorXd::Zero(inst.m() + inst.n()), true, true);
    const MaximizeResult rd = maximize(cb.objective, cb.gradient,
                                       Eigen::VectorXd::Zero(inst.m() + inst.n()),
                                       detail::to_lbfgs_options(so), cb.hook);
    bool hist = rf.stats.history.size() == cb.stats->history.size();
    for (size_t i = 0; hist && i < rf.stats.history.size(); ++i) {
      const auto &a = rf.stats.history[i], &b = cb.stats->history[i];
      hist = a.in_active == b.in_active && a.skipped == b.skipped && a.unskipped == b.unskipped &&
             a.upper_bounds == b.upper_bounds;
    }
    double xd = 0.0;
    for (Eigen::Index i = 0; i < inst.m(); ++i) xd = std::max(xd, std::abs(rd.x[i] - rf.state.alpha[i]));
    std::printf(", \"screened_maximize\": {\"iters\": [%d, %d], \"history_equal\": %d, "
                "\"x_abs\": %.3e, \"skipped\": %lld}",
                rf.iterations, rd.iterations, (int)hist, xd, (long long)cb.stats->blocks_skipped);
  }
  // audit_solve of a fast_no_lower_bound SolverOptions (solver.hpp:271): no active set
  {
    SolverOptions o;
    o.mode = SolverMode::fast_no_lower_bound;
    o.max_outer_loops = 10;
    const auto [r, rr] = groupot::audit_solve(inst, p, o);
    b200::exact_order() = true;
    const auto [d, dr] = b200::audit_solve(inst, p, o);
    b200::exact_order() = false;
    std::printf(", \"audit_nolb\": {\"iters\": [%d, %d], \"grad_calls\": [%ld, %ld], "
                "\"in_active\": [%lld, %lld], \"active_checks\": [%ld, %ld], \"obj_equal\": %d}",
                r.iterations, d.iterations, (long)r.stats.grad_calls, (long)d.stats.grad_calls,
                (long long)r.stats.blocks_in_active_set, (long long)d.stats.blocks_in_active_set,
                (long)rr.active_checks, (long)dr.active_checks, (int)(r.objective == d.objective));
  }
  // run_grid (bench.hpp:137-180): the reference's grid driver vs the drop-in
  // one on a warm device context, exact-order solves (bitwise trajectories):
  // every integer field, the objective, the sparsity and the final active
  // set equal; the residuals within 1e-12
  {
    GridSpec grid;
    grid.gammas = {1.0, 0.1};
    grid.rhos = {0.2, 0.8};
    grid.modes = {SolverMode::baseline, SolverMode::fast, SolverMode::fast_no_lower_bound};
    grid.base.max_outer_loops = 4;
    grid.base.grad_tol = 1e-12;
    int sink_calls = 0;
    const auto ref_rows = groupot::run_grid(inst, grid, 4, 25);
    b200::exact_order() = true;
    const auto dev_rows = b200::run_grid(
        inst, grid, 4, 25,
        [&](const BenchRecord&, const Solution& sol) { sink_calls += sol.stats.grad_calls > 0; });
    b200::exact_order() = false;
    int ints_equal = ref_rows.size() == dev_rows.size(), obj_equal = 1, sparsity_equal = 1;
    int csv_fields = 1;
    double res_abs = 0.0;
    for (size_t i = 0; i < std::min(ref_rows.size(), dev_rows.size()); ++i) {
      const BenchRecord &r = ref_rows[i], &d = dev_rows[i];
      ints_equal &= r.mode == d.mode && r.m == d.m && r.n == d.n && r.gamma == d.gamma &&
                    r.rho == d.rho && r.iterations == d.iterations &&
                    r.outer_loops == d.outer_loops && r.blocks_computed == d.blocks_computed &&
                    r.blocks_skipped == d.blocks_skipped &&
                    r.upper_bounds_evaluated == d.upper_bounds_evaluated &&
                    r.active_set_size_final == d.active_set_size_final &&
                    r.converged == d.converged;
      obj_equal &= r.objective == d.objective;
      sparsity_equal &= r.group_sparsity == d.group_sparsity;
      res_abs = std::max(res_abs, std::max(std::abs(r.marginal_res_a - d.marginal_res_a),
                                           std::abs(r.marginal_res_b - d.marginal_res_b)));
      // the record's CSV row has the schema's 19 fields (bench.hpp:37-68). (The
      // reference's parse_csv_row reads toks[i] and i++ in one call's arguments,
      // bench.hpp:76, an unspecified order that GCC resolves past the last field:
      // it is not used here.)
      const std::string row = to_csv_row(d);
      csv_fields &= std::count(row.begin(), row.end(), ',') == 18 &&
                    row.compare(0, d.mode.size(), d.mode) == 0;
    }
    std::printf(", \"grid\": {\"rows\": [%zu, %zu], \"ints_equal\": %d, \"obj_equal\": %d, "
                "\"sparsity_equal\": %d, \"res_abs\": %.3e, \"sink_calls\": %d, "
                "\"csv_roundtrip\": %d}",
                ref_rows.size(), dev_rows.size(), ints_equal, obj_equal, sparsity_equal, res_abs,
                sink_calls, csv_fields);
  }
  // CSV ingestion (data_io.hpp:270-352) -> make_instance on the device: the
  // reference writes and reads the files, the adapter builds the instance
  // from the samples on the GPU (the cost never on the host); exact-order
  // solves of both are bitwise equal
  {
    const std::string sp = "/tmp/gsot_dropin_src.csv", tp = "/tmp/gsot_dropin_tgt.csv";
    save_source_csv(src, sp);
    save_target_csv(tgt, tp);
    auto [s2, t2] = load_csv(sp, tp);
    const ProblemInstance ri = make_instance(s2, t2, true);
    b200::Device fdev(s2, t2, true, false, p);
    SolverOptions so;
    so.mode = SolverMode::fast;
    so.max_outer_loops = 6;
    so.grad_tol = 1e-12;
    const Solution r = groupot::solve(ri, p, so);
    b200::exact_order() = true;
    const Solution d = b200::solve(fdev, so, true);
    b200::exact_order() = false;
    int x_equal = r.state.alpha.size() == d.state.alpha.size();
    for (Eigen::Index i = 0; x_equal && i < r.state.alpha.size(); ++i)
      x_equal = r.state.alpha[i] == d.state.alpha[i];
    for (Eigen::Index j = 0; x_equal && j < r.state.beta.size(); ++j)
      x_equal = r.state.beta[j] == d.state.beta[j];
    std::printf(", \"csv_device\": {\"iters\": [%d, %d], \"x_equal\": %d, \"obj_equal\": %d, "
                "\"plan_abs\": %.3e}",
                r.iterations, d.iterations, x_equal, (int)(r.objective == d.objective),
                max_abs_diff(r.plan.plan, d.plan.plan));
  }
  // error behaviour: the same exception type and fields
  {
    ProblemInstance bad = inst;
    bad.cost(3, 2) = -1.0;
    int ok = 0;
    try {
      b200::solve(bad, p);
    } catch (const NegativeCost& e) {
      ok = e.row == 3 && e.col == 2 && e.value == -1.0;
    }
    ProblemInstance bad2 = inst;
    bad2.a[0] = -0.5;
    int ok2 = 0;
    try {
      b200::solve(bad2, p);
    } catch (const MarginalNotNormalized& e) {
      ok2 = e.which == 'a' && e.index == 0;
    }
    int ok3 = 0;
    try {
      SolverOptions o;
      o.mode = SolverMode::audit;
      b200::audit_solve(inst, p, o, -1e3);
    } catch (const AuditViolation&) {
      ok3 = 1;
    }
    std::printf(", \"negative_cost_fields\": %d, \"marginal_fields\": %d, \"audit_violation\": %d",
                ok, ok2, ok3);
  }
  std::printf("}\n");
  return 0;
}
