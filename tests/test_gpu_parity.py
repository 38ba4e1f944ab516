"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden fixtures.

Tolerances (BASELINE.json north_star):
* per-block values -- plan entries (gsot_plan_columns), snapshot norms
  z~/k~/o~, the screening decisions and counters, the active set -- BITWISE
  (those kernels compute each block in the reference's order of operations;
  the fused evaluation re-associates its per-column norms, fast mode);
* objective within 1e-9 relative;
* gradient within 1e-9 scale-aware: |g - g_ref| <= 1e-9 * (a_i + sum_j T_ij)
  for grad_alpha and 1e-9 * (b_j + sum_i T_ij) for grad_beta (the sums cancel
  near the optimum);
* final plan within 1e-6 after the solve.
"""
import os

import numpy as np
import pytest

import paper_2303_07597_b200 as G
from oracle_bindings import Oracle, Problem

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
OBJ_RTOL = 1e-9
GRAD_STOL = 1e-9
PLAN_ATOL = 1e-6
SOLVE_OBJ_RTOL = 1e-6


@pytest.fixture(scope="module")
def o():
    return Oracle()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def ctx_of(p: Problem) -> G.Context:
    return G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)


def grad_scale(o, p, x):
    plan = o.plan(p, x[: p.m], x[p.m:])
    return np.concatenate([p.a + plan.sum(axis=1), p.b + plan.sum(axis=0)])


def assert_eval_close(o, p, x, obj, g, obj_ref=None, g_ref=None):
    if obj_ref is None:
        obj_ref = o.objective(p, x[: p.m], x[p.m:])
    if g_ref is None:
        ga, gb = o.gradient(p, x[: p.m], x[p.m:])
        g_ref = np.concatenate([ga, gb])
    assert abs(obj - obj_ref) <= OBJ_RTOL * max(abs(obj_ref), 1e-300), (obj, obj_ref)
    scale = grad_scale(o, p, x)
    err = np.abs(g - g_ref)
    assert np.all(err <= GRAD_STOL * scale), float(np.max(err / scale))


def gold_problem(g, name, pi):
    gamma, mu = g[f"{name}/p{pi}/params"]
    return Problem(g[f"{name}/cost"], g[f"{name}/sizes"], g[f"{name}/a"], g[f"{name}/b"],
                   float(gamma), float(mu))


# ------------------------------------------------------------ golden fixtures


@pytest.mark.parametrize("name", ["synth", "ragged"])
@pytest.mark.parametrize("pi", [0, 1, 2])
def test_golden_eval_plan_snapshot_active(o, gold, name, pi):
    p = gold_problem(gold, name, pi)
    key = f"{name}/p{pi}"
    ctx = ctx_of(p)
    for si in range(3):
        x = gold[f"{key}/s{si}/x"]
        obj, g, st = ctx.eval(x)
        assert_eval_close(o, p, x, obj, g, gold[f"{key}/s{si}/objective"][0],
                          gold[f"{key}/s{si}/grad"])
        assert (st.in_active, st.skipped, st.unskipped, st.upper_bounds) == (0, 0, p.L * p.n, 0)
    x2 = gold[f"{key}/s2/x"]
    assert np.array_equal(ctx.plan_columns(x2, 0, p.n), gold[f"{key}/plan"])
    x0, x1 = gold[f"{key}/s0/x"], gold[f"{key}/s1/x"]
    ctx.init_snapshot(x1)
    z, k, oo = ctx.snapshot_norms()
    assert np.array_equal(z, gold[f"{key}/snap_z"])
    assert np.array_equal(k, gold[f"{key}/snap_k"])
    assert np.array_equal(oo, gold[f"{key}/snap_o"])
    for ua in (0, 1):
        ctx.init_snapshot(x0)
        ctx.refresh(x1, bool(ua))
        mem, cnt = ctx.active_set()
        if ua:
            assert np.array_equal(mem, gold[f"{key}/fast1/member"].astype(bool))
            assert cnt == int(gold[f"{key}/fast1/member"].sum())
        else:
            assert cnt == 0 and not mem.any()
        x = gold[f"{key}/fast{ua}/x"]
        obj_s, g_s, st = ctx.eval(x, screened=True)
        assert [st.in_active, st.skipped, st.unskipped, st.upper_bounds] == \
            gold[f"{key}/fast{ua}/counters"].tolist()
        assert_eval_close(o, p, x, obj_s, g_s, None, gold[f"{key}/fast{ua}/grad"])
        obj_d, g_d, _ = ctx.eval(x)
        assert obj_d == obj_s and np.array_equal(g_d, g_s)  # screen changes no bit
    ctx.close()


@pytest.mark.parametrize("name", ["synth", "ragged"])
@pytest.mark.parametrize("pi", [0, 1, 2])
def test_golden_plan_diagnostics(gold, name, pi):
    """gsot_plan_diagnostics against the reference's plan_diagnostics of its own
    recovered plans (dual.hpp:139-169): the all-zero block fraction exactly;
    residuals and mass within 1e-12 relative (device sums in a fixed order,
    the reference's in Eigen's)."""
    p = gold_problem(gold, name, pi)
    key = f"{name}/p{pi}"
    ctx = ctx_of(p)
    for x, ref in ((gold[f"{key}/s2/x"], gold[f"{key}/plan_diag"]),
                   (gold[f"{key}/solve1/x"], gold[f"{key}/solve_plan_diag"])):
        d = ctx.plan_diagnostics(x)
        assert d.group_sparsity == ref[2]
        for got, want in ((d.marginal_res_a, ref[0]), (d.marginal_res_b, ref[1]), (d.mass, ref[3])):
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (got, want)
    ctx.close()


@pytest.mark.parametrize("name", ["synth", "ragged"])
def test_primal_objective_and_duality_gap(o, gold, name):
    """gsot_primal_objective against primal_objective of the oracle's plan
    (core.hpp:167-180; the mirror's numpy restatement is pinned to the
    reference on CPU), within 1e-12 relative; and the Fenchel-Young identity
    for the plan T = grad psi(f): primal(T) - dual(x) = -x . grad dual(x)."""
    p = gold_problem(gold, name, 1)
    inst = G.ProblemInstance(p.cost, p.a, p.b, G.GroupPartition(p.sizes))
    prm = G.RegParams(p.gamma, p.mu)
    ctx = ctx_of(p)
    for x in (gold[f"{name}/p1/s2/x"], gold[f"{name}/p1/solve1/x"]):
        got = ctx.primal_objective(x)
        want = G.primal_objective(G.TransportPlan(o.plan(p, x[: p.m], x[p.m:])), inst, prm)
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (got, want)
        obj, g, _ = ctx.eval(x)
        gap, fy = got - obj, -float(x @ g)
        assert abs(gap - fy) <= 1e-10 * max(1.0, abs(got), float(np.abs(x).max())), (gap, fy)
    ctx.close()


def test_plan_diagnostics_zero_plan():
    # test_dual.cpp:209-217 on the device: C = 0, x = 0 -> every block z = 0 <= tau
    q = Problem(np.zeros((4, 2)), np.array([2, 2], np.int32), np.full(4, .25), np.full(2, .5),
                1.0, 1.0)
    d = ctx_of(q).plan_diagnostics(np.zeros(6))
    assert (d.marginal_res_a, d.marginal_res_b, d.group_sparsity, d.mass) == (0.25, 0.5, 1.0, 0.0)


def test_golden_hand_examples(gold):
    h = Problem(np.zeros((1, 1)), np.array([1], np.int32), np.ones(1), np.ones(1), 1.0, 0.5)
    ctx = ctx_of(h)
    obj, g, _ = ctx.eval(np.array([1.0, 0.0]))
    assert abs(obj - 0.875) <= 1e-15 and abs(obj - gold["hand/1x1/objective"][0]) <= 1e-15
    assert np.allclose(g, gold["hand/1x1/grad"], atol=1e-15, rtol=0)
    h2 = Problem(np.zeros((2, 1)), np.array([2], np.int32), np.full(2, .5), np.ones(1), 1.0, 1.0)
    pl = ctx_of(h2).plan_columns(np.array([3.0, 4.0, 0.0]), 0, 1)
    assert np.array_equal(pl, gold["hand/plan34"])
    # test_dual.cpp:73-81: C = 1e6 thresholds everything: grad == (a, b) bitwise
    q = Problem(np.full((4, 3), 1e6), np.array([2, 2], np.int32), np.full(4, .25),
                np.full(3, 1 / 3), 1.0, 1.0)
    obj, g, _ = ctx_of(q).eval(np.zeros(7))
    assert np.array_equal(g, np.concatenate([q.a, q.b])) and obj == 0.0


@pytest.mark.parametrize("name", ["synth", "ragged"])
@pytest.mark.parametrize("pi", [0, 1, 2])
def test_golden_solve(o, gold, name, pi):
    """Full solves against the reference's golden results.

    The device re-associates the cross-block sums, so its
    trajectory equals the reference's to ~1e-14 for the first iterations and
    the rounding difference then grows along unconverged trajectories (see
    test_solve_short_horizon_matches_oracle). Criteria: when the reference
    converged (|g|_inf <= tol) the device converges too and the plans agree
    within 1e-6; the final objective agrees within 1e-6 relative always."""
    p = gold_problem(gold, name, pi)
    key = f"{name}/p{pi}"
    ctx = ctx_of(p)
    ref_plan = gold[f"{key}/solve_plan"]
    for mode in (0, 1, 2, 3):
        r = ctx.solve(mode=mode, max_outer_loops=20, grad_tol=1e-7, history_cap=100000)
        ints = gold[f"{key}/solve{mode}/ints"]
        obj_ref = gold[f"{key}/solve{mode}/objective"][0]
        assert abs(r["objective"] - obj_ref) <= SOLVE_OBJ_RTOL * abs(obj_ref)
        assert not r["line_search_failed"]
        if ints[1]:  # the reference converged
            assert r["converged"]
            plan = ctx.plan_columns(r["x"], 0, p.n)
            assert np.max(np.abs(plan - ref_plan)) <= PLAN_ATOL
        # counter identity of GradStats (screening.hpp:168-172)
        h = r["history"]
        assert np.all(h[:, 0] + h[:, 1] + h[:, 2] == p.L * p.n)
        if mode != 0:  # the baseline books every block unskipped, no bounds
            assert np.all(h[:, 3] == h[:, 1] + h[:, 2])
    ctx.close()


@pytest.mark.parametrize("name", ["synth", "ragged"])
@pytest.mark.parametrize("pi", [0, 1, 2])
def test_solve_short_horizon_matches_oracle(o, gold, name, pi):
    """Same number of L-BFGS iterations (2 chunks = 20): iterates, plans,
    objective and the per-call screening counters match the oracle. (Longer
    horizons: the exact-order mode is bitwise, tests/test_gpu_exact.py.)"""
    p = gold_problem(gold, name, pi)
    ctx = ctx_of(p)
    for mode in (0, 1, 2):
        r = ctx.solve(mode=mode, max_outer_loops=2, grad_tol=1e-12, history_cap=10000)
        ro = o.solve(p, mode=mode, max_outer_loops=2, grad_tol=1e-12)
        assert r["iterations"] == ro["iterations"]
        assert r["grad_calls"] == ro["grad_calls"]
        assert np.array_equal(r["history"], ro["history"])
        scale = np.max(np.abs(ro["x"]))
        assert np.max(np.abs(r["x"] - ro["x"])) <= 1e-6 * scale
        assert abs(r["objective"] - ro["objective"]) <= OBJ_RTOL * abs(ro["objective"])
        plan = ctx.plan_columns(r["x"], 0, p.n)
        plan_o = o.plan(p, ro["x"][: p.m], ro["x"][p.m:])
        assert np.max(np.abs(plan - plan_o)) <= PLAN_ATOL
    ctx.close()


# ------------------------------------------------------------ random structures

STRUCTURES = {
    "one_group": ([57], 40),
    "singletons": ([1] * 23, 37),
    "large_groups": ([300, 5, 41], 70),
    "odd_ragged": ([3, 33, 1, 7, 64, 65, 2], 97),
    "n_one": ([4, 5], 1),
    "n_33": ([9, 9, 9], 33),
    "tall_groups": ([1000, 130, 129, 40, 7], 75),
}


def random_problem(sizes, n, gamma, mu, seed, weighted=False):
    rng = np.random.default_rng(seed)
    sizes = np.array(sizes, np.int32)
    m = int(sizes.sum())
    cost = rng.uniform(0, 2, (m, n))
    a = rng.uniform(0.5, 1.5, m) if weighted else np.ones(m)
    a = a / a.sum()
    return Problem(cost, sizes, a, np.full(n, 1 / n), gamma, mu), rng


@pytest.mark.parametrize("struct", sorted(STRUCTURES))
@pytest.mark.parametrize("gamma,mu", [(1.0, 0.1), (0.3, 0.9)])
@pytest.mark.parametrize("summaries", [False, True])
def test_structures_eval_and_screen(o, struct, gamma, mu, summaries, monkeypatch):
    # summaries: the chunk-summary screen (k_screen) forced on these small
    # instances; otherwise they take the small-instance screen (k_screen_rows)
    if summaries:
        monkeypatch.setenv("GSOT_SCREEN_SUMMARIES", "1")
        monkeypatch.setenv("GSOT_CTX_CACHE", "0")
    sizes, n = STRUCTURES[struct]
    p, rng = random_problem(sizes, n, gamma, mu, sum(map(ord, struct)), weighted=True)
    ctx = ctx_of(p)
    x0 = np.zeros(p.m + p.n)
    x1 = np.concatenate([rng.uniform(-0.2, 1.6, p.m), rng.uniform(-0.2, 1.6, p.n)])
    x2 = x1 + 0.05 * rng.normal(size=x1.size)
    obj, g, _ = ctx.eval(x1)
    assert_eval_close(o, p, x1, obj, g)
    assert np.array_equal(ctx.plan_columns(x1, 0, p.n), o.plan(p, x1[: p.m], x1[p.m:]))
    if p.n > 3:
        assert np.array_equal(ctx.plan_columns(x1, 1, p.n - 1),
                              o.plan(p, x1[: p.m], x1[p.m:])[:, 1: p.n - 1])
    z_o, k_o, oo_o = o.snapshot(p, x1[: p.m], x1[p.m:])
    assert np.array_equal(ctx.block_mask(x1), z_o > p.mu * p.gamma)
    ctx.init_snapshot(x0)
    ctx.refresh(x1, True)
    z, k, oo = ctx.snapshot_norms()
    assert np.array_equal(z, z_o) and np.array_equal(k, k_o) and np.array_equal(oo, oo_o)
    mem, cnt = ctx.active_set()
    mem_o, cnt_o = o.active_set(p, x0[: p.m], x0[p.m:], x1[: p.m], x1[p.m:])
    assert cnt == cnt_o and np.array_equal(mem, mem_o.astype(bool))
    obj_s, g_s, st = ctx.eval(x2, screened=True)
    ga, gb, c_o, _ = o.fast_gradient(p, x1[: p.m], x1[p.m:], mem_o, x2[: p.m], x2[p.m:])
    assert [st.in_active, st.skipped, st.unskipped, st.upper_bounds] == c_o.tolist()
    assert_eval_close(o, p, x2, obj_s, g_s, None, np.concatenate([ga, gb]))
    obj_d, g_d, _ = ctx.eval(x2)
    assert obj_d == obj_s and np.array_equal(g_d, g_s)
    ctx.close()


@pytest.mark.parametrize("struct", sorted(STRUCTURES))
def test_structures_plan_diagnostics(o, struct):
    """gsot_plan_diagnostics on every structure (singletons, n = 1, n = 33, tall
    and ragged groups) against the oracle's plan_diagnostics of its own plan:
    the all-zero block fraction exactly, residuals and mass within 1e-12."""
    sizes, n = STRUCTURES[struct]
    p, rng = random_problem(sizes, n, 0.5, 0.4, 7 + len(struct), weighted=True)
    ctx = ctx_of(p)
    for scale in (0.0, 0.5, 1.5):
        x = scale * np.concatenate([rng.uniform(-0.2, 1.6, p.m), rng.uniform(-0.2, 1.6, p.n)])
        d = ctx.plan_diagnostics(x)
        ref = o.plan_diagnostics(p, o.plan(p, x[: p.m], x[p.m:]))
        assert d.group_sparsity == ref[2]
        for got, want in ((d.marginal_res_a, ref[0]), (d.marginal_res_b, ref[1]), (d.mass, ref[3])):
            assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (struct, scale, got, want)
    ctx.close()


def test_python_run_grid_all_modes(o, gold):
    """run_grid over every solver mode: audit and fast-no-lb runs report the final
    active set like fast (bench.hpp:168-175); the same instance context serves
    every run (one upload)."""
    p = gold_problem(gold, "ragged", 1)
    inst = G.ProblemInstance(p.cost, p.a, p.b, G.GroupPartition(p.sizes))
    modes = [G.SolverMode.baseline, G.SolverMode.fast, G.SolverMode.fast_no_lower_bound,
             G.SolverMode.audit]
    grid = G.GridSpec(gammas=[0.5], rhos=[0.3], modes=modes,
                      base=G.SolverOptions(max_outer_loops=3, grad_tol=1e-12))
    rows = G.run_grid(inst, grid, len(p.sizes), 0)
    assert [r.mode for r in rows] == ["baseline", "fast", "fast-no-lb", "audit"]
    assert rows[0].active_set_size_final == 0 and rows[0].blocks_skipped == 0
    # the screened modes reproduce the baseline trajectory bit for bit (Theorem 2):
    # the same solution, hence the same diagnostics and final active set
    for r in rows[1:]:
        assert (r.objective, r.iterations) == (rows[0].objective, rows[0].iterations)
        assert (r.group_sparsity, r.marginal_res_a, r.marginal_res_b) == \
            (rows[0].group_sparsity, rows[0].marginal_res_a, rows[0].marginal_res_b)
        assert r.active_set_size_final == rows[1].active_set_size_final
        assert r.blocks_computed + r.blocks_skipped == rows[0].blocks_computed
    assert rows[1].blocks_skipped > 0


def test_fast_equals_baseline_bitwise_on_device(o):
    # SPEC.md:315/:320 (Theorem 2): the screened solve follows the unscreened
    # trajectory exactly.
    p, _ = random_problem([12, 7, 30, 1, 9], 50, 0.4, 0.7, 3)
    ctx = ctx_of(p)
    rb = ctx.solve(mode=0, max_outer_loops=15, grad_tol=1e-12)
    for mode in (1, 2, 3):
        rf = ctx.solve(mode=mode, max_outer_loops=15, grad_tol=1e-12)
        assert np.array_equal(rf["x"], rb["x"])
        assert rf["objective"] == rb["objective"]
        assert rf["iterations"] == rb["iterations"] and rf["grad_calls"] == rb["grad_calls"]
    ctx.close()


def test_audit_mode_and_fault_injection(o):
    p, _ = random_problem([10, 10, 10], 40, 0.5, 0.8, 4)
    ctx = ctx_of(p)
    r = ctx.solve(mode=3, max_outer_loops=10)
    assert r["audit_gradient_calls"] == r["grad_calls"]
    assert r["audit_column_compares"] == r["grad_calls"] * p.n
    assert r["audit_skip_checks"] == r["blocks_skipped"]
    with pytest.raises(G.AuditViolation):
        ctx.solve(mode=3, max_outer_loops=10, upper_bound_offset=-1e3)
    ctx.close()


def test_validation_matches_reference_semantics(o):
    cost = np.zeros((3, 4))
    cost[2, 1] = -1.0
    cost[0, 3] = np.nan
    sizes, a, b = [2, 1], np.full(3, 1 / 3), np.full(4, 0.25)
    with pytest.raises(G.NegativeCost) as e:
        G.Context.from_arrays(cost, sizes, a, b, 1.0, 1.0)
    assert (e.value.row, e.value.col, e.value.value) == (2, 1, -1.0)
    p = Problem(cost, np.array(sizes, np.int32), a, b, 1.0, 1.0)
    st, d = o.validate(p)
    assert st == 2 and (d["row"], d["col"]) == (2, 1)
    cost[2, 1] = 0.0
    with pytest.raises(G.NegativeCost) as e:  # NaN is rejected too
        G.Context.from_arrays(cost, sizes, a, b, 1.0, 1.0)
    assert (e.value.row, e.value.col) == (0, 3)
    with pytest.raises(G.MarginalNotNormalized) as e:
        G.Context.from_arrays(np.zeros((3, 4)), sizes, [0.6, 0.6, -0.2], b, 1.0, 1.0)
    assert e.value.which == "a" and e.value.index == 2
    with pytest.raises(G.MarginalNotNormalized) as e:
        G.Context.from_arrays(np.zeros((3, 4)), sizes, a, [0.3, 0.3, 0.3, 0.3], 1.0, 1.0)
    assert e.value.which == "b" and e.value.index == -1
    with pytest.raises(G.PartitionMismatch):
        G.Context.from_arrays(np.zeros((3, 4)), [2, 2], a, b, 1.0, 1.0)
    # compensated sum: 12800 x 1/12800 (test_core.cpp:60-67)
    m = 12800
    G.Context.from_arrays(np.zeros((m, 2)), [10] * 1280, np.full(m, 1 / m), [.5, .5], 1., 1.)


def test_python_mirror_api(o):
    p, _ = random_problem([5, 6, 7], 20, 0.5, 0.5, 9)
    inst = G.ProblemInstance(p.cost, p.a, p.b, G.GroupPartition(p.sizes))
    prm = G.RegParams(p.gamma, p.mu)
    s = G.DualState(np.full(p.m, 0.3), np.full(p.n, 0.2))
    assert abs(G.dual_objective(s, inst, prm) - o.objective(p, s.alpha, s.beta)) <= 1e-12
    ga, gb = G.dual_gradient(s, inst, prm)
    oa, ob = o.gradient(p, s.alpha, s.beta)
    assert np.allclose(ga, oa, atol=1e-14) and np.allclose(gb, ob, atol=1e-14)
    assert np.array_equal(G.recover_plan(s, inst, prm).plan, o.plan(p, s.alpha, s.beta))
    for mode in G.SolverMode:
        sol = G.solve(inst, prm, G.SolverOptions(max_outer_loops=5, mode=mode))
        assert sol.iterations > 0 and sol.stats.grad_calls == len(sol.stats.history)
    sol, rep = G.audit_solve(inst, prm, G.SolverOptions(max_outer_loops=5))
    assert rep.gradient_calls == sol.stats.grad_calls
    d = G.plan_diagnostics(sol.plan, inst)
    assert 0.0 <= d.group_sparsity <= 1.0 and d.mass > 0


def test_python_dispatcher_upper_bound_offset(o):
    """FastGradDispatcher(inst, p, stats, use_active_set, upper_bound_offset)
    (screening.hpp:206-215, :264): a negative offset skips blocks the safe
    screen would compute (audit_solve's fault injection), so the gradient
    may differ from the dense one; decisions and counters follow the oracle's
    dispatcher with the same offset, and the gradient is the oracle's."""
    p, rng = random_problem([12, 7, 30, 1, 9], 60, 0.4, 0.7, 5, weighted=True)
    inst = G.ProblemInstance(p.cost, p.a, p.b, G.GroupPartition(p.sizes))
    prm = G.RegParams(p.gamma, p.mu)
    x0 = np.zeros(p.m + p.n)
    x1 = np.concatenate([rng.uniform(-0.1, 1.2, p.m), rng.uniform(-0.1, 1.2, p.n)]) * 0.05
    x2 = x1 + 1e-3 * rng.normal(size=x1.size)
    skipped = [_dispatcher_offset_case(o, p, inst, prm, x0, x1, x2, off)
               for off in (-0.2, 0.0, 0.05)]
    assert skipped[0] >= skipped[1] >= skipped[2]


def _dispatcher_offset_case(o, p, inst, prm, x0, x1, x2, offset):
    st = G.GradStats()
    disp = G.FastGradDispatcher(inst, prm, st, True, offset)
    disp.init(G.DualState(x0[: p.m], x0[p.m:]))
    disp.refresh(G.DualState(x1[: p.m], x1[p.m:]))
    ga, gb, _ = disp.gradient(G.DualState(x2[: p.m], x2[p.m:]))
    mem_o, _ = o.active_set(p, x0[: p.m], x0[p.m:], x1[: p.m], x1[p.m:])
    ga_o, gb_o, cnt, _ = o.fast_gradient(p, x1[: p.m], x1[p.m:], mem_o, x2[: p.m], x2[p.m:],
                                         ub_offset=offset)
    assert list(st.history[-1]) == cnt.tolist()
    scale = grad_scale(o, p, x2)
    err = np.abs(np.concatenate([ga, gb]) - np.concatenate([ga_o, gb_o]))
    assert np.all(err <= GRAD_STOL * scale)
    return int(cnt[1])


def test_python_run_grid(o, gold):
    """run_grid (bench.hpp:137-180) through the Python mirror on the reference's
    own synthetic instance: the reference's (gamma, rho, mode) order, one
    record per run, each record equal to the solve and the device diagnostics
    it summarises, the CSV schema of bench.hpp:37-68; objectives near the
    oracle's solves (fast mode re-associates sums: 1e-6 relative)."""
    p = gold_problem(gold, "synth", 0)
    inst = G.ProblemInstance(p.cost, p.a, p.b, G.GroupPartition(p.sizes))
    grid = G.GridSpec(gammas=[1.0, 0.1], rhos=[0.2, 0.8],
                      modes=[G.SolverMode.baseline, G.SolverMode.fast],
                      base=G.SolverOptions(max_outer_loops=4, grad_tol=1e-12))
    seen = []
    rows = G.run_grid(inst, grid, 5, 20, sink=lambda r, sol: seen.append((r, sol)))
    assert [(r.gamma, r.rho, r.mode) for r in rows] == [
        (g, r, m) for g in (1.0, 0.1) for r in (0.2, 0.8) for m in ("baseline", "fast")]
    assert len(seen) == len(rows) and all(a is r for (a, _), r in zip(seen, rows))
    assert G.bench_csv_header().count(",") == 18
    for rec, sol in seen:
        assert len(G.to_csv_row(rec).split(",")) == 19
        prm = G.params_from_rho(rec.gamma, rec.rho)
        q = Problem(p.cost, p.sizes, p.a, p.b, prm.gamma(), prm.mu())
        mode = 0 if rec.mode == "baseline" else 1
        ro = o.solve(q, mode=mode, max_outer_loops=4, grad_tol=1e-12)
        assert abs(rec.objective - ro["objective"]) <= 1e-6 * abs(ro["objective"])
        assert rec.iterations == sol.iterations and rec.objective == sol.objective
        assert rec.blocks_computed == sol.stats.blocks_in_active_set + sol.stats.blocks_unskipped
        d = G.state_plan_diagnostics(sol.state, inst, prm)
        assert (rec.group_sparsity, rec.marginal_res_a, rec.marginal_res_b) == \
            (d.group_sparsity, d.marginal_res_a, d.marginal_res_b)
        ref = o.plan_diagnostics(q, o.plan(q, sol.state.alpha, sol.state.beta))
        assert rec.group_sparsity == ref[2]
        if rec.mode == "baseline":
            assert rec.active_set_size_final == 0
        else:
            mem, cnt = o.active_set(q, sol.state.alpha, sol.state.beta, sol.state.alpha,
                                    sol.state.beta)
            assert rec.active_set_size_final == cnt


# ------------------------------------------------------------ configs


def config_problem(o, cfg):
    import ctypes as C

    gamma, mu = {1: (1.0, 0.1), 2: (0.1, 0.5)}[cfg]
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    cost = o.cost_matrix(src, tgt)
    cost /= cost.max()
    return Problem(cost, sizes, a, b, gamma, mu), src, tgt


def test_cost_matrix_device_matches_reference_definition(o):
    import ctypes as C

    import torch

    src, tgt, sizes, a, b = G.config_features(1, 1)
    m, n, d = src.shape[0], tgt.shape[0], src.shape[1]
    dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
    G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(
        src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 0,
        C.c_void_p(dev.data_ptr())))
    torch.cuda.synchronize()
    got = dev.cpu().numpy().T
    assert np.array_equal(got, o.cost_matrix(src, tgt))  # data_io.hpp:101-123, bitwise


def test_config1_solve_vs_oracle(o):
    # BASELINE config 1 (m = n = 1000). Fast mode over a 20-iteration
    # horizon: same iterations and calls, iterates within 1e-9 relative,
    # objective within 1e-9, plans within 1e-6. The full 100-iteration solve
    # is compared bitwise in exact-order mode (tests/test_gpu_exact.py): the
    # fast mode's re-associated sums make unconverged trajectories drift
    # apart beyond ~30 iterations.
    p, _, _ = config_problem(o, 1)
    ctx = G.Context.from_config(1, 1, p.gamma, p.mu)
    r = ctx.solve(mode=1, max_outer_loops=2, grad_tol=1e-12)
    ro = o.solve(p, mode=1, max_outer_loops=2, grad_tol=1e-12)
    assert r["iterations"] == ro["iterations"] == 20 and r["grad_calls"] == ro["grad_calls"]
    assert np.max(np.abs(r["x"] - ro["x"])) <= 1e-9 * np.max(np.abs(ro["x"]))
    assert abs(r["objective"] - ro["objective"]) <= OBJ_RTOL * abs(ro["objective"])
    plan = ctx.plan_columns(r["x"], 0, p.n)
    plan_o = o.plan(p, ro["x"][: p.m], ro["x"][p.m:])
    assert np.max(np.abs(plan - plan_o)) <= PLAN_ATOL
    # the device context built from features equals one built from the
    # oracle's cost matrix
    ctx2 = ctx_of(p)
    x = r["x"]
    o1, g1, _ = ctx.eval(x)
    o2, g2, _ = ctx2.eval(x)
    assert o1 == o2 and np.array_equal(g1, g2)
    assert_eval_close(o, p, x, o1, g1)


def test_config2_full_size_properties(o):
    # Full BASELINE size: properties the oracle need not recompute, plus one
    # oracle evaluation at a mid-solve state.
    p, _, _ = config_problem(o, 2)
    ctx = G.Context.from_config(2, 2, p.gamma, p.mu)
    r = ctx.solve(mode=1, max_outer_loops=3, grad_tol=1e-12)
    x = r["x"]
    obj, g, _ = ctx.eval(x)
    ctx.init_snapshot(x * 0.9)
    ctx.refresh(x * 0.95, True)
    obj_s, g_s, st = ctx.eval(x, screened=True)
    assert obj_s == obj and np.array_equal(g_s, g)
    assert st.in_active + st.skipped + st.unskipped == p.L * p.n
    # sum(grad_alpha) = 1 - mass = sum(grad_beta)
    assert abs(g[: p.m].sum() - g[p.m:].sum()) <= 1e-12
    assert_eval_close(o, p, x, obj, g)
    ctx.close()


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_full_size_properties_configs_3_to_5(cfg):
    """BASELINE configs 3-5 at full size (8 / 9.6 / 40 GB of cost), through
    size-independent properties: screened == dense bitwise and repeatable,
    the GradStats identity, sum(grad_alpha) = 1 - mass = sum(grad_beta), the
    device plan diagnostics' mass and nonzero-block count consistent with the
    gradient and the block mask, and the exact-order (reference-order)
    evaluation within 1e-9 of the fast one."""
    gamma, mu = {3: (0.1, 0.2), 4: (0.05, 0.3), 5: (0.1, 0.5)}[cfg]
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    m, n, L = ctx.m, ctx.n, ctx.L
    r = ctx.solve(mode=1, max_outer_loops=1, grad_tol=1e-12)
    x = r["x"]
    obj, g, st_d = ctx.eval(x)
    assert st_d.unskipped == L * n
    obj2, g2, _ = ctx.eval(x)
    assert obj2 == obj and np.array_equal(g2, g)
    ctx.init_snapshot(x * 0.999)
    ctx.refresh(x, True)  # active set from the 0.999 x snapshot, new snapshot at x
    obj_s, g_s, st = ctx.eval(x, screened=True)
    assert obj_s == obj and np.array_equal(g_s, g)
    assert st.in_active + st.skipped + st.unskipped == L * n and st.skipped > 0
    sa, sb = g[:m].sum(), g[m:].sum()
    assert abs(sa - sb) <= 1e-12
    d = ctx.plan_diagnostics(x)
    assert abs(d.mass - (1.0 - sa)) <= 1e-10
    nz = int(ctx.block_mask(x).sum())
    assert nz == round((1.0 - d.group_sparsity) * L * n)
    obj_x, g_x, _ = ctx.eval(x, exact=True)
    assert abs(obj_x - obj) <= 1e-9 * abs(obj)
    assert np.max(np.abs(g_x - g)) <= 1e-9 * max(1.0, float(np.max(np.abs(g))))
    ctx.close()


def test_context_cache_reuse_is_clean(o):
    # gsot_destroy parks a context's device state and gsot_create of the same
    # shape and partition takes it back (buffers, stream, captured graphs).
    # A context created from new data (and new gamma, mu) on reused state must
    # behave exactly as a fresh one.
    sizes = [12, 7, 30, 1, 9]
    p1, _ = random_problem(sizes, 50, 0.4, 0.7, 11)
    p2, _ = random_problem(sizes, 50, 0.25, 0.9, 12)
    kw = dict(mode=1, max_outer_loops=6, grad_tol=1e-12)
    c1 = ctx_of(p1)
    c1.solve(**kw)
    c1.close()  # parked
    c2 = ctx_of(p2)  # same shape: takes the parked state
    c3 = ctx_of(p2)  # fresh state (the cache is empty now)
    rng = np.random.default_rng(2)
    x = rng.normal(scale=0.05, size=p2.m + p2.n)
    for c in (c2, c3):
        obj, g, _ = c.eval(x)
        assert_eval_close(o, p2, x, obj, g)
    r2, r3 = c2.solve(**kw), c3.solve(**kw)
    assert np.array_equal(r2["x"], r3["x"]) and r2["objective"] == r3["objective"]
    assert r2["grad_calls"] == r3["grad_calls"]
    assert r2["blocks_skipped"] == r3["blocks_skipped"]
    c2.close()
    # an invalid instance of the cached shape fails as usual and leaves no state
    bad = Problem(p2.cost.copy(), p2.sizes, p2.a, p2.b, p2.gamma, p2.mu)
    bad.cost[3, 2] = -1.0
    with pytest.raises(G.NegativeCost):
        ctx_of(bad)
    c4 = ctx_of(p1)
    obj, g, _ = c4.eval(x)
    assert_eval_close(o, p1, x, obj, g)
    c4.close()
    c3.close()


@pytest.mark.parametrize("sizes,n", [([70, 100, 64, 9, 130, 33, 65, 80, 77], 200),
                                     ([300, 64, 5, 90], 97)])
def test_summary_screen_and_listed_snapshots(o, sizes, n, monkeypatch):
    # The chunk-summary screen (k_screen: whole chunks decided from the extremes
    # of z~ / dbeta / beta / cmin, mixed chunks walked) forced on a small instance,
    # with groups tall enough for the listed lazy snapshot (k_snapshot_mark /
    # k_snapshot_walk and the zero_chunk flags). Decisions and counters are the
    # reference's; screened == dense bitwise; fast == baseline solve bitwise; and
    # a context whose arrays went through lazy snapshots, full API snapshots and
    # lazy ones again solves exactly as a fresh one.
    monkeypatch.setenv("GSOT_SCREEN_SUMMARIES", "1")
    monkeypatch.setenv("GSOT_CTX_CACHE", "0")
    p, rng = random_problem(sizes, n, 0.3, 0.6, 61 + n, weighted=True)
    kw = dict(max_outer_loops=4, grad_tol=1e-12)
    ctx = ctx_of(p)
    rb = ctx.solve(mode=0, **kw)
    rf = ctx.solve(mode=1, **kw)  # lazy, listed snapshots
    assert np.array_equal(rf["x"], rb["x"]) and rf["objective"] == rb["objective"]
    x0 = np.zeros(p.m + p.n)
    for scale, spread in ((1e-3, 1e-5), (0.6, 1e-3)):
        beta = rng.uniform(-0.1, 1.2, p.n) * scale
        beta[5:40] = -2.0  # whole chunks provably zero
        x1 = np.concatenate([rng.uniform(-0.1, 1.2, p.m) * scale, beta])
        x2 = x1 + spread * rng.normal(size=x1.size)
        ctx.init_snapshot(x0)  # full API snapshots over the lazy ones
        ctx.refresh(x1, True)
        mem_o, _ = o.active_set(p, x0[: p.m], x0[p.m:], x1[: p.m], x1[p.m:])
        obj_s, g_s, st = ctx.eval(x2, screened=True)
        ga, gb, c_o, _ = o.fast_gradient(p, x1[: p.m], x1[p.m:], mem_o, x2[: p.m], x2[p.m:])
        assert [st.in_active, st.skipped, st.unskipped, st.upper_bounds] == c_o.tolist()
        assert_eval_close(o, p, x2, obj_s, g_s, None, np.concatenate([ga, gb]))
        obj_d, g_d, _ = ctx.eval(x2)
        assert obj_d == obj_s and np.array_equal(g_d, g_s)
        z, k, oo = ctx.snapshot_norms()
        z_o, k_o, oo_o = o.snapshot(p, x1[: p.m], x1[p.m:])
        assert np.array_equal(z, z_o) and np.array_equal(k, k_o) and np.array_equal(oo, oo_o)
    again = ctx.solve(mode=1, **kw)  # lazy snapshots over the full ones
    fresh = ctx_of(p)
    rf2 = fresh.solve(mode=1, **kw)
    for r in (again, rf2):
        assert np.array_equal(r["x"], rf["x"]) and r["objective"] == rf["objective"]
        assert r["grad_calls"] == rf["grad_calls"] and r["blocks_skipped"] == rf["blocks_skipped"]
    fresh.close()
    ctx.close()


def test_many_groups_screen_layout(o):
    # L x n large enough (>= 4 CTAs per SM of work) for the transposed screen
    # kernel (lane = chunk, warp = group): decisions and counters still the
    # reference's, screened == dense bitwise, and a fast solve (fused group
    # norms in the screen) follows the baseline solve bit for bit.
    sizes = [3] * 1000
    p, rng = random_problem(sizes, 5000, 0.3, 0.6, 21, weighted=True)
    ctx = ctx_of(p)
    x0 = np.zeros(p.m + p.n)
    x1 = np.concatenate([rng.uniform(-0.1, 1.2, p.m), rng.uniform(-0.1, 1.2, p.n)]) * 1e-3
    x2 = x1 + 1e-5 * rng.normal(size=x1.size)
    ctx.init_snapshot(x0)
    ctx.refresh(x1, True)
    mem_o, _ = o.active_set(p, x0[: p.m], x0[p.m:], x1[: p.m], x1[p.m:])
    obj_s, g_s, st = ctx.eval(x2, screened=True)
    ga, gb, c_o, _ = o.fast_gradient(p, x1[: p.m], x1[p.m:], mem_o, x2[: p.m], x2[p.m:])
    assert [st.in_active, st.skipped, st.unskipped, st.upper_bounds] == c_o.tolist()
    assert_eval_close(o, p, x2, obj_s, g_s, None, np.concatenate([ga, gb]))
    obj_d, g_d, _ = ctx.eval(x2)
    assert obj_d == obj_s and np.array_equal(g_d, g_s)
    rb = ctx.solve(mode=0, max_outer_loops=3, grad_tol=1e-12)
    rf = ctx.solve(mode=1, max_outer_loops=3, grad_tol=1e-12)
    assert np.array_equal(rf["x"], rb["x"]) and rf["objective"] == rb["objective"]
    assert rf["blocks_skipped"] > 0
    ctx.close()


def test_tall_blocks_streamed_twice(o):
    # Blocks taller than one shared-memory segment (128 rows) are streamed
    # twice by one CTA (pass 1 forwards, pass 2 backwards): 30000 rows (235
    # segments), 1000 rows (8), 129 rows (a 1-row last segment). Against the
    # oracle, screened == dense bitwise, repeatable, fast == baseline bitwise.
    sizes = [30000, 1000, 129, 3]
    p, rng = random_problem(sizes, 40, 0.3, 0.6, 31, weighted=True)
    ctx = ctx_of(p)
    x0 = np.zeros(p.m + p.n)
    x1 = np.concatenate([rng.uniform(-0.1, 1.2, p.m) * 1e-4, rng.uniform(-0.1, 1.2, p.n)])
    x2 = x1 + 1e-6 * rng.normal(size=x1.size)
    obj, g, _ = ctx.eval(x1)
    assert_eval_close(o, p, x1, obj, g)
    ctx.init_snapshot(x0)
    ctx.refresh(x1, True)
    mem_o, _ = o.active_set(p, x0[: p.m], x0[p.m:], x1[: p.m], x1[p.m:])
    obj_s, g_s, st = ctx.eval(x2, screened=True)
    ga, gb, c_o, _ = o.fast_gradient(p, x1[: p.m], x1[p.m:], mem_o, x2[: p.m], x2[p.m:])
    assert [st.in_active, st.skipped, st.unskipped, st.upper_bounds] == c_o.tolist()
    assert_eval_close(o, p, x2, obj_s, g_s, None, np.concatenate([ga, gb]))
    obj_d, g_d, _ = ctx.eval(x2)
    assert obj_d == obj_s and np.array_equal(g_d, g_s)
    for _ in range(3):
        obj_r, g_r, _ = ctx.eval(x2)
        assert obj_r == obj_d and np.array_equal(g_r, g_d)
    rb = ctx.solve(mode=0, max_outer_loops=3, grad_tol=1e-12)
    rf = ctx.solve(mode=1, max_outer_loops=3, grad_tol=1e-12)
    assert np.array_equal(rf["x"], rb["x"]) and rf["objective"] == rb["objective"]
    ctx.close()


@pytest.mark.parametrize("sizes", [[100, 28, 5], [300, 129, 7]])
def test_eval_variants_agree_bitwise(o, sizes, monkeypatch):
    # k_eval<false> writes [f]+ in place, k_eval<true> (the two-pass variant for
    # blocks taller than a segment, kept behind GSOT_EVAL_TALL_OLD for comparison
    # with the quarter pipeline) recomputes it in pass 2: the same bits either way.
    p, rng = random_problem(sizes, 70, 0.3, 0.6, 41, weighted=True)
    x = np.concatenate([rng.uniform(-0.1, 1.2, p.m) * 1e-3, rng.uniform(-0.1, 1.2, p.n)])
    out = []
    monkeypatch.setenv("GSOT_EVAL_TALL_OLD", "1")
    for v in ("0", "1"):
        monkeypatch.setenv("GSOT_EVAL_RECOMPUTE", v)
        monkeypatch.setenv("GSOT_CTX_CACHE", "0")
        ctx = ctx_of(p)
        ctx.init_snapshot(np.zeros(p.m + p.n))
        ctx.refresh(x, True)
        out.append((ctx.eval(x)[:2], ctx.eval(x * 1.01, screened=True)[:2]))
        ctx.close()
    (d0, s0), (d1, s1) = out
    assert d0[0] == d1[0] and np.array_equal(d0[1], d1[1])
    assert s0[0] == s1[0] and np.array_equal(s0[1], s1[1])
    assert_eval_close(o, p, x, d1[0], d1[1])


@pytest.mark.parametrize("sizes,n", [([500, 124, 125, 449, 448, 3], 70),
                                     ([1100, 460, 200, 64, 9], 45),
                                     ([129] * 5 + [16, 1], 33)])
def test_quarter_pipeline(o, sizes, n, monkeypatch):
    # k_eval_q (instances with a group taller than a whole-tile segment): short
    # groups as whole tiles, taller ones one 8-column quarter at a time (resident
    # up to the quarter-segment rows, streamed twice above), quarters without a
    # possibly-nonzero block never fetched. beta is pushed far down on runs of
    # columns so that whole quarters are provably zero. Against the oracle;
    # screened == dense bitwise; repeatable; fast == baseline solve bitwise.
    monkeypatch.setenv("GSOT_CTX_CACHE", "0")
    p, rng = random_problem(sizes, n, 0.3, 0.6, 51 + n, weighted=True)
    ctx = ctx_of(p)
    x0 = np.zeros(p.m + p.n)
    beta = rng.uniform(-0.1, 1.2, p.n)
    for lo, hi in ((3, 14), (16, 24), (40, 41), (n - 9, n - 1)):
        beta[lo:hi] = -3.0
    x1 = np.concatenate([rng.uniform(-0.1, 1.2, p.m) * 1e-2, beta])
    x2 = x1 + 1e-5 * rng.normal(size=x1.size)
    obj, g, _ = ctx.eval(x1)
    assert_eval_close(o, p, x1, obj, g)
    ctx.init_snapshot(x0)
    ctx.refresh(x1, True)
    mem_o, _ = o.active_set(p, x0[: p.m], x0[p.m:], x1[: p.m], x1[p.m:])
    obj_s, g_s, st = ctx.eval(x2, screened=True)
    ga, gb, c_o, _ = o.fast_gradient(p, x1[: p.m], x1[p.m:], mem_o, x2[: p.m], x2[p.m:])
    assert [st.in_active, st.skipped, st.unskipped, st.upper_bounds] == c_o.tolist()
    assert_eval_close(o, p, x2, obj_s, g_s, None, np.concatenate([ga, gb]))
    obj_d, g_d, _ = ctx.eval(x2)
    assert obj_d == obj_s and np.array_equal(g_d, g_s)
    for _ in range(3):
        obj_r, g_r, _ = ctx.eval(x2)
        assert obj_r == obj_d and np.array_equal(g_r, g_d)
    rb = ctx.solve(mode=0, max_outer_loops=3, grad_tol=1e-12)
    rf = ctx.solve(mode=1, max_outer_loops=3, grad_tol=1e-12)
    assert np.array_equal(rf["x"], rb["x"]) and rf["objective"] == rb["objective"]
    ctx.close()
