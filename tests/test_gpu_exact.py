"""GPU, exact-order mode: with the reference's own association for every
cross-block sum and every L-BFGS dot (gsot_exact2.cu), the device evaluation
and the whole device solve are BITWISE the reference's (the oracle is
bitwise the reference compiled against the sequential Eigen shim,
tests/test_oracle.py): same iterates, objective, gradient calls, per-call
screening counters and plan, in every solver mode."""
import os

import numpy as np
import pytest

import paper_2303_07597_b200 as G
from oracle_bindings import Oracle, Problem

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def o():
    return Oracle()


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def gold_problem(g, name, pi):
    gamma, mu = g[f"{name}/p{pi}/params"]
    return Problem(g[f"{name}/cost"], g[f"{name}/sizes"], g[f"{name}/a"], g[f"{name}/b"],
                   float(gamma), float(mu))


@pytest.mark.parametrize("name", ["synth", "ragged"])
@pytest.mark.parametrize("pi", [0, 1, 2])
def test_exact_eval_bitwise(gold, name, pi):
    p = gold_problem(gold, name, pi)
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    for si in range(3):
        x = gold[f"{name}/p{pi}/s{si}/x"]
        obj, g, _ = ctx.eval(x, exact=True)
        assert obj == gold[f"{name}/p{pi}/s{si}/objective"][0]
        assert np.array_equal(g, gold[f"{name}/p{pi}/s{si}/grad"])
    ctx.close()


@pytest.mark.parametrize("name", ["synth", "ragged"])
@pytest.mark.parametrize("pi", [0, 1, 2])
def test_exact_solve_matches_reference_golden_bitwise(gold, name, pi):
    p = gold_problem(gold, name, pi)
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    for mode in (0, 1, 2, 3):
        r = ctx.solve(mode=mode, max_outer_loops=20, grad_tol=1e-7, history_cap=100000,
                      exact=True)
        sk = f"{name}/p{pi}/solve{mode}"
        ints = gold[f"{sk}/ints"]
        assert [r["iterations"], r["converged"], r["line_search_failed"], r["outer_loops"],
                r["grad_calls"], r["blocks_in_active_set"], r["blocks_skipped"],
                r["blocks_unskipped"], r["upper_bounds_evaluated"]] == ints.tolist()
        assert np.array_equal(r["x"], gold[f"{sk}/x"])
        assert r["objective"] == gold[f"{sk}/objective"][0]
        assert np.array_equal(r["history"], gold[f"{sk}/history"])
        if mode == 1:
            assert np.array_equal(ctx.plan_columns(r["x"], 0, p.n), gold[f"{name}/p{pi}/solve_plan"])
    ctx.close()


def test_exact_solve_config1_bitwise(o):
    # BASELINE config 1 (m = n = 1000, 100 iterations) against the oracle
    src, tgt, sizes, a, b = G.config_features(1, 1)
    cost = o.cost_matrix(src, tgt)
    cost /= cost.max()
    p = Problem(cost, sizes, a, b, 1.0, 0.1)
    ctx = G.Context.from_config(1, 1, 1.0, 0.1)
    r = ctx.solve(mode=1, max_outer_loops=10, grad_tol=1e-12, history_cap=100000, exact=True)
    ro = o.solve(p, mode=1, max_outer_loops=10, grad_tol=1e-12, plan=True)
    assert r["iterations"] == ro["iterations"] == 100
    assert r["grad_calls"] == ro["grad_calls"]
    assert np.array_equal(r["history"], ro["history"])
    assert np.array_equal(r["x"], ro["x"])
    assert r["objective"] == ro["objective"]
    assert np.array_equal(ctx.plan_columns(r["x"], 0, p.n), ro["plan"])  # final plan bitwise
    ctx.close()


@pytest.mark.parametrize("name", ["synth", "ragged"])
def test_exact_audit_without_active_set_bitwise(o, gold, name):
    """audit_solve of a fast_no_lower_bound SolverOptions (solver.hpp:271: no
    active set, every decision re-verified) through GSOT_SOLVE_NO_ACTIVE_SET:
    bitwise the oracle's mode-4 trajectory, no active-set checks."""
    gamma, mu = gold[f"{name}/p1/params"]
    p = Problem(gold[f"{name}/cost"], gold[f"{name}/sizes"], gold[f"{name}/a"], gold[f"{name}/b"],
                float(gamma), float(mu))
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    r = ctx.solve(mode=3, max_outer_loops=6, grad_tol=1e-12, history_cap=10000, exact=True,
                  no_active_set=True)
    ro = o.solve(p, mode=4, max_outer_loops=6, grad_tol=1e-12)
    assert np.array_equal(r["history"], ro["history"]) and r["blocks_in_active_set"] == 0
    assert np.array_equal(r["x"], ro["x"]) and r["objective"] == ro["objective"]
    assert r["audit_active_checks"] == 0 and r["audit_gradient_calls"] == r["grad_calls"]
    ctx.close()


def test_exact_solve_config2_full_budget_bitwise(o):
    """BASELINE config 2 (m = n = 10,000) over its full 200-iteration budget:
    the exact-order device solve equals the oracle's (the reference's order of
    operations) bit for bit -- iterations, gradient calls, per-call screening
    counters, final state, objective and plan columns (north_star: plan within
    1e-6 after the same number of iterations; here the difference is 0)."""
    src, tgt, sizes, a, b = G.config_features(2, 2)
    cost = o.cost_matrix(src, tgt)
    cost /= cost.max()
    p = Problem(cost, sizes, a, b, 0.1, 0.5)
    ctx = G.Context.from_config(2, 2, 0.1, 0.5)
    r = ctx.solve(mode=1, max_outer_loops=20, grad_tol=1e-12, history_cap=100000, exact=True)
    ro = o.solve(p, mode=1, max_outer_loops=20, grad_tol=1e-12)
    assert r["iterations"] == ro["iterations"] == 200
    assert r["grad_calls"] == ro["grad_calls"]
    assert np.array_equal(r["history"], ro["history"])
    assert np.array_equal(r["x"], ro["x"]) and r["objective"] == ro["objective"]
    cols = np.arange(0, p.n, 7)[:1024]
    plan_o = o.plan(Problem(cost[:, cols], sizes, a, b[cols], 0.1, 0.5), ro["x"][:p.m],
                    ro["x"][p.m:][cols])
    plan = np.concatenate([ctx.plan_columns(r["x"], j, j + 1) for j in cols[:64]], axis=1)
    assert np.array_equal(plan, plan_o[:, :64])
    ctx.close()


def _adversarial(rng, kind, n):
    if kind == 0:  # half-ulp ties galore on a unit start
        return rng.integers(-8, 9, size=n) * 2.0 ** -54 + (rng.random(n) < 0.01) * 1.0
    if kind == 1:  # zeros mixed with normals
        return np.where(rng.random(n) < 0.5, 0.0, rng.normal(size=n))
    if kind == 2:  # few-bit terms over 60 binades, random signs
        return ((rng.integers(0, 4, size=n) * 0.5 + 1) * 2.0 ** rng.integers(-60, 3, size=n)
                * np.sign(rng.normal(size=n)))
    if kind == 3:  # 1 then +-ulp-scale terms (ties at the binade top)
        return np.concatenate([[1.0], rng.integers(-3, 4, size=n - 1) * 2.0 ** -53])
    if kind == 4:  # subnormal scale
        return rng.normal(size=n) * 1e-310
    if kind == 5:  # cancellation: a random walk around zero
        return rng.normal(size=n) * 10.0 ** rng.integers(-3, 3, size=n)
    return rng.random(n)  # monotone growth


@pytest.mark.parametrize("n", [1, 7, 300, 5000, 100_000, 1_200_000])
def test_sequential_sum_engine_bitwise(n):
    """gsot_sequential_sum (the exact-order engine, gsot_seqsum.cuh) equals the
    left-to-right loop ((s0 + t0) + t1) + ... bit for bit on adversarial
    inputs: exact ties, zeros, few-bit terms across 60 binades, subnormals,
    cancellation around zero, monotone growth; several starts."""
    ctx = G.Context.from_arrays(np.full((4, 3), 0.5), [4], np.full(4, 0.25), np.full(3, 1 / 3),
                                1.0, 1.0)
    rng = np.random.default_rng(n)
    for kind in range(7):
        v = _adversarial(rng, kind, n)
        for s0 in (0.0, 1.0, -0.75, 1e-5):
            ref = np.cumsum(np.concatenate([[s0], v]))[-1]  # sequential (np.add.accumulate)
            got = ctx.sequential_sum(v, s0)
            assert got == ref or (np.isnan(got) and np.isnan(ref)), (kind, s0, got, ref)
    ctx.close()


@pytest.mark.parametrize("sizes", [[300, 17, 170, 64, 161, 1], [700, 33], [300, 170, 161, 700]])
def test_exact_tall_groups_eval_and_solve_bitwise(o, sizes):
    """Groups taller than the exact column kernel's resident ring (more than 5
    segments of 32 rows: streamed twice, the second pass only for tiles with a
    nonzero block) next to short ones and a one-row group, and an instance
    whose groups are all tall (the 12-warp, 2-slot kernel variant): the
    exact-order evaluation at several states and a 30-iteration exact solve
    equal the oracle bit for bit."""
    rng = np.random.default_rng(len(sizes))
    sizes = np.array(sizes, np.int32)
    m, n = int(sizes.sum()), 200
    cost = rng.uniform(0.0, 1.0, (m, n))
    p = Problem(cost, sizes, np.full(m, 1.0 / m), np.full(n, 1.0 / n), 0.3, 0.2)
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    for scale in (0.2, 0.6, 1.0):
        x = scale * rng.uniform(0.0, 1.0, m + n)
        obj, g, _ = ctx.eval(x, exact=True)
        obj_o = o.objective(p, x[:m], x[m:])
        ga, gb = o.gradient(p, x[:m], x[m:])
        assert obj == obj_o
        assert np.array_equal(g, np.concatenate([ga, gb]))
    r = ctx.solve(mode=1, max_outer_loops=3, grad_tol=1e-12, history_cap=10000, exact=True)
    ro = o.solve(p, mode=1, max_outer_loops=3, grad_tol=1e-12)
    assert r["iterations"] == ro["iterations"] and r["grad_calls"] == ro["grad_calls"]
    assert np.array_equal(r["history"], ro["history"])
    assert np.array_equal(r["x"], ro["x"]) and r["objective"] == ro["objective"]
    ctx.close()
