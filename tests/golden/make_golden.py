"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref).

The reference headers (/root/reference/proj/include/groupot) compiled
against oracle/shim are run here, in the container that holds the
reference; the outputs are committed so that the GPU box (which has no
/root/reference) can check the CUDA path against the reference's own
numbers. Re-run: `python tests/golden/make_golden.py`.

Instances:
  synth   the reference's own generator gen_synthetic(5 classes x 20, seed 3)
          + make_instance(normalize_cost=true)   (data_io.hpp:67-98, :157-181)
  ragged  random cost in [0,2), groups of sizes 1..37 (odd, >32), n = 45
          (not a multiple of 32), uniform marginals
  hand    the hand examples of test_regularizer.cpp / test_dual.cpp
Per instance and (gamma, mu): eval at 3 states, plan at one state, snapshot
at one state, the active set and one screened gradient call with counters,
and solve() in all four modes (x, objective, iterations, history).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import Problem, RefLib  # noqa: E402

PARAMS = [(1.0, 0.1), (0.1, 0.5), (0.5, 0.8)]


def states(p: Problem, rng):
    m, n = p.m, p.n
    s1 = (np.zeros(m), np.zeros(n))
    s2 = (rng.normal(size=m) * 0.05 + 0.02, rng.normal(size=n) * 0.05 + 0.02)
    s3 = (rng.uniform(-0.5, 1.5, m), rng.uniform(-0.5, 1.5, n))
    return [s1, s2, s3]


def record(ref: RefLib, name: str, p: Problem, seed: int, out: dict):
    rng = np.random.default_rng(seed)
    out[f"{name}/cost"] = np.asfortranarray(p.cost)
    out[f"{name}/sizes"] = p.sizes
    out[f"{name}/a"] = p.a
    out[f"{name}/b"] = p.b
    for pi, (gamma, mu) in enumerate(PARAMS):
        q = Problem(p.cost, p.sizes, p.a, p.b, gamma, mu)
        key = f"{name}/p{pi}"
        out[f"{key}/params"] = np.array([gamma, mu])
        sts = states(q, rng)
        for si, (al, be) in enumerate(sts):
            obj, ga, gb = ref.eval(q, al, be)
            out[f"{key}/s{si}/x"] = np.concatenate([al, be])
            out[f"{key}/s{si}/objective"] = np.array([obj])
            out[f"{key}/s{si}/grad"] = np.concatenate([ga, gb])
        al, be = sts[2]
        out[f"{key}/plan"] = ref.plan(q, al, be)
        z, k, o = ref.snapshot(q, *sts[1])
        out[f"{key}/snap_z"], out[f"{key}/snap_k"], out[f"{key}/snap_o"] = z, k, o
        # dispatcher after init(x_a = s0) and refresh(x_s = s1): active set
        # from lower bounds at s1 against the snapshot at s0; gradient at x =
        # s1 + small step.
        x_a, x_s = sts[0], sts[1]
        x = (x_s[0] + 0.01 * rng.normal(size=q.m), x_s[1] + 0.01 * rng.normal(size=q.n))
        for ua in (0, 1):
            ga, gb, cnt, mem = ref.fast_gradient(q, x_a, x_s, x, use_active_set=bool(ua))
            out[f"{key}/fast{ua}/x"] = np.concatenate(x)
            out[f"{key}/fast{ua}/grad"] = np.concatenate([ga, gb])
            out[f"{key}/fast{ua}/counters"] = cnt
            out[f"{key}/fast{ua}/member"] = mem
        for mode in (0, 1, 2, 3):
            r = ref.solve(q, mode=mode, max_outer_loops=20, grad_tol=1e-7)
            sk = f"{key}/solve{mode}"
            out[f"{sk}/x"] = r["x"]
            out[f"{sk}/objective"] = np.array([r["objective"]])
            out[f"{sk}/ints"] = np.array([r["iterations"], r["converged"],
                                          r["line_search_failed"], r["outer_loops"],
                                          r["grad_calls"], r["blocks_in_active_set"],
                                          r["blocks_skipped"], r["blocks_unskipped"],
                                          r["upper_bounds_evaluated"]])
            out[f"{sk}/history"] = r["history"]
        rp = ref.solve(q, mode=1, max_outer_loops=20, grad_tol=1e-7, plan=True)
        out[f"{key}/solve_plan"] = rp["plan"]
        # plan_diagnostics (dual.hpp:139-169) of the plan at s2 and at the solution
        out[f"{key}/plan_diag"] = ref.plan_diagnostics(q, out[f"{key}/plan"])
        out[f"{key}/solve_plan_diag"] = ref.plan_diagnostics(q, rp["plan"])


def main():
    ref = RefLib()
    out = {}
    cost, a, b, sizes, _, _ = ref.gen_synthetic(5, 20, 3, True)
    record(ref, "synth", Problem(cost, sizes, a, b, 1.0, 1.0), 11, out)
    rng = np.random.default_rng(5)
    sizes = np.array([1, 37, 3, 12, 33, 2, 8], np.int32)
    m, n = int(sizes.sum()), 45
    record(ref, "ragged", Problem(rng.uniform(0, 2, (m, n)), sizes, np.full(m, 1 / m),
                                  np.full(n, 1 / n), 1.0, 1.0), 12, out)
    # hand examples (test_dual.cpp:28-35, :83-91, :172-181)
    h = Problem(np.zeros((1, 1)), np.array([1], np.int32), np.ones(1), np.ones(1), 1.0, 0.5)
    obj, ga, gb = ref.eval(h, np.ones(1), np.zeros(1))
    out["hand/1x1/objective"] = np.array([obj])
    out["hand/1x1/grad"] = np.concatenate([ga, gb])
    h2 = Problem(np.zeros((2, 1)), np.array([2], np.int32), np.full(2, 0.5), np.ones(1), 1.0, 1.0)
    out["hand/plan34"] = ref.plan(h2, np.array([3.0, 4.0]), np.zeros(1))
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
