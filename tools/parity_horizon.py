"""Diagnostic: device fast / exact solves at the full BASELINE budget against
the oracle (the reference's own order of operations).

    python tools/parity_horizon.py [--configs 1,2]

Prints, per config: iterations, gradient calls, max |x - x_ref| / max|x_ref|,
objective difference, max plan difference, and the solve times of both
device modes."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2303_07597_b200 as G  # noqa: E402
from oracle_bindings import Oracle, Problem  # noqa: E402

CONFIGS = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2")
    args = ap.parse_args()
    o = Oracle()
    for cfg in [int(c) for c in args.configs.split(",")]:
        gamma, mu, iters = CONFIGS[cfg]
        src, tgt, sizes, a, b = G.config_features(cfg, cfg)
        cost = o.cost_matrix(src, tgt)
        cost /= cost.max()
        p = Problem(cost, sizes, a, b, gamma, mu)
        t0 = time.time()
        ro = o.solve(p, mode=1, max_outer_loops=iters // 10, grad_tol=1e-12, plan=True)
        t_o = time.time() - t0
        ctx = G.Context.from_config(cfg, cfg, gamma, mu)
        out = {"config": cfg, "oracle_s": t_o, "oracle_iters": ro["iterations"],
               "oracle_calls": ro["grad_calls"]}
        for name, exact in (("fast", False), ("exact", True)):
            ctx.solve(mode=1, max_outer_loops=iters // 10, grad_tol=1e-12, exact=exact)
            r = ctx.solve(mode=1, max_outer_loops=iters // 10, grad_tol=1e-12, exact=exact,
                          history_cap=100000)
            plan = ctx.plan_columns(r["x"], 0, p.n)
            hist_eq = bool(np.array_equal(r["history"], ro["history"]))
            out[name] = {"iters": r["iterations"], "calls": r["grad_calls"],
                         "solve_ms": 1e3 * r["wall_seconds"],
                         "x_rel": float(np.max(np.abs(r["x"] - ro["x"])) / np.max(np.abs(ro["x"]))),
                         "obj_diff": float(r["objective"] - ro["objective"]),
                         "obj_rel": float(abs(r["objective"] - ro["objective"]) / abs(ro["objective"])),
                         "plan_maxdiff": float(np.max(np.abs(plan - ro["plan"]))),
                         "plan_max": float(np.max(ro["plan"])),
                         "history_equal": hist_eq}
        ctx.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
