"""End-to-end L-BFGS solve times for the five BASELINE.json configs on one GPU.

    python tools/solve_configs.py [--configs 1,2,3,4,5] [--e2e] [--out gpurun_out/configs.json]

Per config (SURVEY.md §8(d) recipe, seed = config id, cost generated on device):
fast mode (screening + active set) and baseline mode (every block, every
call) over the config's iteration budget (snapshot interval 10, memory 10,
grad_tol 1e-12 so the solve runs to budget unless it converges first).
Reports the maximize span (the reference's Solution::wall_time), device
evals/s, screening statistics and, with --e2e, the time including the upload
of the host cost matrix through the C ABI (gsot_create).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
           5: (0.1, 0.5, 300)}


def run(cfg: int, e2e: bool, reps: int):
    import paper_2303_07597_b200 as G

    gamma, mu, iters = CONFIGS[cfg]
    t0 = time.perf_counter()
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    t_gen = time.perf_counter() - t0
    kw = dict(snapshot_interval=10, grad_tol=1e-12, max_outer_loops=iters // 10, lbfgs_memory=10,
              history_cap=0)
    out = {"config": cfg, "m": ctx.m, "n": ctx.n, "L": ctx.L, "gamma": gamma, "mu": mu,
           "iteration_budget": iters, "setup_s": t_gen}
    for mode, name in ((1, "fast"), (0, "baseline")):
        ctx.solve(mode=mode, **kw)  # warm-up (graph capture)
        walls = []
        for _ in range(reps):
            r = ctx.solve(mode=mode, **kw)
            walls.append(r["wall_seconds"])
        w = min(walls)
        out[name] = {"solve_ms": 1e3 * w, "solve_ms_all": [1e3 * x for x in walls],
                     "iterations": r["iterations"], "grad_calls": r["grad_calls"],
                     "evals_per_s": r["grad_calls"] / w, "objective": r["objective"],
                     "converged": bool(r["converged"]),
                     "blocks_computed_frac": r["eval_blocks"] / (r["grad_calls"] * ctx.L * ctx.n)}
    out["fast_vs_baseline_speedup"] = out["baseline"]["solve_ms"] / out["fast"]["solve_ms"]
    ctx.close()
    if e2e:
        import numpy as np
        import torch

        m, n, L, d = G.config_shape(cfg)
        src, tgt, sizes, a, b = G.config_features(cfg, cfg)
        host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        cost = host.numpy().T
        dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
        st = G._lib.lib().gsot_cost_matrix_device(
            src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 1,
            C.c_void_p(dev.data_ptr()))
        G.groupot._raise(st)
        host.copy_(dev)
        del dev
        torch.cuda.synchronize()
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            c2 = G.Context.from_arrays(cost, sizes, a, b, gamma, mu)
            t1 = time.perf_counter()
            r = c2.solve(mode=1, **kw)
            c2.close()
            t2 = time.perf_counter()
            cur = {"total_ms": 1e3 * (t2 - t0), "create_ms": 1e3 * (t1 - t0),
                   "solve_ms": 1e3 * (t2 - t1), "h2d_bytes": 8 * m * n + 8 * (m + n) + 4 * L}
            if best is None or cur["total_ms"] < best["total_ms"]:
                best = cur
        out["e2e_fast"] = best
        del host, cost
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--e2e", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    args = ap.parse_args()
    res = []
    for cfg in [int(c) for c in args.configs.split(",")]:
        r = run(cfg, args.e2e, args.reps)
        print(json.dumps(r), flush=True)
        res.append(r)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
