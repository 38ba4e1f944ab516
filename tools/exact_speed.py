"""Exact-order (bitwise-reference) vs fast mode: solve times per config and
the per-kernel-class device time of one profiled exact solve.

    python tools/exact_speed.py [--configs 1,2,3,4,5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
           5: (0.1, 0.5, 300)}
KINDS = {0: "eval", 1: "snapshot", 2: "screen", 3: "active", 4: "finalize", 5: "lbfgs",
         6: "delta", 7: "misc"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    args = ap.parse_args()
    import paper_2303_07597_b200 as G

    for cfg in [int(c) for c in args.configs.split(",")]:
        gamma, mu, iters = CONFIGS[cfg]
        ctx = G.Context.from_config(cfg, cfg, gamma, mu)
        kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=iters // 10)
        out = {"config": cfg}
        for name, ex in (("fast", False), ("exact", True)):
            ctx.solve(exact=ex, **kw)
            ctx.timer_start()
            r = ctx.solve(exact=ex, **kw)
            ms = ctx.timer_stop()
            out[name] = {"ms": ms, "calls": r["grad_calls"], "iters": r["iterations"],
                         "objective": r["objective"]}
        ctx.profile(True)
        ctx.solve(exact=True, **kw)
        ctx.profile_reset()
        ctx.solve(exact=True, **kw)
        ctx.profile(False)
        out["exact_kinds_ms"] = {KINDS[k]: round(ctx.profile_read(k)[0], 3) for k in KINDS
                                 if ctx.profile_read(k)[2]}
        out["exact_launches"] = {KINDS[k]: ctx.profile_read(k)[2] for k in KINDS
                                 if ctx.profile_read(k)[2]}
        ctx.close()
        G.cache_clear()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
