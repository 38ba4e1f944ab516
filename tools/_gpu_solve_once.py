"""GPU helper (not a test): two solves of one config; prints the second.
The second solve is bracketed by cudaProfilerStart/Stop (ncu
--profile-from-start off captures exactly that solve).

    python tools/_gpu_solve_once.py [MODE] [prof] [--config C] [--exact]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_07597_b200 as G  # noqa: E402

CONFIGS = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
           5: (0.1, 0.5, 300)}
ap = argparse.ArgumentParser()
ap.add_argument("mode", nargs="?", type=int, default=1)
ap.add_argument("prof", nargs="?", default=None)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--exact", action="store_true")
args = ap.parse_args()
rt = ctypes.CDLL("libcudart.so.12") if args.prof else None
gamma, mu, iters = CONFIGS[args.config]
ctx = G.Context.from_config(args.config, args.config, gamma, mu)
kw = dict(mode=args.mode, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=iters // 10,
          exact=args.exact)
ctx.solve(**kw)
if rt:
    rt.cudaProfilerStart()
r = ctx.solve(**kw)
if rt:
    rt.cudaProfilerStop()
print('config', args.config, 'exact', args.exact, 'calls', r['grad_calls'], 'iters', r['iterations'],
      'obj', repr(r['objective']), 'wall_ms', r['wall_seconds'] * 1e3)
