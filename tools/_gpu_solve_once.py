"""GPU helper (not a test): two fast-mode config-2 solves; prints the second.
The second solve is bracketed by cudaProfilerStart/Stop (ncu
--profile-from-start off captures exactly that solve)."""
import ctypes
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_07597_b200 as G
rt = ctypes.CDLL("libcudart.so.12") if len(sys.argv) > 2 else None
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
kw = dict(mode=int(sys.argv[1]) if len(sys.argv) > 1 else 1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20)
ctx.solve(**kw)
if rt: rt.cudaProfilerStart()
r = ctx.solve(**kw)
if rt: rt.cudaProfilerStop()
print('calls', r['grad_calls'], 'iters', r['iterations'], 'obj', repr(r['objective']), 'wall_ms', r['wall_seconds'] * 1e3)
