"""GPU helper: fast-mode solve of config N twice; the second bracketed by
cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import ctypes
import sys
sys.path.insert(0, '.')
import paper_2303_07597_b200 as G
cfg = int(sys.argv[1])
gam, mu, it = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200), 5: (0.1, 0.5, 300)}[cfg]
rt = ctypes.CDLL("libcudart.so.12")
ctx = G.Context.from_config(cfg, cfg, gam, mu)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=int(sys.argv[2]) if len(sys.argv) > 2 else it // 10)
ctx.solve(**kw)
rt.cudaProfilerStart()
r = ctx.solve(**kw)
rt.cudaProfilerStop()
print('calls', r['grad_calls'], 'wall_ms', r['wall_seconds'] * 1e3)
