import sys, time, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2303_07597_b200 as G
cfg = 2
m, n, L, d = G.config_shape(cfg)
src, tgt, sizes, a, b = G.config_features(cfg, cfg)
host = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
cost = host.numpy().T
dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 1, C.c_void_p(dev.data_ptr())))
host.copy_(dev); del dev; torch.cuda.synchronize()
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20, lbfgs_memory=10)
for it in range(4):
    t0 = time.perf_counter(); c2 = G.Context.from_arrays(cost, sizes, a, b, 0.1, 0.5); t1 = time.perf_counter()
    r = c2.solve(**kw); t2 = time.perf_counter(); c2.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  solve {1e3*(t2-t1):.1f} ms (maximize {1e3*r['wall_seconds']:.1f})  close {1e3*(t3-t2):.1f} ms")
