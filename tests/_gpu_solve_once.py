import sys
sys.path.insert(0, '.')
import paper_2303_07597_b200 as G
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
kw = dict(mode=int(sys.argv[1]) if len(sys.argv) > 1 else 1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20)
ctx.solve(**kw)
r = ctx.solve(**kw)
print('calls', r['grad_calls'])
