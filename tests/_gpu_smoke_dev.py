import sys, time, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2303_07597_b200 as G
from oracle_bindings import Oracle, Problem
o = Oracle()
rng = np.random.default_rng(0)
m, n, sizes = 37, 45, [5, 1, 8, 3, 12, 8]
cost = rng.uniform(0, 2, (m, n))
a = np.full(m, 1/m); b = np.full(n, 1/n)
for gamma, mu in [(1.0, 0.1), (0.5, 0.8), (0.3, 2.0)]:
    p = Problem(cost, np.array(sizes), a, b, gamma, mu)
    ctx = G.Context.from_arrays(cost, sizes, a, b, gamma, mu)
    x = np.concatenate([rng.uniform(-0.5, 2, m), rng.uniform(-0.5, 2, n)])
    obj, g, st = ctx.eval(x)
    oo = o.objective(p, x[:m], x[m:]); ga, gb = o.gradient(p, x[:m], x[m:])
    print('obj', obj, oo, abs(obj-oo)/abs(oo), 'grad', np.max(np.abs(g - np.concatenate([ga, gb]))))
    pl = ctx.plan_columns(x, 0, n); po = o.plan(p, x[:m], x[m:])
    print('plan bitwise', np.array_equal(pl, po))
    ctx.init_snapshot(np.zeros(m+n)); ctx.refresh(x*0.9, True); 
    z,k,oo2 = ctx.snapshot_norms(); zo,ko,oo3 = o.snapshot(p, x[:m]*0.9, x[m:]*0.9)
    print('snapshot bitwise', np.array_equal(z,zo), np.array_equal(k,ko), np.array_equal(oo2,oo3))
    mem, cnt = ctx.active_set(); memo, cnto = o.active_set(p, np.zeros(m), np.zeros(n), x[:m]*0.9, x[m:]*0.9)
    print('active', cnt, cnto, np.array_equal(mem, memo.astype(bool)))
    obj2, g2, st2 = ctx.eval(x, screened=True)
    gao, gbo, cnto2, _ = o.fast_gradient(p, x[:m]*0.9, x[m:]*0.9, memo, x[:m], x[m:])
    print('screened==dense', obj2 == obj, np.array_equal(g2, g), st2, cnto2)
    for mode in [0, 1, 2, 3]:
        t = time.time(); r = ctx.solve(mode=mode, max_outer_loops=20, history_cap=10000); t1 = time.time()-t
        ro = o.solve(p, mode=mode, max_outer_loops=20)
        print('solve', mode, r['iterations'], ro['iterations'], r['grad_calls'], ro['grad_calls'], r['objective'], ro['objective'],
              np.max(np.abs(r['x']-ro['x'])), (r['history']==ro['history']).all() if r['history'].shape==ro['history'].shape else 'shape', '%.3fs'%t1)
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
print('cfg2 ctx bytes', ctx.device_bytes)
t=time.time(); r = ctx.solve(mode=1, max_outer_loops=20, grad_tol=1e-12); print('cfg2 solve', r['iterations'], r['grad_calls'], r['objective'], time.time()-t)
t=time.time(); r = ctx.solve(mode=0, max_outer_loops=20, grad_tol=1e-12); print('cfg2 solve base', r['iterations'], r['grad_calls'], r['objective'], time.time()-t)
