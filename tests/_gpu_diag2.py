import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2303_07597_b200 as G
from oracle_bindings import Oracle, Problem
o = Oracle(); g = np.load('tests/golden/reference_golden.npz')
for name, pi in [('ragged', 1), ('synth', 1), ('ragged', 2)]:
    gamma, mu = g[f'{name}/p{pi}/params']
    p = Problem(g[f'{name}/cost'], g[f'{name}/sizes'], g[f'{name}/a'], g[f'{name}/b'], float(gamma), float(mu))
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    ro = o.solve(p, mode=0, max_outer_loops=20, grad_tol=1e-12, trace=400)
    tr = ro['trace']
    print(name, pi, 'oracle iters', ro['iterations'], 'obj', ro['objective'])
    for k in [1, 2, 3, 5, 8, 12, 16, 20]:
        r = ctx.solve(mode=0, max_outer_loops=k, grad_tol=1e-12)
        it = r['iterations']
        if it < len(tr):
            dx = np.max(np.abs(r['x'] - tr[it])); sc = np.max(np.abs(tr[it]))
            plan = ctx.plan_columns(r['x'], 0, p.n); po = o.plan(p, tr[it][:p.m], tr[it][p.m:])
            print('  chunks', k, 'iters', it, 'max|dx|', '%.3e' % dx, 'scale %.3e' % sc, 'plan diff %.3e' % np.max(np.abs(plan - po)), 'calls', r['grad_calls'])
    r7 = ctx.solve(mode=1, max_outer_loops=20, grad_tol=1e-7)
    ro7 = o.solve(p, mode=1, max_outer_loops=20, grad_tol=1e-7)
    plan = ctx.plan_columns(r7['x'], 0, p.n); po = o.plan(p, ro7['x'][:p.m], ro7['x'][p.m:])
    print('  tol1e-7: gpu iters', r7['iterations'], 'conv', r7['converged'], 'oracle iters', ro7['iterations'], ro7['converged'], 'plan diff %.3e' % np.max(np.abs(plan-po)), 'plan max %.3e' % np.max(po), 'obj rel %.3e' % abs(r7['objective']/ro7['objective']-1))
