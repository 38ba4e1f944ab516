# timing diagnostics (dev only)
import sys, time
sys.path.insert(0, '.')
import paper_2303_07597_b200 as G
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20)
for prof in (False, True, False):
    ctx.profile(prof)
    ts = []
    for i in range(4):
        t = time.perf_counter(); r = ctx.solve(**kw); ts.append(time.perf_counter() - t)
    print('profile', prof, ['%.1f' % (1e3 * x) for x in ts], r['grad_calls'])
for mode in (0, 2):
    ts = []
    for i in range(3):
        t = time.perf_counter(); r = ctx.solve(**dict(kw, mode=mode)); ts.append(time.perf_counter() - t)
    print('mode', mode, ['%.1f' % (1e3 * x) for x in ts], r['grad_calls'])
ctx.close()
for i in range(2):
    t = time.perf_counter(); c2 = G.Context.from_config(2, 2, 0.1, 0.5); t1 = time.perf_counter()
    r = c2.solve(**kw); t2 = time.perf_counter(); r = c2.solve(**kw); t3 = time.perf_counter()
    print('new ctx: create %.1f ms, first solve %.1f ms, second %.1f ms' % (1e3*(t1-t), 1e3*(t2-t1), 1e3*(t3-t2)))
    c2.close()
