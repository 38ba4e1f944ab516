import sys, time
sys.path.insert(0, '.')
import paper_2303_07597_b200 as G
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20)
names = {0: "eval", 1: "snapshot", 2: "bounds", 3: "active", 4: "finalize", 5: "lbfgs", 6: "delta", 7: "misc"}
for mode in (1, 0):
    ctx.profile(True); ctx.solve(**dict(kw, mode=mode)); ctx.profile_reset()
    r = ctx.solve(**dict(kw, mode=mode))
    tot = 0
    for k, nm in names.items():
        ms, by, n = ctx.profile_read(k)
        if n:
            tot += ms
            print(f"mode {mode} {nm:9s} n={n:5d} total={ms:7.2f} ms  mean={1e3*ms/n:7.2f} us  GB/s={by/ms/1e6 if ms else 0:8.1f}")
    print('mode', mode, 'sum kernels %.2f ms' % tot, 'blocks frac %.3f lanes/task %.2f' % (r['eval_blocks'] / (r['grad_calls'] * ctx.L * ctx.n), r['eval_blocks'] / max(1, r['eval_tasks'])))
ctx.profile(False)
t = time.perf_counter(); r = ctx.solve(**kw); print('unprofiled solve %.1f ms' % (1e3 * (time.perf_counter() - t)))
