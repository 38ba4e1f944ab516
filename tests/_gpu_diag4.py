import os, sys, time, subprocess
for buf in ['0', '100', '96', '64', '48']:
    r = subprocess.run([sys.executable, '-c', f'''
import sys, time
sys.path.insert(0, ".")
import paper_2303_07597_b200 as G
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20)
ctx.solve(**kw)
ts = []
for i in range(3):
    t = time.perf_counter(); r = ctx.solve(**kw); ts.append(time.perf_counter() - t)
kw0 = dict(kw, mode=0); ctx.solve(**kw0)
t = time.perf_counter(); r0 = ctx.solve(**kw0); t0 = time.perf_counter() - t
print("buf {buf}: fast %.1f ms  baseline %.1f ms  calls %d" % (1e3 * min(ts), 1e3 * t0, r["grad_calls"]))
'''], env=dict(os.environ, GSOT_EVAL_BUF=buf), capture_output=True, text=True)
    print(r.stdout.strip(), r.stderr.strip()[-300:])
