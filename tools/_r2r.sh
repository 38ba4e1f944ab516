# round-2 r: device-resident sharded solve tests, skip-bound study, sharded N=1 speed
set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/pytest_r2r.log 2>&1; echo pytest $?
timeout 600 python -c "
import sys, json; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, paper_2303_07597_b200 as G
for cfg in (2, 5):
    gamma, mu, iters = bench.CONFIGS[cfg]
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    kw = bench.solve_kw(iters); ctx.solve(**kw)
    h = bench.timed_solves(ctx, kw, 3); ctx.close(); G.cache_clear()
    r = bench.sharded_n1(cfg, h['ms']/3, h['x'], 3)
    print(json.dumps({'cfg': cfg, 'single_ms': h['ms']/3, **r}), flush=True)
" > gpurun_out/shard1_r2r.log 2>&1; echo shard1 $?
timeout 600 python tools/skip_bounds.py --config 5 > gpurun_out/skip5_r2r.log 2>&1; echo skip5 $?
timeout 600 python tools/skip_bounds.py --config 4 > gpurun_out/skip4_r2r.log 2>&1; echo skip4 $?
timeout 300 python tools/skip_bounds.py --config 2 > gpurun_out/skip2_r2r.log 2>&1; echo skip2 $?
