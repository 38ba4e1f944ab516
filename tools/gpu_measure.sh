#!/bin/bash
# Round measurement on one GPU box: tests, bench (both arms), ncu launch list
# + --set full captures (bench workload), dense-eval captures, all five
# configs.   bash tools/gpu_measure.sh TAG
TAG=${1:-r1h}
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo pytest $?
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke $?
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
timeout 600 python bench.py --impl reference > gpurun_out/benchref_$TAG.log 2>&1; echo benchref $?
timeout 1200 bash tools/ncu_profile.sh $TAG; echo ncu $?
timeout 900 bash tools/ncu_dense.sh $TAG > gpurun_out/ncu_dense_$TAG.log 2>&1; echo ncudense $?
timeout 1500 python tools/solve_configs.py --e2e --reps 2 --out gpurun_out/configs_$TAG.json > gpurun_out/configs_$TAG.log 2>&1; echo configs $?
