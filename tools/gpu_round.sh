#!/bin/bash
# One measurement round on a GPU box: smoke, GPU tests, bench (both arms).
#   bash tools/gpu_round.sh TAG [pytest -k expr]
TAG=${1:-r2}
K=${2:-}
set -x
nproc; lscpu | grep -E "Model name" ; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke $?
if [ -n "$K" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -k "$K" --durations=25 > gpurun_out/pytest_$TAG.log 2>&1; echo pytest $?
else
  timeout 1800 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_$TAG.log 2>&1; echo pytest $?
fi
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo bench $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/benchref_$TAG.log 2>&1; echo benchref $?
