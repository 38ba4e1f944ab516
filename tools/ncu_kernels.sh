#!/bin/bash
# Warm-cache per-kernel durations of one fast-mode config-2 solve (the
# second solve of the process): python tools/_gpu_solve_once.py
TAG=${1:-k}
python tools/_gpu_solve_once.py > gpurun_out/solve_once_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python tools/_gpu_solve_once.py 1 prof > gpurun_out/ncu_$TAG.log 2>&1
echo DONE $?
