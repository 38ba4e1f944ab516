#!/bin/bash
# --set full on selected kernels of the second fast-mode config-2 solve
# (the solve bracketed by cudaProfilerStart/Stop in tools/_gpu_solve_once.py).
#   bash tools/ncu_full.sh TAG KERNEL_REGEX [SKIP] [COUNT]
TAG=${1:-f}
REGEX=${2:-k_eval}
python tools/_gpu_solve_once.py > gpurun_out/solve_once_$TAG.log 2>&1 && \
ncu --set full --import-source on --cache-control none --clock-control none --profile-from-start off -k regex:"$REGEX" -s ${3:-100} -c ${4:-2} -o gpurun_out/prof_$TAG python tools/_gpu_solve_once.py 1 prof > gpurun_out/ncu_$TAG.log 2>&1
echo DONE $?
