#!/bin/bash
# ncu evidence for profiles/: launch list (device time per kernel, cold-cache,
# serialised) and one --set full capture of the hot kernels. Run on the GPU box
# only after the same bench command exited 0 without ncu.
set -x
TAG=${1:-r1}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_snapshot|k_eval|k_finalize|k_lbfgs_step|k_screen|k_delta|k_publish" -s 400 -c 16 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_f_$TAG.log 2>&1
echo DONE $?
