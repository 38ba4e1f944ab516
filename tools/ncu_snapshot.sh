#!/bin/bash
# ncu of one k_snapshot launch per config (the refresh pass of the fast solve)
#   bash tools/ncu_snapshot.sh TAG
TAG=${1:-snap}
for c in 2 3 4 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread --clock-control none --profile-from-start off -k regex:k_snapshot -s 1 -c 1 --csv python tools/_gpu_solve_cfg.py $c 1 > gpurun_out/${TAG}_c$c.csv 2>&1
  echo c$c $?
done
