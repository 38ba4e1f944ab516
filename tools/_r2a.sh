set -x
nproc; free -g; lscpu | grep -E "Model name|Socket|Thread|Core" ; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench5.log 2>&1; echo bench5 $?
timeout 300 bash tools/timeline.sh 5 > gpurun_out/r2a_tl5.log 2>&1; echo tl5 $?
timeout 300 bash tools/timeline.sh 4 > gpurun_out/r2a_tl4.log 2>&1; echo tl4 $?
