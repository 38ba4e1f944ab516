set -x
timeout 900 python tools/skip_bounds.py --config 5 > gpurun_out/skip5_r2s.log 2>&1; echo skip5 $?
timeout 600 python tools/skip_bounds.py --config 2 > gpurun_out/skip2_r2s.log 2>&1; echo skip2 $?
timeout 600 python tools/skip_bounds.py --config 4 > gpurun_out/skip4_r2s.log 2>&1; echo skip4 $?
