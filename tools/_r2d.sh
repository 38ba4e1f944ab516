set -x
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q --durations=10 > gpurun_out/r2d_exact_tests.log 2>&1; echo exacttests $?
timeout 600 python tools/exact_speed.py --configs 2,5 > gpurun_out/r2d_exact.log 2>&1; echo exact $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r2d5x.csv python tools/_gpu_solve_once.py 1 prof --config 5 --exact > gpurun_out/r2d_ncul5x.log 2>&1; echo ncul5x $?
