# round-2 measurement b: parity horizon, exact-mode breakdown, config-5 launch list + full captures
set -x
timeout 900 python tools/parity_horizon.py --configs 1,2 > gpurun_out/r2b_horizon.log 2>&1; echo horizon $?
timeout 600 python tools/exact_speed.py --configs 2,5 > gpurun_out/r2b_exact.log 2>&1; echo exact $?
python tools/_gpu_solve_once.py 1 --config 5 > gpurun_out/r2b_once5.log 2>&1; echo once5 $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r2b5.csv python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/r2b_ncul5.log 2>&1; echo ncul5 $?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_eval|k_snapshot" -s 2 -c 3 -o gpurun_out/prof_r2b5a python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/r2b_ncuf5a.log 2>&1; echo ncuf5a $?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_eval" -s 150 -c 2 -o gpurun_out/prof_r2b5b python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/r2b_ncuf5b.log 2>&1; echo ncuf5b $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r2b5x.csv python tools/_gpu_solve_once.py 1 prof --config 5 --exact > gpurun_out/r2b_ncul5x.log 2>&1; echo ncul5x $?
