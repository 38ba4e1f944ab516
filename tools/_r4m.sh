# round-2 measurement 4a (final of the round): GPU tests, bench (both arms), launch lists (config 5 fast + exact),
# full captures of the headline solve's k_eval (near-dense + screened)
set -x
nproc; lscpu | grep -E "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke_r4m.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_r4m.log 2>&1; echo pytest $?
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r4m.log 2>&1; echo bench $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/benchref_r4m.log 2>&1; echo benchref $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r4m5.csv python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/ncul_r4m5.log 2>&1; echo ncul5 $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r4m5x.csv python tools/_gpu_solve_once.py 1 prof --config 5 --exact > gpurun_out/ncul_r4m5x.log 2>&1; echo ncul5x $?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_eval" -s 15 -c 1 -o gpurun_out/prof_r4m5_dense python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/ncuf_r4m5a.log 2>&1; echo ncufa $?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_eval" -s 150 -c 1 -o gpurun_out/prof_r4m5_screened python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/ncuf_r4m5b.log 2>&1; echo ncufb $?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_snapshot_walk" -s 5 -c 1 -o gpurun_out/prof_r4m5_snap python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/ncuf_r4m5c.log 2>&1; echo ncufc $?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_screen" -s 150 -c 1 -o gpurun_out/prof_r4m5_screen python tools/_gpu_solve_once.py 1 prof --config 5 > gpurun_out/ncuf_r4m5d.log 2>&1; echo ncufd $?
