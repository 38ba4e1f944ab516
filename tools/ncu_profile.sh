set -x
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_snapshot|k_eval|k_finalize|k_two_loop|k_delta|k_bounds|k_objective" -s 40 -c 14 -o gpurun_out/prof1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
echo DONE $?
