set -x
GSOT_LIB=paper_2303_07597_b200/lib/libgsot_seqprof.so timeout 300 python tools/seq_prof.py 2 > gpurun_out/r2c_seq2.log 2>&1; echo seq2 $?
GSOT_LIB=paper_2303_07597_b200/lib/libgsot_seqprof.so timeout 300 python tools/seq_prof.py 5 > gpurun_out/r2c_seq5.log 2>&1; echo seq5 $?
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:"k_ex_direction|k_ex_cols|k_ex_scalars" -s 30 -c 3 -o gpurun_out/prof_r2c5x python tools/_gpu_solve_once.py 1 prof --config 5 --exact > gpurun_out/r2c_ncuf5x.log 2>&1; echo ncuf5x $?
