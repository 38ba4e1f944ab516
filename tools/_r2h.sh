for ns in 2 3 4 6; do GSOT_EVAL_CL_SLOTS=$ns GSOT_DIAG_SEQ=1 timeout 300 python tools/_gpu_solve_once.py 1 --config 5 2>&1 | grep -v 'diag] seq' | tail -2; done
GSOT_EVAL_CLUSTER=0 timeout 300 python tools/_gpu_solve_once.py 1 --config 5 2>&1 | tail -1
