#!/bin/bash
# --set full captures of dense (or near-dense) k_eval launches:
#   config 2 in baseline mode (every call dense), configs 4 and 5 early fast-mode calls.
#   bash tools/ncu_dense.sh TAG
TAG=${1:-d}
NCU="ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_eval"
python tools/_gpu_solve_once.py 0 prof > gpurun_out/dense2_$TAG.log 2>&1 && \
  $NCU -s 6 -c 2 -o gpurun_out/prof_${TAG}_c2 python tools/_gpu_solve_once.py 0 prof >> gpurun_out/dense2_$TAG.log 2>&1
echo c2 $?
for c in 4 5; do
  $NCU -s 4 -c 2 -o gpurun_out/prof_${TAG}_c$c python tools/_gpu_solve_cfg.py $c 1 > gpurun_out/dense${c}_$TAG.log 2>&1
  echo c$c $?
done
