#!/bin/bash
# A/B of solve times on one box with the same library under two environment
# settings:  bash tools/ab_env.sh CONFIGS TAG "ENV_A" "ENV_B"
CFG=${1:-3}
TAG=${2:-abenv}
env $3 timeout 900 python tools/solve_configs.py --configs $CFG --out gpurun_out/${TAG}_A.json > gpurun_out/${TAG}_A.log 2>&1
env $4 timeout 900 python tools/solve_configs.py --configs $CFG --out gpurun_out/${TAG}_B.json > gpurun_out/${TAG}_B.log 2>&1
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
def load(s):
    out = {}
    for line in open(f"gpurun_out/{tag}_{s}.log"):
        if line.startswith("{"):
            d = json.loads(line); out[d["config"]] = d
    return out
A, B = load("A"), load("B")
for c in sorted(A):
    if c in B:
        print(f"cfg{c}: fast {A[c]['fast']['solve_ms']:.1f} -> {B[c]['fast']['solve_ms']:.1f} ms, "
              f"baseline {A[c]['baseline']['solve_ms']:.1f} -> {B[c]['baseline']['solve_ms']:.1f} ms")
PY
