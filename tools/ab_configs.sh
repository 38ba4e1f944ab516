#!/bin/bash
# A/B of solve times on one box: the library built from HEAD
# (paper_2303_07597_b200/lib/libgsot_head.so, see below) against the working
# tree's build.  bash tools/ab_configs.sh CONFIGS TAG
# Build the A side here first:
#   git archive HEAD paper_2303_07597_b200 include | tar -x -C /tmp/h && (cd /tmp/h &&
#   GSOT_LIB_OUT=$PWD/paper_2303_07597_b200/lib/libgsot_head.so python -m paper_2303_07597_b200.build)
CFG=${1:-2,4,5}
TAG=${2:-ab}
GSOT_LIB=paper_2303_07597_b200/lib/libgsot_head.so timeout 600 python tools/solve_configs.py --configs $CFG --out gpurun_out/${TAG}_A.json > gpurun_out/${TAG}_A.log 2>&1
timeout 600 python tools/solve_configs.py --configs $CFG --out gpurun_out/${TAG}_B.json > gpurun_out/${TAG}_B.log 2>&1
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
def load(s):
    out = {}
    for line in open(f"gpurun_out/{tag}_{s}.log"):
        if line.startswith("{"):
            d = json.loads(line); out[d["config"]] = d
    return out
a, b = load("A"), load("B")
for c in sorted(a):
    if c in b:
        print(f"cfg{c}: fast {a[c]['fast']['solve_ms']:.1f} -> {b[c]['fast']['solve_ms']:.1f} ms, "
              f"baseline {a[c]['baseline']['solve_ms']:.1f} -> {b[c]['baseline']['solve_ms']:.1f} ms")
PY
