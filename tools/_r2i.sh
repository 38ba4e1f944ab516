timeout 600 python -m pytest tests/test_gpu_exact.py -x -q 2>&1 | tail -2
for v in 0 1; do GSOT_EXACT_COLS=$v timeout 300 python tools/exact_speed.py --configs 2,5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['exact']['ms'], d['exact_kinds_ms']['eval'])"; done
