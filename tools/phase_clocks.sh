#!/bin/bash
# Diagnostic: per-phase SM cycles of k_lbfgs_step (rank 0, thread 0) over one
# fast-mode config-2 solve, from a -DGSOT_PHASE_CLOCKS build of the library.
set -e
GSOT_NVCC_DEFINES="-DGSOT_PHASE_CLOCKS" GSOT_LIB_OUT=/tmp/libgsot_diag.so python -m paper_2303_07597_b200.build > /dev/null
GSOT_LIB=/tmp/libgsot_diag.so python - <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
import paper_2303_07597_b200 as G
from paper_2303_07597_b200 import _lib
h = _lib.lib()
buf = (C.c_ulonglong * 16)()
ctx = G.Context.from_config(2, 2, 0.1, 0.5)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=20)
ctx.solve(**kw)
h.gsot_debug_phase_clocks(buf, 16)
r = ctx.solve(**kw)
h.gsot_debug_phase_clocks(buf, 16)
n = r['grad_calls']
print('calls', n, 'per-launch cycles by phase:', [round(buf[i] / max(1, r['iterations'])) for i in range(14)])
PY
