#!/bin/bash
# Diagnostic: average in-graph kernel timeline of one fast-mode config-2 solve
# (first block entry / last block exit per kernel, offsets from the first
# kernel entry of each device sequence; globaltimer), from a
# -DGSOT_PHASE_CLOCKS build of the library.
set -e
GSOT_NVCC_DEFINES="-DGSOT_PHASE_CLOCKS" GSOT_LIB_OUT=/tmp/libgsot_diag.so python -m paper_2303_07597_b200.build > /dev/null
GSOT_TIMELINE=1 GSOT_LIB=/tmp/libgsot_diag.so python - "$@" <<'PY'
import ctypes as C, sys
sys.path.insert(0, '.')
import paper_2303_07597_b200 as G
from paper_2303_07597_b200 import _lib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
gam, mu, it = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200), 5: (0.1, 0.5, 300)}[cfg]
h = _lib.lib()
ctx = G.Context.from_config(cfg, cfg, gam, mu)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=it // 10)
ctx.solve(**kw)
buf = (C.c_ulonglong * 64)()
h.gsot_debug_timeline(ctx._h, buf)
base = list(buf)
r = ctx.solve(**kw)
h.gsot_debug_timeline(ctx._h, buf)
names = ['screen', 'eval', 'finalize', 'publish', 'step', 'axpy', 'delta', 'snapshot']
seqs = buf[63] - base[63]
print(f'config {cfg}: sequences {seqs}, wall {r["wall_seconds"]*1e3:.2f} ms, calls {r["grad_calls"]}')
for k, nm in enumerate(names):
    n = buf[16 + 4 * k + 2] - base[16 + 4 * k + 2]
    if n == 0:
        continue
    s = (buf[16 + 4 * k] - base[16 + 4 * k]) / n / 1e3
    e = (buf[16 + 4 * k + 1] - base[16 + 4 * k + 1]) / n / 1e3
    print(f'  {nm:9s} n={n:4d}  start {s:7.2f} us  end {e:7.2f} us  window {e - s:6.2f} us')
ns = buf[57] - base[57]
if ns:
    print(f'  sparse evals (< 40 us): n={ns}  eval window {(buf[56] - base[56]) / ns / 1e3:.2f} us  '
          f'sequence span {(buf[58] - base[58]) / ns / 1e3:.2f} us')
    for k, nm in enumerate(names[:4]):
        s = (buf[48 + 2 * k] - base[48 + 2 * k]) / ns / 1e3
        e = (buf[49 + 2 * k] - base[49 + 2 * k]) / ns / 1e3
        print(f'    sparse {nm:9s} start {s:7.2f} us  end {e:7.2f} us  window {e - s:6.2f} us')
    nst = buf[61] - base[61]
    if nst:
        s = (buf[59] - base[59]) / nst / 1e3
        e = (buf[60] - base[60]) / nst / 1e3
        print(f'    sparse step      start {s:7.2f} us  end {e:7.2f} us  window {e - s:6.2f} us (n={nst})')
PY
