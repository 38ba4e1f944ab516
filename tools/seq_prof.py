"""Diagnostic: engine phase clocks of one exact-order solve (CTA 0 cycles,
summed over engine calls) from a -DGSOT_SEQ_PROF build:

    GSOT_LIB=paper_2303_07597_b200/lib/libgsot_seqprof.so python tools/seq_prof.py 2
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_07597_b200 as G  # noqa: E402
from paper_2303_07597_b200 import _lib  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
gam, mu, it = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
               5: (0.1, 0.5, 300)}[cfg]
h = _lib.lib()
h.gsot_debug_seq_prof.argtypes = [C.c_void_p]
ctx = G.Context.from_config(cfg, cfg, gam, mu)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=it // 10, exact=True)
ctx.solve(**kw)
buf = (C.c_ulonglong * 16)()
h.gsot_debug_seq_prof(buf)
r = ctx.solve(**kw)
h.gsot_debug_seq_prof(buf)
n = max(1, buf[7])
names = ["A", "bar-A", "starts", "B", "bar-B", "C", "wait-C"]
print(f"config {cfg}: solve {r['wall_seconds']*1e3:.1f} ms, engine calls {buf[7]}")
for i, nm in enumerate(names):
    print(f"  {nm:7s} {buf[i] / n / 1.9e3:8.2f} us/call  total {buf[i] / 1.9e6:8.1f} ms")
print(f"  C1+bar  {buf[10] / n / 1.9e3:8.2f} us/call")
print(f"  pieces applied {buf[8]}, fallbacks {buf[9]} ({buf[10]} terms), serial tails {buf[13]} terms, "
      f"pieces emitted {buf[12]} covering {buf[11]} terms")
