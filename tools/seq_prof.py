"""Diagnostic: stitch counters of the exact-order engine (gsot_seqsum.cuh)
from a -DGSOT_SEQ_PROF build: random sums, then one exact-order solve.

    GSOT_LIB=paper_2303_07597_b200/lib/libgsot_seqprof.so python tools/seq_prof.py 2
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_07597_b200 as G  # noqa: E402
from paper_2303_07597_b200 import _lib  # noqa: E402

NAMES = {7: "engine calls", 8: "leaf pieces (cta0 ch0)", 9: "warp-list pieces", 11: "CTA lists too long"}
PHASES = ["sums+scan", "barrier1", "runs+warp trees", "CTA root", "barrier2", "stitch"]
h = _lib.lib()
h.gsot_debug_seq_prof.argtypes = [C.c_void_p]
buf = (C.c_ulonglong * 16)()


def show(tag):
    h.gsot_debug_seq_prof(buf)
    n = max(1, buf[7])
    print(tag, {NAMES[k]: buf[k] for k in NAMES})
    print("   us/call:", {PHASES[i]: round(buf[i] / n / 1.9e3, 2) for i in range(6) if i != 6},
          "of which runs (chain 0):", round(buf[15] / n / 1.9e3, 2))


ctx = G.Context.from_arrays(np.full((4, 3), 0.5), [4], np.full(4, 0.25), np.full(3, 1 / 3), 1.0, 1.0)
rng = np.random.default_rng(0)
h.gsot_debug_seq_prof(buf)
for n in (3000, 20000, 150000):
    for kind in ("normal", "positive", "dot-like"):
        v = rng.normal(size=n) if kind == "normal" else rng.random(n) if kind == "positive" else \
            rng.normal(size=n) * rng.normal(size=n) * 1e-3
        got = ctx.sequential_sum(v, 0.0)
        ref = np.cumsum(np.concatenate([[0.0], v]))[-1]
        show(f"n={n} {kind} ok={got == ref}")
ctx.close()
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
gam, mu, it = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
               5: (0.1, 0.5, 300)}[cfg]
ctx = G.Context.from_config(cfg, cfg, gam, mu)
kw = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=it // 10, exact=True)
ctx.solve(**kw)
h.gsot_debug_seq_prof(buf)
t0 = time.time()
r = ctx.solve(**kw)
print(f"config {cfg}: solve {1e3 * (time.time() - t0):.1f} ms")
show("solve")
