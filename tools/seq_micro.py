"""Diagnostic: engine phase clocks on synthetic vectors (-DGSOT_SEQ_PROF build).
    GSOT_LIB=paper_2303_07597_b200/lib/libgsot_seqprof.so python tools/seq_micro.py"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2303_07597_b200 as G  # noqa: E402
from paper_2303_07597_b200 import _lib  # noqa: E402

h = _lib.lib()
h.gsot_debug_seq_prof.argtypes = [C.c_void_p]
ctx = G.Context.from_arrays(np.full((4, 3), 0.5), [4], np.full(4, 0.25), np.full(3, 1 / 3), 1.0, 1.0)
rng = np.random.default_rng(0)
buf = (C.c_ulonglong * 16)()
names = ["A", "bar-A", "starts", "B", "bar-B", "C", "wait-C"]
for name, v in (("pos", rng.random(150000)), ("walk", rng.normal(size=150000)),
                ("prod", rng.normal(size=150000) * 1e-3 * rng.normal(size=150000) * 1e-5)):
    ctx.sequential_sum(v)
    h.gsot_debug_seq_prof(buf)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        r = ctx.sequential_sum(v)
    dt = (time.perf_counter() - t0) / reps
    h.gsot_debug_seq_prof(buf)
    n = max(1, buf[7])
    assert r == np.cumsum(v)[-1]
    print(f"{name}: {dt*1e6:.1f} us/call (host incl. H2D)  " +
          "  ".join(f"{nm} {buf[i] / n / 1.9e3:.2f}" for i, nm in enumerate(names)) +
          f"  C1 {buf[10] / n / 1.9e3:.2f}"
          f"  pieces/call {buf[8] / n / 8:.1f} fallbacks {buf[9] / n / 8:.2f} serial/call {buf[13] / n / 8:.1f}")
