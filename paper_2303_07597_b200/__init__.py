"""B200-native (sm_100a) group-sparse OT smoothed-dual solver.

Drop-in for the hot path of the reference `groupot` library (arXiv
2303.07597): the fused dual objective/gradient with upper-bound block
skipping and the lower-bound active set, inside L-BFGS. The compute lives in
lib/libgsot.so (CUDA, C ABI in include/gsot.h); `groupot` mirrors the
reference API on top of it.
"""
from . import groupot  # noqa: F401
from .groupot import *  # noqa: F401,F403

__all__ = [n for n in dir(groupot) if not n.startswith("_")]
