"""B200-native (sm_100a) group-sparse OT smoothed-dual solver.

Drop-in for the hot path of the reference `groupot` library (arXiv
2303.07597): the fused dual objective/gradient with upper-bound block
skipping and the lower-bound active set, inside L-BFGS. The compute lives in
lib/libgsot.so (CUDA, C ABI in include/gsot.h); `groupot` mirrors the
reference API on top of it.
"""
from . import data_io, groupot  # noqa: F401
from .data_io import (InconsistentDimension, LabeledSamples, MissingLabelColumn,  # noqa: F401
                      ParseError, UnlabeledSamples, load_csv, make_device_instance,
                      make_instance, partition_from_labels, read_csv, save_matrix_csv,
                      save_source_csv, save_target_csv)
from .groupot import *  # noqa: F401,F403

__all__ = [n for n in dir(groupot) if not n.startswith("_")] + [
    "InconsistentDimension", "LabeledSamples", "MissingLabelColumn", "ParseError",
    "UnlabeledSamples", "load_csv", "make_device_instance", "make_instance",
    "partition_from_labels", "read_csv", "save_matrix_csv", "save_source_csv", "save_target_csv"]
