"""ctypes binding of libgsot.so (include/gsot.h).

The library is the product: there is no Python or CPU fallback. Importing
this module loads lib/libgsot.so and fails loudly when it is missing; every
compute call returns GSOT_ERR_CUDA without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSOT_LIB") or os.path.join(HERE, "lib", "libgsot.so")

GSOT_OK = 0
STATUS_NAMES = {
    0: "GSOT_OK",
    1: "GSOT_ERR_DIMENSION_MISMATCH",
    2: "GSOT_ERR_NEGATIVE_COST",
    3: "GSOT_ERR_MARGINAL_NOT_NORMALIZED",
    4: "GSOT_ERR_PARTITION_MISMATCH",
    5: "GSOT_ERR_INVALID_ARGUMENT",
    6: "GSOT_ERR_RHO_OUT_OF_RANGE",
    7: "GSOT_ERR_AUDIT_VIOLATION",
    8: "GSOT_ERR_CUDA",
    9: "GSOT_ERR_OUT_OF_MEMORY",
    10: "GSOT_ERR_STATE",
}


class ErrorDetail(C.Structure):
    _fields_ = [("status", C.c_int32), ("row", C.c_int64), ("col", C.c_int64),
                ("value", C.c_double), ("which", C.c_char), ("index", C.c_int64)]


class CallStats(C.Structure):
    _fields_ = [("in_active", C.c_int64), ("skipped", C.c_int64), ("unskipped", C.c_int64),
                ("upper_bounds", C.c_int64)]


class SolverOptionsC(C.Structure):
    _fields_ = [("snapshot_interval", C.c_int32), ("grad_tol", C.c_double),
                ("max_outer_loops", C.c_int32), ("lbfgs_memory", C.c_int32),
                ("mode", C.c_int32), ("upper_bound_offset", C.c_double), ("flags", C.c_int32)]


class SolveResultC(C.Structure):
    _fields_ = [("objective", C.c_double), ("iterations", C.c_int32), ("chunks", C.c_int32),
                ("converged", C.c_int32), ("line_search_failed", C.c_int32),
                ("blocks_in_active_set", C.c_int64), ("blocks_skipped", C.c_int64),
                ("blocks_unskipped", C.c_int64), ("upper_bounds_evaluated", C.c_int64),
                ("outer_loops", C.c_int64), ("grad_calls", C.c_int64),
                ("wall_seconds", C.c_double), ("audit_skip_checks", C.c_int64),
                ("audit_active_checks", C.c_int64), ("audit_column_compares", C.c_int64),
                ("audit_gradient_calls", C.c_int64), ("eval_blocks", C.c_int64),
                ("eval_tasks", C.c_int64)]


# Every entry point of include/gsot.h with its C signature.
class PlanDiagC(C.Structure):
    """gsot_plan_diag (PlanDiagnostics, dual.hpp:130-135)."""
    _fields_ = [("marginal_res_a", C.c_double), ("marginal_res_b", C.c_double),
                ("group_sparsity", C.c_double), ("mass", C.c_double)]


_vp, _dp, _ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32)
SIGNATURES = {
    "gsot_last_error": (C.c_char_p, []),
    "gsot_last_error_detail": (C.c_int, [C.POINTER(ErrorDetail)]),
    "gsot_version": (C.c_char_p, []),
    "gsot_params_from_rho": (C.c_int, [C.c_double, C.c_double, _dp, _dp]),
    "gsot_create": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, C.c_int32, _vp, _vp, C.c_double,
                              C.c_double, C.POINTER(_vp)]),
    "gsot_create_device": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, C.c_int32, _vp, _vp,
                                     C.c_double, C.c_double, C.POINTER(_vp)]),
    "gsot_create_shard": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, C.c_int32, _vp, _vp,
                                    C.c_double, C.c_double, C.POINTER(_vp)]),
    "gsot_create_shard_device": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, C.c_int32, _vp, _vp,
                                           C.c_double, C.c_double, C.POINTER(_vp)]),
    "gsot_destroy": (None, [_vp]),
    "gsot_cache_clear": (C.c_int64, []),
    "gsot_set_params": (C.c_int, [_vp, C.c_double, C.c_double]),
    "gsot_set_upper_bound_offset": (C.c_int, [_vp, C.c_double]),
    "gsot_sequential_sum": (C.c_int, [_vp, _vp, C.c_int64, C.c_double, _dp]),
    "gsot_shape": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _ip,
                             C.POINTER(C.c_int64)]),
    "gsot_eval": (C.c_int, [_vp, _vp, C.c_int, _dp, _vp, C.POINTER(CallStats)]),
    "gsot_eval_device": (C.c_int, [_vp, _vp, C.c_int, _dp, _vp, C.POINTER(CallStats)]),
    "gsot_init_snapshot": (C.c_int, [_vp, _vp]),
    "gsot_refresh": (C.c_int, [_vp, _vp, C.c_int]),
    "gsot_snapshot_norms": (C.c_int, [_vp, _vp, _vp, _vp]),
    "gsot_active_set": (C.c_int, [_vp, _vp, C.POINTER(C.c_int64)]),
    "gsot_block_mask": (C.c_int, [_vp, _vp, _vp]),
    "gsot_plan_columns": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, _vp]),
    "gsot_plan_diagnostics": (C.c_int, [_vp, _vp, C.POINTER(PlanDiagC)]),
    "gsot_primal_objective": (C.c_int, [_vp, _vp, _dp]),
    "gsot_default_solver_options": (None, [C.POINTER(SolverOptionsC)]),
    "gsot_solve": (C.c_int, [_vp, C.POINTER(SolverOptionsC), _vp, C.POINTER(SolveResultC), _vp,
                             C.c_int64]),
    "gsot_config_shape": (C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _ip,
                                    C.POINTER(C.c_int64)]),
    "gsot_config_features": (C.c_int, [C.c_int32, C.c_uint64, _vp, _vp, _vp, _vp, _vp]),
    "gsot_cost_matrix_device": (C.c_int, [_vp, C.c_int64, _vp, C.c_int64, C.c_int64, C.c_int,
                                          _vp]),
    "gsot_create_config": (C.c_int, [C.c_int32, C.c_uint64, C.c_double, C.c_double,
                                     C.POINTER(_vp)]),
    "gsot_create_features": (C.c_int, [_vp, C.c_int64, _vp, C.c_int64, C.c_int64, _vp, C.c_int32,
                                       _vp, _vp, C.c_int, C.c_double, C.c_double,
                                       C.POINTER(_vp)]),
    "gsot_profile_enable": (C.c_int, [_vp, C.c_int]),
    "gsot_profile_read": (C.c_int, [_vp, C.c_int, _dp, _dp, C.POINTER(C.c_int64)]),
    "gsot_profile_reset": (C.c_int, [_vp]),
    "gsot_kernel_launches": (C.c_int64, [_vp]),
    "gsot_set_device": (C.c_int, [C.c_int32]),
    "gsot_timer": (C.c_int, [_vp, C.c_int, _dp]),
    "gsot_comm_unique_id": (C.c_int, [_vp]),
    "gsot_comm_attach_nccl": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32]),
    "gsot_comm_attach_host": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp]),
    "gsot_comm_detach": (C.c_int, [_vp]),
}

# gsot_allreduce_fn (include/gsot.h): in-place reduction of host doubles.
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_int32, C.c_void_p)

_lib = None


def lib() -> C.CDLL:
    """Load libgsot.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2303_07597_b200.build` "
                "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def last_error() -> tuple[str, ErrorDetail]:
    h = lib()
    d = ErrorDetail()
    h.gsot_last_error_detail(C.byref(d))
    msg = h.gsot_last_error()
    return (msg.decode() if msg else ""), d
