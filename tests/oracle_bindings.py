"""ctypes bindings to the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> oracle/_build/libgsot_oracle.so, the plain-C restatement.
* ``RefLib``  -> oracle/_ref/libgroupot_ref.so, the unmodified reference
  headers compiled against the Eigen shim.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU arms load
these; the product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libgsot_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libgroupot_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@dataclass
class Problem:
    """Column-major cost + marginals + group sizes (reference layout)."""

    cost: np.ndarray  # (m, n) float64, any order; stored Fortran-contiguous
    sizes: np.ndarray  # (L,) int32
    a: np.ndarray
    b: np.ndarray
    gamma: float
    mu: float

    def __post_init__(self):
        self.cost = np.asfortranarray(self.cost, dtype=np.float64)
        self.sizes = np.ascontiguousarray(self.sizes, dtype=np.int32)
        self.a = np.ascontiguousarray(self.a, dtype=np.float64)
        self.b = np.ascontiguousarray(self.b, dtype=np.float64)

    @property
    def m(self) -> int:
        return self.cost.shape[0]

    @property
    def n(self) -> int:
        return self.cost.shape[1]

    @property
    def L(self) -> int:
        return len(self.sizes)

    @property
    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int32)

    def cost_flat(self) -> np.ndarray:
        return np.ascontiguousarray(self.cost.reshape(-1, order="F"))


class _GoProblem(C.Structure):
    _fields_ = [
        ("cost", C.c_void_p),
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("L", C.c_int32),
        ("sizes", C.c_void_p),
        ("offsets", C.c_void_p),
        ("a", C.c_void_p),
        ("b", C.c_void_p),
        ("gamma", C.c_double),
        ("mu", C.c_double),
    ]


class _GoSolverOptions(C.Structure):
    _fields_ = [
        ("snapshot_interval", C.c_int),
        ("grad_tol", C.c_double),
        ("max_outer_loops", C.c_int),
        ("lbfgs_memory", C.c_int),
        ("mode", C.c_int),
    ]


class _GoSolveResult(C.Structure):
    _fields_ = [
        ("objective", C.c_double),
        ("iterations", C.c_int),
        ("chunks", C.c_int),
        ("converged", C.c_int),
        ("line_search_failed", C.c_int),
        ("blocks_in_active_set", C.c_int64),
        ("blocks_skipped", C.c_int64),
        ("blocks_unskipped", C.c_int64),
        ("upper_bounds_evaluated", C.c_int64),
        ("outer_loops", C.c_int64),
        ("grad_calls", C.c_int64),
        ("wall_seconds", C.c_double),
        ("audit_skip_checks", C.c_int64),
        ("audit_active_checks", C.c_int64),
        ("audit_column_compares", C.c_int64),
        ("audit_gradient_calls", C.c_int64),
    ]


class _GoRng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("mti", C.c_int), ("has_spare", C.c_int),
                ("spare", C.c_double)]


class Oracle:
    """Plain-C restatement of the reference path (oracle/gsot_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        self.lib = C.CDLL(path)
        L = self.lib
        L.go_dual_objective.restype = C.c_double
        L.go_pos_part_norm.restype = C.c_double
        L.go_pos_part_norm.argtypes = [_dp, C.c_int]
        L.go_build_active_set.restype = C.c_int64
        L.go_rng_next.restype = C.c_uint64
        L.go_rng_uniform01.restype = C.c_double
        L.go_rng_normal.restype = C.c_double
        L.go_rng_index.restype = C.c_uint64
        L.go_rng_index.argtypes = [C.c_void_p, C.c_uint64]
        L.go_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.go_compensated_sum.restype = C.c_double
        L.go_compensated_sum.argtypes = [_dp, C.c_int64]

    def _gp(self, p: Problem):
        keep = (p.cost_flat(), p.sizes, p.offsets, p.a, p.b)
        gp = _GoProblem(keep[0].ctypes.data, p.m, p.n, p.L, keep[1].ctypes.data,
                        keep[2].ctypes.data, keep[3].ctypes.data, keep[4].ctypes.data,
                        p.gamma, p.mu)
        return gp, keep

    def validate(self, p: Problem):
        gp, keep = self._gp(p)
        row, col, idx = C.c_int64(-2), C.c_int64(-2), C.c_int64(-2)
        which = C.c_char(b"?")
        st = self.lib.go_validate(C.byref(gp), C.byref(row), C.byref(col), C.byref(which),
                                  C.byref(idx))
        return st, dict(row=row.value, col=col.value, which=which.value.decode(),
                        index=idx.value)

    def objective(self, p: Problem, alpha, beta) -> float:
        gp, keep = self._gp(p)
        al = np.ascontiguousarray(alpha, np.float64)
        be = np.ascontiguousarray(beta, np.float64)
        return self.lib.go_dual_objective(C.byref(gp), al.ctypes.data_as(C.c_void_p),
                                          be.ctypes.data_as(C.c_void_p))

    def gradient(self, p: Problem, alpha, beta):
        gp, keep = self._gp(p)
        al = np.ascontiguousarray(alpha, np.float64)
        be = np.ascontiguousarray(beta, np.float64)
        ga = np.empty(p.m)
        gb = np.empty(p.n)
        self.lib.go_dual_gradient(C.byref(gp), al.ctypes.data_as(C.c_void_p),
                                  be.ctypes.data_as(C.c_void_p), ga.ctypes.data_as(C.c_void_p),
                                  gb.ctypes.data_as(C.c_void_p))
        return ga, gb

    def plan(self, p: Problem, alpha, beta) -> np.ndarray:
        gp, keep = self._gp(p)
        al = np.ascontiguousarray(alpha, np.float64)
        be = np.ascontiguousarray(beta, np.float64)
        out = np.empty(p.m * p.n)
        self.lib.go_recover_plan(C.byref(gp), al.ctypes.data_as(C.c_void_p),
                                 be.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
        return out.reshape(p.m, p.n, order="F")

    def plan_diagnostics(self, p: Problem, plan) -> np.ndarray:
        """dual.hpp:139-169 on an m x n plan: [res_a, res_b, group_sparsity, mass]."""
        gp, keep = self._gp(p)
        pl = np.asfortranarray(plan, np.float64)
        out = np.empty(4)
        self.lib.go_plan_diagnostics(C.byref(gp), pl.ctypes.data_as(C.c_void_p),
                                     out.ctypes.data_as(C.c_void_p))
        return out

    def snapshot(self, p: Problem, alpha, beta):
        gp, keep = self._gp(p)
        al = np.ascontiguousarray(alpha, np.float64)
        be = np.ascontiguousarray(beta, np.float64)
        z, k, o = (np.empty(p.L * p.n) for _ in range(3))
        self.lib.go_take_snapshot(C.byref(gp), al.ctypes.data_as(C.c_void_p),
                                  be.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p),
                                  k.ctypes.data_as(C.c_void_p), o.ctypes.data_as(C.c_void_p))
        f = lambda v: v.reshape(p.L, p.n, order="F")  # noqa: E731
        return f(z), f(k), f(o)

    def delta_norms(self, p: Problem, alpha, beta, alpha_s, beta_s):
        gp, keep = self._gp(p)
        arrs = [np.ascontiguousarray(v, np.float64) for v in (alpha, beta, alpha_s, beta_s)]
        dpos, dfull, dneg, sg = (np.empty(p.L) for _ in range(4))
        db = np.empty(p.n)
        self.lib.go_delta_norms(C.byref(gp), *[v.ctypes.data_as(C.c_void_p) for v in arrs],
                                *[v.ctypes.data_as(C.c_void_p) for v in (dpos, dfull, dneg, sg, db)])
        return dpos, dfull, dneg, sg, db

    def active_set(self, p: Problem, alpha_s, beta_s, alpha, beta):
        z, k, o = self.snapshot(p, alpha_s, beta_s)
        gp, keep = self._gp(p)
        kf = np.asfortranarray(k).reshape(-1, order="F").copy()
        of = np.asfortranarray(o).reshape(-1, order="F").copy()
        arrs = [np.ascontiguousarray(v, np.float64) for v in (alpha_s, beta_s)]
        cur = [np.ascontiguousarray(v, np.float64) for v in (alpha, beta)]
        member = np.zeros(p.L * p.n, np.uint8)
        cnt = self.lib.go_build_active_set(C.byref(gp), arrs[0].ctypes.data_as(C.c_void_p),
                                           arrs[1].ctypes.data_as(C.c_void_p),
                                           kf.ctypes.data_as(C.c_void_p),
                                           of.ctypes.data_as(C.c_void_p),
                                           cur[0].ctypes.data_as(C.c_void_p),
                                           cur[1].ctypes.data_as(C.c_void_p),
                                           member.ctypes.data_as(C.c_void_p))
        return member.reshape(p.L, p.n, order="F"), cnt

    def fast_gradient(self, p: Problem, alpha_s, beta_s, member, alpha, beta, ub_offset=0.0):
        """Gradient call of FastGradDispatcher with the snapshot at
        (alpha_s, beta_s) and the given active set (L x n or None)."""
        z, k, o = self.snapshot(p, alpha_s, beta_s)
        gp, keep = self._gp(p)
        zf = np.asfortranarray(z).reshape(-1, order="F").copy()
        mem = None
        if member is not None:
            mem = np.asfortranarray(member.astype(np.uint8)).reshape(-1, order="F").copy()
        arrs = [np.ascontiguousarray(v, np.float64) for v in (alpha_s, beta_s, alpha, beta)]
        ga, gb = np.empty(p.m), np.empty(p.n)
        cnt = np.zeros(4, np.int64)
        path = np.zeros(p.L * p.n, np.uint8)
        self.lib.go_fast_gradient(
            C.byref(gp), arrs[0].ctypes.data_as(C.c_void_p), arrs[1].ctypes.data_as(C.c_void_p),
            zf.ctypes.data_as(C.c_void_p),
            None if mem is None else mem.ctypes.data_as(C.c_void_p), C.c_double(ub_offset),
            arrs[2].ctypes.data_as(C.c_void_p), arrs[3].ctypes.data_as(C.c_void_p),
            ga.ctypes.data_as(C.c_void_p), gb.ctypes.data_as(C.c_void_p),
            cnt.ctypes.data_as(C.c_void_p), path.ctypes.data_as(C.c_void_p))
        return ga, gb, cnt, path.reshape(p.L, p.n, order="F")

    def solve(self, p: Problem, mode=1, snapshot_interval=10, grad_tol=1e-6, max_outer_loops=200,
              lbfgs_memory=10, ub_offset=0.0, plan=False, trace=0):
        gp, keep = self._gp(p)
        o = _GoSolverOptions(snapshot_interval, grad_tol, max_outer_loops, lbfgs_memory, mode)
        x = np.empty(p.m + p.n)
        r = _GoSolveResult()
        cap = snapshot_interval * max_outer_loops * 60 + 8
        hist = np.zeros(cap * 4, np.int64)
        pl = np.empty(p.m * p.n) if plan else None
        tr = np.empty(trace * (p.m + p.n)) if trace else None
        rows = C.c_int64(0)
        st = self.lib.go_solve(C.byref(gp), C.byref(o), C.c_double(ub_offset),
                               x.ctypes.data_as(C.c_void_p), C.byref(r),
                               hist.ctypes.data_as(C.c_void_p), C.c_int64(cap),
                               None if pl is None else pl.ctypes.data_as(C.c_void_p),
                               None if tr is None else tr.ctypes.data_as(C.c_void_p),
                               C.c_int64(trace), C.byref(rows))
        res = {f: getattr(r, f) for f, _ in _GoSolveResult._fields_}
        res["status"] = st
        res["x"] = x
        res["history"] = hist[: 4 * min(cap, r.grad_calls)].reshape(-1, 4)
        if pl is not None:
            res["plan"] = pl.reshape(p.m, p.n, order="F")
        if tr is not None:
            res["trace"] = tr[: rows.value * (p.m + p.n)].reshape(rows.value, p.m + p.n)
        return res

    # --- Rng
    def rng_stream(self, seed: int, kind: int, count: int, bound: int = 0):
        r = _GoRng()
        self.lib.go_rng_seed(C.byref(r), C.c_uint64(seed))
        fn = {0: self.lib.go_rng_next, 1: self.lib.go_rng_uniform01,
              2: self.lib.go_rng_normal}.get(kind)
        if kind == 3:
            return np.array([self.lib.go_rng_index(C.byref(r), bound) for _ in range(count)],
                            dtype=np.uint64)
        fn.argtypes = [C.c_void_p]
        vals = [fn(C.byref(r)) for _ in range(count)]
        return np.array(vals, dtype=np.uint64 if kind == 0 else np.float64)

    def cost_matrix(self, src: np.ndarray, tgt: np.ndarray) -> np.ndarray:
        src = np.ascontiguousarray(src, np.float64)
        tgt = np.ascontiguousarray(tgt, np.float64)
        m, d = src.shape
        n = tgt.shape[0]
        out = np.empty(m * n)
        self.lib.go_cost_matrix(src.ctypes.data_as(C.c_void_p), C.c_int64(m),
                                tgt.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_int64(d),
                                out.ctypes.data_as(C.c_void_p))
        return out.reshape(m, n, order="F")


class RefLib:
    """The reference itself (oracle/_ref/libgroupot_ref.so)."""

    def __init__(self, path: str = REF_SO):
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _args(self, p: Problem):
        keep = (p.cost_flat(), p.sizes, p.a, p.b)
        return keep, [keep[0].ctypes.data_as(C.c_void_p), C.c_int64(p.m), C.c_int64(p.n),
                      keep[1].ctypes.data_as(C.c_void_p), C.c_int32(p.L),
                      keep[2].ctypes.data_as(C.c_void_p), keep[3].ctypes.data_as(C.c_void_p)]

    @staticmethod
    def _v(x):
        x = np.ascontiguousarray(x, np.float64)
        return x, x.ctypes.data_as(C.c_void_p)

    def validate(self, p: Problem):
        keep, a = self._args(p)
        row, col, idx = C.c_int64(-2), C.c_int64(-2), C.c_int64(-2)
        which = C.c_char(b"?")
        st = self.lib.ref_validate(*a, C.c_double(p.gamma), C.c_double(p.mu), C.byref(row),
                                   C.byref(col), C.byref(which), C.byref(idx))
        return st, dict(row=row.value, col=col.value, which=which.value.decode(),
                        index=idx.value)

    def eval(self, p: Problem, alpha, beta):
        keep, a = self._args(p)
        al, alp = self._v(alpha)
        be, bep = self._v(beta)
        obj = C.c_double()
        ga, gb = np.empty(p.m), np.empty(p.n)
        st = self.lib.ref_eval(*a, C.c_double(p.gamma), C.c_double(p.mu), alp, bep, C.byref(obj),
                               ga.ctypes.data_as(C.c_void_p), gb.ctypes.data_as(C.c_void_p))
        assert st == 0, self.lib.ref_last_error()
        return obj.value, ga, gb

    def plan(self, p: Problem, alpha, beta):
        keep, a = self._args(p)
        al, alp = self._v(alpha)
        be, bep = self._v(beta)
        out = np.empty(p.m * p.n)
        st = self.lib.ref_plan(*a, C.c_double(p.gamma), C.c_double(p.mu), alp, bep,
                               out.ctypes.data_as(C.c_void_p))
        assert st == 0
        return out.reshape(p.m, p.n, order="F")

    def primal_objective(self, p: Problem, plan) -> float:
        keep, a = self._args(p)
        pl = np.asfortranarray(plan, np.float64)
        out = C.c_double()
        st = self.lib.ref_primal_objective(*a, C.c_double(p.gamma), C.c_double(p.mu),
                                           pl.ctypes.data_as(C.c_void_p), C.byref(out))
        assert st == 0, self.lib.ref_last_error()
        return out.value

    def plan_diagnostics(self, p: Problem, plan) -> np.ndarray:
        keep, a = self._args(p)
        pl = np.asfortranarray(plan, np.float64)
        out = np.empty(4)
        st = self.lib.ref_plan_diagnostics(*a, pl.ctypes.data_as(C.c_void_p),
                                           out.ctypes.data_as(C.c_void_p))
        assert st == 0, self.lib.ref_last_error()
        return out

    def snapshot(self, p: Problem, alpha, beta):
        keep, a = self._args(p)
        al, alp = self._v(alpha)
        be, bep = self._v(beta)
        z, k, o = (np.empty(p.L * p.n) for _ in range(3))
        st = self.lib.ref_snapshot(*a, alp, bep, z.ctypes.data_as(C.c_void_p),
                                   k.ctypes.data_as(C.c_void_p), o.ctypes.data_as(C.c_void_p))
        assert st == 0
        f = lambda v: v.reshape(p.L, p.n, order="F")  # noqa: E731
        return f(z), f(k), f(o)

    def active_set(self, p: Problem, alpha_s, beta_s, alpha, beta):
        keep, a = self._args(p)
        vs = [self._v(v) for v in (alpha_s, beta_s, alpha, beta)]
        member = np.zeros(p.L * p.n, np.uint8)
        cnt = C.c_int64()
        st = self.lib.ref_active_set(*a, C.c_double(p.gamma), C.c_double(p.mu),
                                     *[v[1] for v in vs], member.ctypes.data_as(C.c_void_p),
                                     C.byref(cnt))
        assert st == 0
        return member.reshape(p.L, p.n, order="F"), cnt.value

    def fast_gradient(self, p: Problem, x_a, x_s, x, use_active_set=True, ub_offset=0.0):
        """Dispatcher after init(x_a), refresh(x_s); gradient at x. Each x is
        (alpha, beta)."""
        keep, a = self._args(p)
        vs = [self._v(v) for v in (*x_a, *x_s, *x)]
        ga, gb = np.empty(p.m), np.empty(p.n)
        cnt = np.zeros(4, np.int64)
        member = np.zeros(p.L * p.n, np.uint8)
        st = self.lib.ref_fast_gradient(
            *a, C.c_double(p.gamma), C.c_double(p.mu), vs[0][1], vs[1][1], vs[2][1], vs[3][1],
            C.c_int(int(use_active_set)), C.c_double(ub_offset), vs[4][1], vs[5][1],
            ga.ctypes.data_as(C.c_void_p), gb.ctypes.data_as(C.c_void_p),
            cnt.ctypes.data_as(C.c_void_p), member.ctypes.data_as(C.c_void_p))
        assert st == 0, self.lib.ref_last_error()
        return ga, gb, cnt, member.reshape(p.L, p.n, order="F")

    def time_eval(self, p: Problem, x_a, x_s, x, reps: int = 1):
        """ref_time_eval: the reference's dispatcher init(x_a) + refresh(x_s),
        dual_objective(x) and the screened dual_gradient(x), each timed with
        steady_clock (instance copy excluded). Returns (t_obj, t_grad,
        t_refresh) in seconds summed over reps, the counters and the objective."""
        keep, a = self._args(p)
        vs = [self._v(v) for v in (*x_a, *x_s, *x)]
        times = np.zeros(3)
        cnt = np.zeros(4, np.int64)
        obj = C.c_double()
        st = self.lib.ref_time_eval(*a, C.c_double(p.gamma), C.c_double(p.mu),
                                    *[v[1] for v in vs], C.c_int(reps),
                                    times.ctypes.data_as(C.c_void_p),
                                    cnt.ctypes.data_as(C.c_void_p), C.byref(obj))
        assert st == 0, self.lib.ref_last_error()
        return times, cnt, obj.value

    def solve(self, p: Problem, mode=1, snapshot_interval=10, grad_tol=1e-6, max_outer_loops=200,
              lbfgs_memory=10, ub_offset=0.0, plan=False):
        keep, a = self._args(p)
        x = np.empty(p.m + p.n)
        sc = np.zeros(2)
        ints = np.zeros(9, np.int64)
        cap = snapshot_interval * max_outer_loops * 60 + 8
        hist = np.zeros(cap * 4, np.int64)
        pl = np.empty(p.m * p.n) if plan else None
        st = self.lib.ref_solve(*a, C.c_double(p.gamma), C.c_double(p.mu), C.c_int(mode),
                                C.c_int(snapshot_interval), C.c_double(grad_tol),
                                C.c_int(max_outer_loops), C.c_int(lbfgs_memory),
                                C.c_double(ub_offset), x.ctypes.data_as(C.c_void_p),
                                sc.ctypes.data_as(C.c_void_p), ints.ctypes.data_as(C.c_void_p),
                                hist.ctypes.data_as(C.c_void_p), C.c_int64(cap),
                                None if pl is None else pl.ctypes.data_as(C.c_void_p))
        res = dict(status=st, x=x, objective=sc[0], wall_seconds=sc[1],
                   iterations=int(ints[0]), converged=int(ints[1]),
                   line_search_failed=int(ints[2]), outer_loops=int(ints[3]),
                   grad_calls=int(ints[4]), blocks_in_active_set=int(ints[5]),
                   blocks_skipped=int(ints[6]), blocks_unskipped=int(ints[7]),
                   upper_bounds_evaluated=int(ints[8]))
        res["history"] = hist[: 4 * min(cap, res["grad_calls"])].reshape(-1, 4)
        if st != 0:
            res["error"] = self.lib.ref_last_error().decode()
        if pl is not None:
            res["plan"] = pl.reshape(p.m, p.n, order="F")
        return res

    def rng_stream(self, seed: int, kind: int, count: int, bound: int = 0):
        d = np.zeros(count)
        u = np.zeros(count, np.uint64)
        self.lib.ref_rng_stream(C.c_uint64(seed), C.c_int(kind), C.c_uint64(bound),
                                C.c_int64(count), d.ctypes.data_as(C.c_void_p),
                                u.ctypes.data_as(C.c_void_p))
        return u if kind in (0, 3) else d

    def gen_synthetic(self, num_classes: int, per_class: int, seed: int, normalize=True):
        m = num_classes * per_class
        cost = np.empty(m * m)
        a, b = np.empty(m), np.empty(m)
        sizes = np.empty(num_classes, np.int32)
        sf, tf = np.empty(m * 2), np.empty(m * 2)
        st = self.lib.ref_gen_synthetic(C.c_int(num_classes), C.c_int(per_class),
                                        C.c_uint64(seed), C.c_int(int(normalize)),
                                        cost.ctypes.data_as(C.c_void_p),
                                        a.ctypes.data_as(C.c_void_p),
                                        b.ctypes.data_as(C.c_void_p),
                                        sizes.ctypes.data_as(C.c_void_p),
                                        sf.ctypes.data_as(C.c_void_p),
                                        tf.ctypes.data_as(C.c_void_p))
        assert st == 0
        return cost.reshape(m, m, order="F"), a, b, sizes, sf.reshape(m, 2), tf.reshape(m, 2)

    def cost_matrix(self, src, tgt):
        src = np.ascontiguousarray(src, np.float64)
        tgt = np.ascontiguousarray(tgt, np.float64)
        m, d = src.shape
        n = tgt.shape[0]
        out = np.empty(m * n)
        self.lib.ref_cost_matrix(src.ctypes.data_as(C.c_void_p), C.c_int64(m),
                                 tgt.ctypes.data_as(C.c_void_p), C.c_int64(n), C.c_int64(d),
                                 out.ctypes.data_as(C.c_void_p))
        return out.reshape(m, n, order="F")


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class ColumnParallelOracle:
    """The oracle over column ranges of a large instance on host threads
    (ctypes releases the GIL): every per-block quantity -- snapshot norms,
    screening decisions, active-set membership, plan entries -- is the
    oracle's own (bitwise), and the column-separable sums are recombined:
    objective = sum_r obj_r - (R-1) a.alpha, grad_alpha = sum_r ga_r - (R-1) a
    (dual.hpp:38-52, :85-100 restricted to columns J_r). Test infrastructure
    for BASELINE configs 3-5 (8 - 40 GB), where one single-threaded pass is
    a minute of CPU."""

    def __init__(self, p: Problem, threads: int = 0):
        self.o = Oracle()
        self.p = p
        threads = threads or (os.cpu_count() or 1)
        self.ranges = [(int(r[0]), int(r[-1]) + 1)
                       for r in np.array_split(np.arange(p.n), min(threads, p.n))]
        self.subs = [Problem(p.cost[:, j0:j1], p.sizes, p.a, p.b[j0:j1], p.gamma, p.mu)
                     for j0, j1 in self.ranges]

    def _map(self, fn):
        import threading

        out = [None] * len(self.subs)

        def run(i):
            out[i] = fn(i, self.subs[i], *self.ranges[i])

        ths = [threading.Thread(target=run, args=(i,)) for i in range(len(self.subs))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return out

    def eval(self, x):
        """(objective, grad) at x = [alpha; beta]."""
        m, R = self.p.m, len(self.subs)
        al = x[:m]
        res = self._map(lambda i, q, j0, j1: (
            self.o.objective(q, al, x[m + j0:m + j1]), *self.o.gradient(q, al, x[m + j0:m + j1])))
        obj = sum(r[0] for r in res) - (R - 1) * float(self.p.a @ al)
        ga = sum(r[1] for r in res) - (R - 1) * self.p.a
        gb = np.concatenate([r[2] for r in res])
        return obj, np.concatenate([ga, gb])

    def block_mask(self, x):
        """Nonzero (l, j) blocks at x: z > tau (regularizer.hpp:67), L x n."""
        m = self.p.m
        tau = self.p.gamma * self.p.mu
        res = self._map(lambda i, q, j0, j1: self.o.snapshot(q, x[:m], x[m + j0:m + j1])[0])
        return np.concatenate(res, axis=1) > tau

    def fast_gradient(self, x_a, x_s, x):
        """FastGradDispatcher after init(x_a), refresh(x_s); gradient at x:
        (grad, counters[4])."""
        m, R = self.p.m, len(self.subs)

        def one(i, q, j0, j1):
            sl = slice(m + j0, m + j1)
            mem, _ = self.o.active_set(q, x_a[:m], x_a[sl], x_s[:m], x_s[sl])
            ga, gb, cnt, _ = self.o.fast_gradient(q, x_s[:m], x_s[sl], mem, x[:m], x[sl])
            return ga, gb, cnt

        res = self._map(one)
        ga = sum(r[0] for r in res) - (R - 1) * self.p.a
        gb = np.concatenate([r[1] for r in res])
        return np.concatenate([ga, gb]), sum(r[2] for r in res)

    def plan_columns(self, x, cols):
        """Plan columns `cols` (m x len(cols))."""
        m = self.p.m
        q = Problem(self.p.cost[:, cols], self.p.sizes, self.p.a, self.p.b[cols], self.p.gamma,
                    self.p.mu)
        return self.o.plan(q, x[:m], x[m:][cols])


def ref_load_csv(src_path: str, tgt_path: str):
    """The reference's load_csv (data_io.hpp:270-352) through ref_driver:
    ('ok', src_features, labels, src_weights, tgt_features, tgt_weights) or
    ('error', status, line, column, message)."""
    lib = RefLib().lib
    shape = np.zeros(5, np.int64)
    det = np.zeros(2, np.int64)
    st = lib.ref_load_csv(src_path.encode(), tgt_path.encode(), shape.ctypes.data_as(C.c_void_p),
                          det.ctypes.data_as(C.c_void_p), None, None, None, None, None)
    if st != 0:
        return ("error", int(st), int(det[0]), int(det[1]), lib.ref_last_error().decode())
    m, n, d, sw, tw = (int(v) for v in shape)
    sf, tf = np.empty((m, d)), np.empty((n, d))
    lab = np.empty(m, np.int32)
    swv, twv = np.empty(max(sw, 1)), np.empty(max(tw, 1))
    st = lib.ref_load_csv(src_path.encode(), tgt_path.encode(), shape.ctypes.data_as(C.c_void_p),
                          det.ctypes.data_as(C.c_void_p), sf.ctypes.data_as(C.c_void_p),
                          lab.ctypes.data_as(C.c_void_p), swv.ctypes.data_as(C.c_void_p),
                          tf.ctypes.data_as(C.c_void_p), twv.ctypes.data_as(C.c_void_p))
    assert st == 0
    return ("ok", sf, lab.tolist(), swv[:sw], tf, twv[:tw])


def ref_make_instance(src_path: str, tgt_path: str, m: int, n: int, normalize: bool,
                      use_weights: bool):
    """The reference's make_instance from the CSV pair: (cost, a, b, sizes)
    or ('error', status, message)."""
    lib = RefLib().lib
    cost = np.empty(m * n)
    a, b = np.empty(m), np.empty(n)
    sizes = np.empty(m, np.int32)
    L = C.c_int32()
    st = lib.ref_make_instance(src_path.encode(), tgt_path.encode(), C.c_int(int(normalize)),
                               C.c_int(int(use_weights)), cost.ctypes.data_as(C.c_void_p),
                               a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                               sizes.ctypes.data_as(C.c_void_p), C.byref(L))
    if st != 0:
        return ("error", int(st), lib.ref_last_error().decode())
    return cost.reshape(m, n, order="F"), a, b, sizes[: L.value]


def ref_partition_from_labels(labels):
    """('ok', sizes) or ('error', status, message)."""
    lib = RefLib().lib
    lab = np.ascontiguousarray(labels, np.int32)
    out = np.empty(max(1, lab.size), np.int32)
    L = C.c_int32()
    st = lib.ref_partition_from_labels(lab.ctypes.data_as(C.c_void_p), C.c_int64(lab.size),
                                       out.ctypes.data_as(C.c_void_p), C.byref(L))
    if st != 0:
        return ("error", int(st), lib.ref_last_error().decode())
    return ("ok", out[: L.value].tolist())
