"""Python mirror of the reference `groupot` API, backed by libgsot.so.

Same names, argument meanings and error behaviour as the reference C++
library (/root/reference/proj/include/groupot): the exception classes of
errors.hpp, GroupPartition / ProblemInstance / RegParams (core.hpp),
dual_objective / dual_gradient / recover_plan (dual.hpp), take_snapshot /
build_active_set / FastGradDispatcher / GradStats (screening.hpp) and
SolverMode / SolverOptions / Solution / solve / solve_baseline / solve_fast
/ audit_solve (solver.hpp). Every computation runs on the GPU through the
C ABI of include/gsot.h; nothing here computes the objective, the gradient
or a bound on the host.

Arrays: cost is m x n (any numpy order; passed to the library column-major
as Eigen::MatrixXd is), vectors are float64 1-D arrays. Snapshot matrices
and the active set are returned as (L, n) arrays, element [l, j].
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from datetime import timedelta

import numpy as np

from . import _lib

# ----------------------------------------------------------------- errors.hpp


class Error(RuntimeError):
    """Base of every error raised by this library (errors.hpp:9-12)."""


class DimensionMismatch(Error):
    pass


class NegativeCost(Error):
    def __init__(self, msg: str, row: int, col: int, value: float):
        super().__init__(msg)
        self.row, self.col, self.value = row, col, value


class MarginalNotNormalized(Error):
    def __init__(self, msg: str, which: str, index: int):
        super().__init__(msg)
        self.which, self.index = which, index


class PartitionMismatch(Error):
    pass


class RhoOutOfRange(Error):
    def __init__(self, msg: str, rho: float = float("nan")):
        super().__init__(msg)
        self.rho = rho


class AuditViolation(Error):
    pass


class CudaError(Error):
    """No usable GPU / CUDA failure (the library has no CPU fallback)."""


class StateError(Error):
    pass


def _raise(status: int) -> None:
    if status == _lib.GSOT_OK:
        return
    msg, d = _lib.last_error()
    if status == 1:
        raise DimensionMismatch(msg)
    if status == 2:
        raise NegativeCost(msg, d.row, d.col, d.value)
    if status == 3:
        raise MarginalNotNormalized(msg, d.which.decode() if d.which else "?", d.index)
    if status == 4:
        raise PartitionMismatch(msg)
    if status == 6:
        raise RhoOutOfRange(msg, d.value)
    if status == 7:
        raise AuditViolation(msg)
    if status == 8:
        raise CudaError(msg)
    if status == 9:
        raise MemoryError(msg)
    if status == 10:
        raise StateError(msg)
    raise Error(msg)


def _f64(v) -> np.ndarray:
    return np.ascontiguousarray(v, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------- core.hpp


class GroupPartition:
    """Contiguous labelled row blocks (core.hpp:17-43)."""

    def __init__(self, sizes):
        sizes = [int(s) for s in sizes]
        if not sizes:
            raise PartitionMismatch("group partition: at least one group required")
        for l, g in enumerate(sizes):
            if g < 1:
                raise PartitionMismatch(
                    f"group partition: group {l} has non-positive size {g}")
        self._sizes = np.asarray(sizes, dtype=np.int32)
        self._offsets = np.concatenate([[0], np.cumsum(self._sizes)]).astype(np.int64)

    def num_groups(self) -> int:
        return len(self._sizes)

    def total_size(self) -> int:
        return int(self._offsets[-1])

    def offset(self, l: int) -> int:
        return int(self._offsets[l])

    def size(self, l: int) -> int:
        return int(self._sizes[l])

    def sizes(self) -> list[int]:
        return self._sizes.tolist()

    def offsets(self) -> list[int]:
        return self._offsets.tolist()


class RegParams:
    """(gamma, mu); tau = mu * gamma is derived, never stored (core.hpp:59-75)."""

    def __init__(self, gamma: float, mu: float):
        if not (gamma > 0.0) or not math.isfinite(gamma):
            raise Error(f"gamma must be positive, got {gamma}")
        if not (mu > 0.0) or not math.isfinite(mu):
            raise Error(f"mu must be positive, got {mu}")
        self._gamma, self._mu = float(gamma), float(mu)

    def gamma(self) -> float:
        return self._gamma

    def mu(self) -> float:
        return self._mu

    def tau(self) -> float:
        return self._mu * self._gamma


def params_from_rho(gamma: float, rho: float) -> RegParams:
    """core.hpp:148-151, computed by gsot_params_from_rho."""
    ge, me = C.c_double(), C.c_double()
    st = _lib.lib().gsot_params_from_rho(float(gamma), float(rho), C.byref(ge), C.byref(me))
    if st == 6:
        msg, _ = _lib.last_error()
        raise RhoOutOfRange(msg, rho)
    _raise(st)
    return RegParams(ge.value, me.value)


class ProblemInstance:
    """Cost (m x n), marginals a (m), b (n), source groups (core.hpp:47-55).

    The cost array is frozen (read-only) so that the device-resident copy
    the library keeps cannot go stale; assign a new array to change it.
    """

    def __init__(self, cost, a, b, groups: GroupPartition):
        self.groups = groups
        self.cost = cost
        self.a = a
        self.b = b

    @property
    def cost(self) -> np.ndarray:
        return self._cost

    @cost.setter
    def cost(self, value) -> None:
        c = np.array(value, dtype=np.float64, order="F", copy=True)
        if c.ndim != 2:
            raise DimensionMismatch("dimension mismatch: cost must be a matrix")
        c.flags.writeable = False
        self._cost = c
        self._drop_context()

    @property
    def a(self) -> np.ndarray:
        return self._a

    @a.setter
    def a(self, value) -> None:
        self._a = np.array(value, dtype=np.float64).reshape(-1)
        self._a.flags.writeable = False
        self._drop_context()

    @property
    def b(self) -> np.ndarray:
        return self._b

    @b.setter
    def b(self, value) -> None:
        self._b = np.array(value, dtype=np.float64).reshape(-1)
        self._b.flags.writeable = False
        self._drop_context()

    def m(self) -> int:
        return self._cost.shape[0]

    def n(self) -> int:
        return self._cost.shape[1]

    def __setattr__(self, k, v):
        if k == "groups" and "_ctx" in self.__dict__:
            self._drop_context()
        object.__setattr__(self, k, v)

    def _drop_context(self) -> None:
        ctx = self.__dict__.get("_ctx")
        if ctx is not None:
            ctx.close()
        self.__dict__["_ctx"] = None

    def context(self, p: RegParams) -> "Context":
        """The device-resident copy of this instance (created on first use)."""
        ctx = self.__dict__.get("_ctx")
        if ctx is None:
            ctx = Context.from_instance(self, p)
            self.__dict__["_ctx"] = ctx
        else:
            ctx.set_params(p.gamma(), p.mu())
        return ctx


@dataclass
class TransportPlan:
    plan: np.ndarray


def _check_marginal_lengths(cost: np.ndarray, a: np.ndarray, b: np.ndarray) -> None:
    """validate_instance's order (core.hpp:117-131) when a marginal has the
    wrong length: the library cannot take such a pair, so the cost scan that
    comes first in the reference (first offender in j-major order) runs here
    before the DimensionMismatch; both messages are the reference's."""
    m, n = cost.shape
    if a.size == m and b.size == n:
        return
    flat = np.asarray(cost, dtype=np.float64).reshape(-1, order="F")
    bad = np.flatnonzero(~(np.isfinite(flat) & (flat >= 0.0)))
    if bad.size:
        k = int(bad[0])
        i, j, v = k % m, k // m, float(flat[k])
        raise NegativeCost(f"cost({i},{j}) = {v:.6f} is negative or non-finite", i, j, v)
    if a.size != m:
        raise DimensionMismatch(
            f"dimension mismatch: marginal a has length {a.size}, cost has {m} rows")
    raise DimensionMismatch(
        f"dimension mismatch: marginal b has length {b.size}, cost has {n} columns")


def validate_instance(inst: ProblemInstance) -> None:
    """core.hpp:117-139 (run by the library while uploading the cost)."""
    _check_marginal_lengths(inst.cost, inst.a, inst.b)
    ctx = Context.from_instance(inst, RegParams(1.0, 1.0))
    ctx.close()


# ------------------------------------------------------------------- context


class Context:
    """Owner of one gsot_ctx: the resident instance on one CUDA stream."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        shape = (C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64())
        _raise(_lib.lib().gsot_shape(self._h, *[C.byref(s) for s in shape]))
        self.m, self.n, self.L, self.device_bytes = (int(s.value) for s in shape)

    @classmethod
    def from_instance(cls, inst: ProblemInstance, p: RegParams) -> "Context":
        _check_marginal_lengths(inst.cost, inst.a, inst.b)
        return cls.from_arrays(inst.cost, inst.groups.sizes(), inst.a, inst.b, p.gamma(), p.mu())

    @classmethod
    def from_arrays(cls, cost, sizes, a, b, gamma: float, mu: float) -> "Context":
        cost = np.asfortranarray(cost, dtype=np.float64)
        m, n = cost.shape
        sizes = np.ascontiguousarray(sizes, dtype=np.int32)
        a, b = _f64(a), _f64(b)
        _check_marginal_lengths(cost, a, b)
        h = C.c_void_p()
        st = _lib.lib().gsot_create(_ptr(cost), m, n, _ptr(sizes), len(sizes), _ptr(a), _ptr(b),
                                    float(gamma), float(mu), C.byref(h))
        _raise(st)
        return cls(h.value)

    @classmethod
    def shard_from_arrays(cls, cost_block, sizes, a, b_block, gamma: float,
                          mu: float) -> "Context":
        """A column shard (gsot_create_shard): marginals checked entrywise only."""
        cost = np.asfortranarray(cost_block, dtype=np.float64)
        m, n = cost.shape
        sizes = np.ascontiguousarray(sizes, dtype=np.int32)
        a, b = _f64(a), _f64(b_block)
        h = C.c_void_p()
        st = _lib.lib().gsot_create_shard(_ptr(cost), m, n, _ptr(sizes), len(sizes), _ptr(a),
                                          _ptr(b), float(gamma), float(mu), C.byref(h))
        _raise(st)
        return cls(h.value)

    @classmethod
    def shard_from_device(cls, d_cost_ptr: int, m: int, n_shard: int, sizes, a, b_block,
                          gamma: float, mu: float) -> "Context":
        """gsot_create_shard_device: the m x n_shard column block (column-major) at
        device address d_cost_ptr."""
        sizes = np.ascontiguousarray(sizes, dtype=np.int32)
        a, b = _f64(a), _f64(b_block)
        h = C.c_void_p()
        st = _lib.lib().gsot_create_shard_device(C.c_void_p(d_cost_ptr), int(m), int(n_shard),
                                                 _ptr(sizes), len(sizes), _ptr(a), _ptr(b),
                                                 float(gamma), float(mu), C.byref(h))
        _raise(st)
        return cls(h.value)

    @classmethod
    def from_config(cls, cfg: int, seed: int, gamma: float, mu: float) -> "Context":
        h = C.c_void_p()
        _raise(_lib.lib().gsot_create_config(int(cfg), int(seed), float(gamma), float(mu),
                                             C.byref(h)))
        return cls(h.value)

    def close(self) -> None:
        if self._h is not None and self._h.value:
            _lib.lib().gsot_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_params(self, gamma: float, mu: float) -> None:
        _raise(_lib.lib().gsot_set_params(self._h, float(gamma), float(mu)))

    def eval(self, x, screened: bool = False, exact: bool = False):
        x = _f64(x)
        if x.size != self.m + self.n:
            raise DimensionMismatch(
                f"dimension mismatch: state has {x.size} entries, instance is "
                f"({self.m},{self.n})")
        g = np.empty(self.m + self.n)
        obj = C.c_double()
        st = CallStatsPy()
        cs = _lib.CallStats()
        mode = (1 if screened else 0) | (2 if exact else 0)
        _raise(_lib.lib().gsot_eval(self._h, _ptr(x), mode, C.byref(obj), _ptr(g), C.byref(cs)))
        st.in_active, st.skipped, st.unskipped, st.upper_bounds = (
            cs.in_active, cs.skipped, cs.unskipped, cs.upper_bounds)
        return obj.value, g, st

    def sequential_sum(self, terms, s0: float = 0.0) -> float:
        """((s0 + t0) + t1) + ... exactly as a sequential loop rounds it, computed
        by the device's exact-order engine (gsot_sequential_sum)."""
        t = _f64(terms)
        out = C.c_double()
        _raise(_lib.lib().gsot_sequential_sum(self._h, _ptr(t), t.size, float(s0), C.byref(out)))
        return out.value

    def set_upper_bound_offset(self, offset: float) -> None:
        _raise(_lib.lib().gsot_set_upper_bound_offset(self._h, float(offset)))

    def init_snapshot(self, x) -> None:
        _raise(_lib.lib().gsot_init_snapshot(self._h, _ptr(_f64(x))))

    def refresh(self, x, use_active_set: bool) -> None:
        _raise(_lib.lib().gsot_refresh(self._h, _ptr(_f64(x)), int(bool(use_active_set))))

    def snapshot_norms(self):
        z, k, o = (np.empty(self.L * self.n) for _ in range(3))
        _raise(_lib.lib().gsot_snapshot_norms(self._h, _ptr(z), _ptr(k), _ptr(o)))
        f = lambda v: v.reshape(self.L, self.n, order="F")  # noqa: E731
        return f(z), f(k), f(o)

    def active_set(self):
        mem = np.zeros(self.L * self.n, np.uint8)
        cnt = C.c_int64()
        _raise(_lib.lib().gsot_active_set(self._h, _ptr(mem), C.byref(cnt)))
        return mem.reshape(self.L, self.n, order="F").astype(bool), int(cnt.value)

    def block_mask(self, x) -> np.ndarray:
        out = np.zeros(self.L * self.n, np.uint8)
        _raise(_lib.lib().gsot_block_mask(self._h, _ptr(_f64(x)), _ptr(out)))
        return out.reshape(self.L, self.n, order="F").astype(bool)

    def plan_columns(self, x, j0: int, j1: int) -> np.ndarray:
        out = np.empty(self.m * (j1 - j0))
        _raise(_lib.lib().gsot_plan_columns(self._h, _ptr(_f64(x)), int(j0), int(j1), _ptr(out)))
        return out.reshape(self.m, j1 - j0, order="F")

    def primal_objective(self, x) -> float:
        """primal_objective(recover_plan(x)) on the device (gsot_primal_objective)."""
        v = C.c_double()
        _raise(_lib.lib().gsot_primal_objective(self._h, _ptr(_f64(x)), C.byref(v)))
        return v.value

    def plan_diagnostics(self, x) -> "PlanDiagnostics":
        """plan_diagnostics(recover_plan(x)) on the device (gsot_plan_diagnostics)."""
        d = _lib.PlanDiagC()
        _raise(_lib.lib().gsot_plan_diagnostics(self._h, _ptr(_f64(x)), C.byref(d)))
        return PlanDiagnostics(d.marginal_res_a, d.marginal_res_b, d.group_sparsity, d.mass)

    def solve(self, mode: int = 1, snapshot_interval: int = 10, grad_tol: float = 1e-6,
              max_outer_loops: int = 200, lbfgs_memory: int = 10,
              upper_bound_offset: float = 0.0, history_cap: int = 0, exact: bool = False,
              no_active_set: bool = False):
        """gsot_solve; exact=True runs the reference-order sums (bitwise trajectory);
        no_active_set=True with mode 3 audits a fast_no_lower_bound solve."""
        o = _lib.SolverOptionsC(int(snapshot_interval), float(grad_tol), int(max_outer_loops),
                                int(lbfgs_memory), int(mode), float(upper_bound_offset),
                                (1 if exact else 0) | (2 if no_active_set else 0))
        x = np.empty(self.m + self.n)
        r = _lib.SolveResultC()
        hist = np.zeros(max(1, history_cap) * 4, np.int64)
        _raise(_lib.lib().gsot_solve(self._h, C.byref(o), _ptr(x), C.byref(r), _ptr(hist),
                                     int(history_cap)))
        res = {f: getattr(r, f) for f, _ in _lib.SolveResultC._fields_}
        res["x"] = x
        res["history"] = hist[: 4 * min(history_cap, r.grad_calls)].reshape(-1, 4)
        return res

    # ---- multi-GPU column sharding on the device (gsot_comm_*)
    def attach_nccl(self, unique_id: bytes, world: int, rank: int) -> None:
        """Attach an NCCL communicator (collective over the ranks); gsot_solve on
        this shard context then runs the sharded solve with its all-reduces on
        the context stream, inside the solver's CUDA graphs."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _raise(_lib.lib().gsot_comm_attach_nccl(self._h, buf, int(world), int(rank)))

    def attach_host(self, world: int, rank: int, allreduce) -> None:
        """Attach a host transport: allreduce(np.ndarray view, op) reduces the
        doubles in place over the ranks (op 0 sum, 1 max)."""
        def cb(ptr, count, op, _user):
            try:
                allreduce(np.ctypeslib.as_array(ptr, shape=(int(count),)), int(op))
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failure
                import traceback

                traceback.print_exc()
                return 1

        self._comm_cb = _lib.ALLREDUCE_FN(cb)  # kept alive with the context
        _raise(_lib.lib().gsot_comm_attach_host(self._h, int(world), int(rank), self._comm_cb,
                                                None))

    def detach_comm(self) -> None:
        _raise(_lib.lib().gsot_comm_detach(self._h))
        self._comm_cb = None

    def profile(self, enable) -> None:
        """False: off; True: time every kernel class; int: bit mask (1 << kind)."""
        if enable is True:
            enable = -1
        _raise(_lib.lib().gsot_profile_enable(self._h, int(enable)))

    def profile_read(self, kind: int):
        ms, by, n = C.c_double(), C.c_double(), C.c_int64()
        _raise(_lib.lib().gsot_profile_read(self._h, int(kind), C.byref(ms), C.byref(by),
                                            C.byref(n)))
        return ms.value, by.value, int(n.value)

    def profile_reset(self) -> None:
        _raise(_lib.lib().gsot_profile_reset(self._h))

    def kernel_launches(self) -> int:
        return int(_lib.lib().gsot_kernel_launches(self._h))

    def timer_start(self) -> None:
        _raise(_lib.lib().gsot_timer(self._h, 0, None))

    def timer_stop(self) -> float:
        ms = C.c_double()
        _raise(_lib.lib().gsot_timer(self._h, 1, C.byref(ms)))
        return ms.value


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id for Context.attach_nccl (rank 0; broadcast it)."""
    buf = C.create_string_buffer(128)
    _raise(_lib.lib().gsot_comm_unique_id(buf))
    return buf.raw


def cache_clear() -> int:
    """Free the device state parked by closed contexts (gsot_cache_clear)."""
    return int(_lib.lib().gsot_cache_clear())


def set_device(device: int) -> None:
    """CUDA device for contexts created afterwards on this thread."""
    _raise(_lib.lib().gsot_set_device(int(device)))


@dataclass
class CallStatsPy:
    in_active: int = 0
    skipped: int = 0
    unskipped: int = 0
    upper_bounds: int = 0


# ------------------------------------------------------------------- dual.hpp


@dataclass
class DualState:
    alpha: np.ndarray
    beta: np.ndarray


def _state_vec(s: DualState, inst: ProblemInstance) -> np.ndarray:
    alpha, beta = _f64(s.alpha).reshape(-1), _f64(s.beta).reshape(-1)
    if alpha.size != inst.m() or beta.size != inst.n():  # dual.hpp:17-23
        raise DimensionMismatch(
            f"dimension mismatch: dual state is ({alpha.size},{beta.size}), instance is "
            f"({inst.m()},{inst.n()})")
    return np.concatenate([alpha, beta])


def dual_objective(s: DualState, inst: ProblemInstance, p: RegParams) -> float:
    """a.alpha + b.beta - sum psi (dual.hpp:38-52)."""
    x = _state_vec(s, inst)
    obj, _, _ = inst.context(p).eval(x)
    return obj


def dual_gradient(s: DualState, inst: ProblemInstance, p: RegParams):
    """(grad_alpha, grad_beta) with the unscreened provider (dual.hpp:85-130)."""
    x = _state_vec(s, inst)
    _, g, _ = inst.context(p).eval(x)
    return g[: inst.m()], g[inst.m():]


def recover_plan(s: DualState, inst: ProblemInstance, p: RegParams) -> TransportPlan:
    """T[:, j] = grad psi(f_j) (dual.hpp:116-128), streamed from the device."""
    x = _state_vec(s, inst)
    return TransportPlan(inst.context(p).plan_columns(x, 0, inst.n()))


@dataclass
class PlanDiagnostics:
    marginal_res_a: float = 0.0
    marginal_res_b: float = 0.0
    group_sparsity: float = 0.0
    mass: float = 0.0


def regularizer_value(column, groups: GroupPartition, p: RegParams) -> float:
    """gamma (|t|^2 / 2 + mu sum_l |t_[l]|) of one plan column (core.hpp:153-165)."""
    col = _f64(column).reshape(-1)
    if col.size != groups.total_size():
        raise DimensionMismatch(f"dimension mismatch: column length {col.size} vs partition size "
                                f"{groups.total_size()}")
    norms = sum(float(np.linalg.norm(col[groups.offset(l): groups.offset(l) + groups.size(l)]))
                for l in range(groups.num_groups()))
    return p.gamma() * (0.5 * float(col @ col) + p.mu() * norms)


def primal_objective(t: TransportPlan, inst: ProblemInstance, p: RegParams) -> float:
    """<T, C> plus the regularizer over the plan's columns (core.hpp:167-180);
    numpy on a given plan (state_primal_objective computes it on the device)."""
    P = t.plan
    if P.shape != (inst.m(), inst.n()):
        raise DimensionMismatch(f"dimension mismatch: plan is {P.shape[0]}x{P.shape[1]}, cost is "
                                f"{inst.m()}x{inst.n()}")
    return float(np.sum(P * inst.cost)) + sum(regularizer_value(P[:, j], inst.groups, p)
                                              for j in range(P.shape[1]))


def state_primal_objective(s: DualState, inst: ProblemInstance, p: RegParams) -> float:
    """primal_objective(recover_plan(s), inst, p) on the device (gsot_primal_objective)."""
    return inst.context(p).primal_objective(_state_vec(s, inst))


def state_plan_diagnostics(s: DualState, inst: ProblemInstance, p: RegParams) -> PlanDiagnostics:
    """plan_diagnostics(recover_plan(s, inst, p), inst) computed on the device
    without materialising the m x n plan (gsot_plan_diagnostics)."""
    return inst.context(p).plan_diagnostics(_state_vec(s, inst))


def plan_diagnostics(t: TransportPlan, inst: ProblemInstance) -> PlanDiagnostics:
    """Reporting only (dual.hpp:139-169); numpy on a downloaded plan."""
    P = t.plan
    if P.shape != (inst.m(), inst.n()):
        raise DimensionMismatch(f"dimension mismatch: plan is {P.shape[0]}x{P.shape[1]}")
    d = PlanDiagnostics()
    d.marginal_res_a = float(np.max(np.abs(P.sum(axis=1) - inst.a)))
    d.marginal_res_b = float(np.max(np.abs(P.sum(axis=0) - inst.b)))
    d.mass = float(P.sum())
    zero = 0
    for l in range(inst.groups.num_groups()):
        o, g = inst.groups.offset(l), inst.groups.size(l)
        zero += int(np.sum(np.all(P[o:o + g, :] == 0.0, axis=0)))
    d.group_sparsity = zero / (inst.groups.num_groups() * inst.n())
    return d


# -------------------------------------------------------------- screening.hpp


@dataclass
class SnapshotStore:
    alpha_snap: np.ndarray
    beta_snap: np.ndarray
    z_snap: np.ndarray  # (L, n)
    k_snap: np.ndarray
    o_snap: np.ndarray
    stamp: int = 0


def take_snapshot(s: DualState, inst: ProblemInstance, stamp: int = 0,
                  p: RegParams | None = None) -> SnapshotStore:
    """screening.hpp:24-50, computed by the snapshot kernel."""
    x = _state_vec(s, inst)
    ctx = inst.context(p or RegParams(1.0, 1.0))
    ctx.init_snapshot(x)
    z, k, o = ctx.snapshot_norms()
    return SnapshotStore(x[: inst.m()].copy(), x[inst.m():].copy(), z, k, o, stamp)


@dataclass
class ActiveSet:
    num_groups: int
    n: int
    member: np.ndarray  # (L, n) bool
    count: int

    def contains(self, l: int, j: int) -> bool:
        return bool(self.member[l, j])


def build_active_set(snap_state: DualState, state: DualState, inst: ProblemInstance,
                     p: RegParams) -> ActiveSet:
    """screening.hpp:147-166: lower bounds at `state` against the snapshot
    taken at `snap_state` (the device keeps the snapshot, not the caller)."""
    ctx = inst.context(p)
    ctx.init_snapshot(_state_vec(snap_state, inst))
    ctx.refresh(_state_vec(state, inst), True)
    mem, cnt = ctx.active_set()
    return ActiveSet(inst.groups.num_groups(), inst.n(), mem, cnt)


@dataclass
class GradStats:
    """screening.hpp:173-188."""

    blocks_in_active_set: int = 0
    blocks_skipped: int = 0
    blocks_unskipped: int = 0
    upper_bounds_evaluated: int = 0
    outer_loops: int = 0
    grad_calls: int = 0
    history: list = field(default_factory=list)  # rows (in_active, skipped, unskipped, ub)


class FastGradDispatcher:
    """Screened gradient provider (screening.hpp:206-315), on the device.

    init / refresh / gradient keep the reference's call protocol; one
    `gradient` call is the reference's begin_call + n column calls + end_call.
    """

    def __init__(self, inst: ProblemInstance, p: RegParams, stats: GradStats,
                 use_active_set: bool, upper_bound_offset: float = 0.0):
        self.inst, self.p, self.stats = inst, p, stats
        self.use_active_set = use_active_set
        self.upper_bound_offset = float(upper_bound_offset)
        self._ctx = inst.context(p)

    def init(self, s: DualState) -> None:
        self._ctx.init_snapshot(_state_vec(s, self.inst))

    def refresh(self, s: DualState, stamp: int = 0) -> None:
        self._ctx.refresh(_state_vec(s, self.inst), self.use_active_set)

    def gradient(self, s: DualState):
        self._ctx.set_upper_bound_offset(self.upper_bound_offset)
        try:
            obj, g, st = self._ctx.eval(_state_vec(s, self.inst), screened=True)
        finally:
            self._ctx.set_upper_bound_offset(0.0)
        self.stats.blocks_in_active_set += st.in_active
        self.stats.blocks_skipped += st.skipped
        self.stats.blocks_unskipped += st.unskipped
        self.stats.upper_bounds_evaluated += st.upper_bounds
        self.stats.grad_calls += 1
        self.stats.history.append((st.in_active, st.skipped, st.unskipped, st.upper_bounds))
        m = self.inst.m()
        return g[:m], g[m:], obj

    def snapshot(self) -> SnapshotStore:
        z, k, o = self._ctx.snapshot_norms()
        return SnapshotStore(np.empty(0), np.empty(0), z, k, o)

    def active_set(self) -> ActiveSet:
        mem, cnt = self._ctx.active_set()
        return ActiveSet(self.inst.groups.num_groups(), self.inst.n(), mem, cnt)


# ----------------------------------------------------------------- solver.hpp


class SolverMode(enum.IntEnum):
    baseline = 0
    fast = 1
    fast_no_lower_bound = 2
    audit = 3


def to_string(m: SolverMode) -> str:
    return {0: "baseline", 1: "fast", 2: "fast-no-lb", 3: "audit"}[int(m)]


@dataclass
class SolverOptions:
    snapshot_interval: int = 10
    grad_tol: float = 1e-6
    max_outer_loops: int = 200
    lbfgs_memory: int = 10
    mode: SolverMode = SolverMode.fast


@dataclass
class AuditReport:
    skip_checks: int = 0
    active_checks: int = 0
    column_compares: int = 0
    gradient_calls: int = 0


class Solution:
    """solver.hpp:33-42. The plan is recovered from the device on first
    access (column-streamed), not materialised by the solve."""

    def __init__(self, inst: ProblemInstance, p: RegParams, res: dict):
        m = inst.m()
        self._inst, self._p = inst, p
        self.state = DualState(res["x"][:m].copy(), res["x"][m:].copy())
        self.objective = res["objective"]
        self.iterations = res["iterations"]
        self.converged = bool(res["converged"])
        self.line_search_failed = bool(res["line_search_failed"])
        self.wall_time = timedelta(seconds=res["wall_seconds"])
        self.stats = GradStats(res["blocks_in_active_set"], res["blocks_skipped"],
                               res["blocks_unskipped"], res["upper_bounds_evaluated"],
                               res["outer_loops"], res["grad_calls"],
                               [tuple(r) for r in res["history"].tolist()])
        self._plan = None

    @property
    def plan(self) -> TransportPlan:
        if self._plan is None:
            self._plan = recover_plan(self.state, self._inst, self._p)
        return self._plan


def _run(inst: ProblemInstance, p: RegParams, opts: SolverOptions, mode: int,
         ub_offset: float = 0.0, no_active_set: bool = False):
    ctx = inst.context(p)
    cap = opts.snapshot_interval * opts.max_outer_loops * 64 + 16
    res = ctx.solve(mode=mode, snapshot_interval=opts.snapshot_interval, grad_tol=opts.grad_tol,
                    max_outer_loops=opts.max_outer_loops, lbfgs_memory=opts.lbfgs_memory,
                    upper_bound_offset=ub_offset, history_cap=cap, no_active_set=no_active_set)
    return res


def solve_baseline(inst: ProblemInstance, p: RegParams,
                   opts: SolverOptions | None = None) -> Solution:
    opts = opts or SolverOptions()
    return Solution(inst, p, _run(inst, p, opts, 0))


def solve_fast(inst: ProblemInstance, p: RegParams, opts: SolverOptions | None = None) -> Solution:
    opts = opts or SolverOptions()
    mode = 2 if opts.mode == SolverMode.fast_no_lower_bound else 1
    return Solution(inst, p, _run(inst, p, opts, mode))


def audit_solve(inst: ProblemInstance, p: RegParams, opts: SolverOptions | None = None,
                upper_bound_offset: float = 0.0):
    opts = opts or SolverOptions()
    if opts.mode == SolverMode.baseline:
        return solve_baseline(inst, p, opts), AuditReport()
    # solver.hpp:271: the active set is used unless the options say fast_no_lower_bound
    res = _run(inst, p, opts, 3, upper_bound_offset,
               no_active_set=opts.mode == SolverMode.fast_no_lower_bound)
    rep = AuditReport(res["audit_skip_checks"], res["audit_active_checks"],
                      res["audit_column_compares"], res["audit_gradient_calls"])
    return Solution(inst, p, res), rep


def solve(inst: ProblemInstance, p: RegParams, opts: SolverOptions | None = None) -> Solution:
    opts = opts or SolverOptions()
    if opts.mode == SolverMode.baseline:
        return solve_baseline(inst, p, opts)
    if opts.mode in (SolverMode.fast, SolverMode.fast_no_lower_bound):
        return solve_fast(inst, p, opts)
    if opts.mode == SolverMode.audit:
        return audit_solve(inst, p, opts)[0]
    raise Error("unknown solver mode")


# --------------------------------------------------------------- bench.hpp


@dataclass
class BenchRecord:
    """One row of benchmark output; field order is the CSV schema (bench.hpp:15-35)."""
    mode: str = ""
    num_classes: int = 0
    per_class: int = 0
    m: int = 0
    n: int = 0
    gamma: float = 0.0
    rho: float = 0.0
    iterations: int = 0
    outer_loops: int = 0
    wall_ms: float = 0.0
    objective: float = 0.0
    blocks_computed: int = 0
    blocks_skipped: int = 0
    upper_bounds_evaluated: int = 0
    active_set_size_final: int = 0
    group_sparsity: float = 0.0
    marginal_res_a: float = 0.0
    marginal_res_b: float = 0.0
    converged: bool = False


def bench_csv_header() -> str:
    """bench.hpp:37-42."""
    return ("mode,num_classes,per_class,m,n,gamma,rho,iterations,outer_loops,"
            "wall_ms,objective,blocks_computed,blocks_skipped,"
            "upper_bounds_evaluated,active_set_size_final,group_sparsity,"
            "marginal_res_a,marginal_res_b,converged")


def _fmt(v: float) -> str:  # detail::format_double, data_io.hpp:185-189 ("%.17g")
    return "%.17g" % v


def to_csv_row(r: BenchRecord) -> str:
    """bench.hpp:44-68."""
    ints = lambda *v: [str(int(x)) for x in v]  # noqa: E731
    return ",".join([r.mode] + ints(r.num_classes, r.per_class, r.m, r.n)
                    + [_fmt(r.gamma), _fmt(r.rho)] + ints(r.iterations, r.outer_loops)
                    + [_fmt(r.wall_ms), _fmt(r.objective)]
                    + ints(r.blocks_computed, r.blocks_skipped, r.upper_bounds_evaluated,
                           r.active_set_size_final)
                    + [_fmt(r.group_sparsity), _fmt(r.marginal_res_a), _fmt(r.marginal_res_b)]
                    + ints(1 if r.converged else 0))


@dataclass
class GridSpec:
    """bench.hpp:130-136: four group-term balances by seven strengths, both modes."""
    gammas: list = field(default_factory=lambda: [1e3, 1e2, 1e1, 1e0, 1e-1, 1e-2, 1e-3])
    rhos: list = field(default_factory=lambda: [0.2, 0.4, 0.6, 0.8])
    modes: list = field(default_factory=lambda: [SolverMode.baseline, SolverMode.fast])
    base: SolverOptions = field(default_factory=SolverOptions)


def run_grid(inst: ProblemInstance, grid: GridSpec, num_classes: int, per_class: int,
             sink=None) -> list:
    """run_grid (bench.hpp:137-180) in the reference's (gamma, rho, mode) order on the
    instance's one device context (the cost is uploaded and validated once; each
    (gamma, rho) only swaps the parameters). Plan diagnostics are computed on the
    device (gsot_plan_diagnostics); active_set_size_final is the active set built at
    the solution for non-baseline modes. sink(record, solution) fires after every run."""
    rows = []
    for gamma in grid.gammas:
        for rho in grid.rhos:
            p = params_from_rho(gamma, rho)
            for mode in grid.modes:
                opts = SolverOptions(grid.base.snapshot_interval, grid.base.grad_tol,
                                     grid.base.max_outer_loops, grid.base.lbfgs_memory,
                                     SolverMode(mode))
                sol = solve(inst, p, opts)
                ctx = inst.context(p)
                x = _state_vec(sol.state, inst)
                d = ctx.plan_diagnostics(x)
                rec = BenchRecord(
                    to_string(mode), num_classes, per_class, inst.m(), inst.n(), gamma, rho,
                    sol.iterations, sol.stats.outer_loops,
                    sol.wall_time.total_seconds() * 1e3, sol.objective,
                    sol.stats.blocks_in_active_set + sol.stats.blocks_unskipped,
                    sol.stats.blocks_skipped, sol.stats.upper_bounds_evaluated, 0,
                    d.group_sparsity, d.marginal_res_a, d.marginal_res_b, sol.converged)
                if mode != SolverMode.baseline:
                    ctx.init_snapshot(x)
                    ctx.refresh(x, True)
                    rec.active_set_size_final = ctx.active_set()[1]
                if sink is not None:
                    sink(rec, sol)
                rows.append(rec)
    return rows


# --------------------------------------------------------------- data inputs


def config_shape(cfg: int):
    m, n, d = C.c_int64(), C.c_int64(), C.c_int64()
    L = C.c_int32()
    _raise(_lib.lib().gsot_config_shape(int(cfg), C.byref(m), C.byref(n), C.byref(L),
                                        C.byref(d)))
    return int(m.value), int(n.value), int(L.value), int(d.value)


def config_features(cfg: int, seed: int):
    """Host features of BASELINE config `cfg` (SURVEY.md §8(d) recipe)."""
    m, n, L, d = config_shape(cfg)
    src, tgt = np.empty((m, d)), np.empty((n, d))
    sizes = np.empty(L, np.int32)
    a, b = np.empty(m), np.empty(n)
    _raise(_lib.lib().gsot_config_features(int(cfg), int(seed), _ptr(src), _ptr(tgt),
                                           _ptr(sizes), _ptr(a), _ptr(b)))
    return src, tgt, sizes, a, b
