"""Column-sharded solve across GPUs.

Rank p of P owns the column block J_p of the cost and evaluates it on its own
GPU through a shard context (``gsot_create_shard``: cost[:, J_p], a = 0,
b[J_p]). alpha is replicated on every rank, beta is sharded. The evaluation's
one exchange step is a sum all-reduce of m + 1 doubles per call:

* the shard's ``grad[0, m)`` is minus its plan row sums (a = 0), so
  grad_alpha = a + sum_p (-rowsum_p)                    (dual.hpp:91, :96);
* grad_beta_p is complete on its rank                   (dual.hpp:97-98);
* objective = a.alpha + sum_p (b_p.beta_p - psi_p)      (dual.hpp:51).

The L-BFGS ascent is the reference's ``maximize`` (lbfgs.hpp:61-274) restated
over the distributed vector [alpha; beta_p]: every dot product is the alpha
part (identical on every rank) plus the all-reduced beta parts, and the
infinity norm is an all-reduced max, so every rank takes the same scalar
decisions. Screening is per rank: the blocks of column shard J_p, their
snapshot, bounds and active set live on rank p (screening.hpp:206-315 over the
rank's columns); the GradStats counters are all-reduced sums.

The collective is ``torch.distributed`` (NCCL on GPU ranks, gloo for the CPU
tests); the evaluations are this library's kernels.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import groupot as G


def shard_columns(n: int, world: int, rank: int, align: int = 32) -> tuple[int, int]:
    """Contiguous column block of rank `rank`: equal shares in units of `align`
    columns (whole 32-column chunks), the remainder on the last ranks."""
    units = (n + align - 1) // align
    base, extra = divmod(units, world)
    u0 = rank * base + max(0, rank - (world - extra))
    u1 = u0 + base + (1 if rank >= world - extra else 0)
    return min(n, u0 * align), min(n, u1 * align)


class Comm:
    """Sum / max all-reduce of float64 numpy arrays over torch.distributed
    (identical results on every rank)."""

    def __init__(self, pg=None, device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.on = pg is not None and dist.is_initialized() and dist.get_world_size() > 1
        self.device = device if device is not None else (
            "cuda" if self.on and dist.get_backend() == "nccl" else "cpu")

    def allreduce(self, v: np.ndarray, op: str = "sum") -> np.ndarray:
        if not self.on:
            return np.array(v, dtype=np.float64, copy=True)
        t = self.torch.from_numpy(np.ascontiguousarray(v, np.float64)).to(self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX)
        return t.cpu().numpy()


@dataclass
class ShardStats:
    """GradStats (screening.hpp:173-188) summed over ranks."""
    blocks_in_active_set: int = 0
    blocks_skipped: int = 0
    blocks_unskipped: int = 0
    upper_bounds_evaluated: int = 0
    grad_calls: int = 0
    history: list = field(default_factory=list)


class ShardedProblem:
    """One rank's share of an instance: the shard context and the global
    marginal a. `evaluator` (tests only) replaces the device evaluation:
    evaluator(x_local, screened) -> (objective_p, grad_local, counters4)."""

    def __init__(self, cost_block, sizes, a, b_block, gamma: float, mu: float, comm: Comm,
                 evaluator=None, ctx=None):
        self.a = np.ascontiguousarray(a, np.float64)
        self.m = self.a.size
        self.n_p = int(np.asarray(b_block).size)
        self.comm = comm
        self.evaluator = evaluator
        self.ctx = ctx  # a prebuilt shard context (Context.shard_from_device)
        if evaluator is None and ctx is None:
            self.ctx = G.Context.shard_from_arrays(cost_block, sizes, np.zeros(self.m), b_block,
                                                   gamma, mu)

    def close(self) -> None:
        if self.ctx is not None:
            self.ctx.close()
            self.ctx = None

    # ---- evaluation: one all-reduce of m + 1 doubles (+ 4 counters)
    def eval(self, x: np.ndarray, screened: bool):
        if self.evaluator is not None:
            obj_p, g, cnt = self.evaluator(x, screened)
        else:
            obj_p, g, st = self.ctx.eval(x, screened=screened)
            cnt = (st.in_active, st.skipped, st.unskipped, st.upper_bounds)
        m = self.m
        buf = np.empty(m + 5)
        buf[:m] = g[:m]  # minus the shard's row sums
        buf[m] = obj_p   # b_p.beta_p - psi_p
        buf[m + 1:] = cnt
        red = self.comm.allreduce(buf, "sum")
        grad = np.empty_like(g)
        grad[:m] = self.a + red[:m]
        grad[m:] = g[m:]
        obj = float(np.dot(self.a, x[:m]) + red[m])
        return obj, grad, tuple(int(v) for v in red[m + 1:])

    def init_snapshot(self, x) -> None:
        if self.ctx is not None:
            self.ctx.init_snapshot(x)

    def refresh(self, x, use_active_set: bool) -> None:
        if self.ctx is not None:
            self.ctx.refresh(x, use_active_set)

    # ---- distributed vector algebra on [alpha; beta_p]
    def dot(self, u: np.ndarray, v: np.ndarray) -> float:
        m = self.m
        return float(np.dot(u[:m], v[:m]) + self.comm.allreduce(np.array([np.dot(u[m:], v[m:])]))[0])

    def norm(self, u: np.ndarray) -> float:
        return math.sqrt(self.dot(u, u))

    def inf_norm(self, u: np.ndarray) -> float:
        m = self.m
        loc = float(np.max(np.abs(u[m:]))) if u.size > m else 0.0
        return max(float(np.max(np.abs(u[:m]))),
                   float(self.comm.allreduce(np.array([loc]), "max")[0]))


@dataclass
class ShardedResult:
    x: np.ndarray  # this rank's [alpha; beta_p]
    objective: float
    iterations: int
    outer_loops: int
    converged: bool
    line_search_failed: bool
    stats: ShardStats
    wall_seconds: float


def solve_sharded(sp: ShardedProblem, mode: int = 1, snapshot_interval: int = 10,
                  grad_tol: float = 1e-6, max_outer_loops: int = 200, memory: int = 10,
                  wolfe_c1: float = 1e-4, wolfe_c2: float = 0.9, max_bracket: int = 40,
                  max_zoom: int = 12) -> ShardedResult:
    """solve_baseline (mode 0) / solve_fast (1) / fast_no_lower_bound (2)
    (solver.hpp:92-258) with maximize (lbfgs.hpp:61-274) over the shards."""
    screened = mode in (1, 2)
    use_active = mode == 1
    dim = sp.m + sp.n_p
    stats = ShardStats()

    def evaluate(x):
        obj, g, cnt = sp.eval(x, screened)
        stats.grad_calls += 1
        stats.blocks_in_active_set += cnt[0]
        stats.blocks_skipped += cnt[1]
        stats.blocks_unskipped += cnt[2]
        stats.upper_bounds_evaluated += cnt[3]
        stats.history.append(cnt)
        return obj, g

    x = np.zeros(dim)
    if screened:
        sp.init_snapshot(x)  # FastGradDispatcher::init at the zero state (solver.hpp:143)
    t0 = time.perf_counter()
    # maximize: gradient then objective at x0 (lbfgs.hpp:70-71), one fused call
    fx, gx = evaluate(x)
    s_hist, y_hist, rho_hist = [], [], []
    iterations = chunks = 0
    stalled = zero_gradient = converged = False
    for chunk in range(max_outer_loops):
        if stalled or zero_gradient:
            break
        chunks += 1
        for _ in range(snapshot_interval):
            accepted = False
            trial = None
            for attempt in range(2):
                if accepted:
                    break
                if attempt == 1:
                    if not s_hist:
                        break
                    s_hist.clear()
                    y_hist.clear()
                    rho_hist.clear()
                q = gx.copy()  # two-loop recursion (lbfgs.hpp:107-123)
                k = len(s_hist)
                al = [0.0] * k
                for i in range(k - 1, -1, -1):
                    al[i] = rho_hist[i] * sp.dot(s_hist[i], q)
                    q -= al[i] * y_hist[i]
                if k > 0:
                    yy = sp.dot(y_hist[-1], y_hist[-1])
                    if yy > 0.0:
                        q *= sp.dot(s_hist[-1], y_hist[-1]) / yy
                for i in range(k):
                    b = rho_hist[i] * sp.dot(y_hist[i], q)
                    q += (al[i] - b) * s_hist[i]
                d = q
                dir_slope = sp.dot(gx, d)
                if not dir_slope > 0.0:  # lbfgs.hpp:126-135
                    s_hist.clear()
                    y_hist.clear()
                    rho_hist.clear()
                    d = gx.copy()
                    dir_slope = sp.dot(gx, gx)
                    if dir_slope == 0.0:
                        zero_gradient = True
                        break
                f0 = fx
                armijo = wolfe_c1 * dir_slope

                def at(t):
                    xt = x + t * d
                    ft, gt = evaluate(xt)
                    return {"t": t, "value": ft, "slope": sp.dot(gt, d), "x": xt, "grad": gt}

                def sufficient(pt):
                    return pt["value"] >= f0 + armijo * pt["t"]

                def curvature_ok(pt):
                    return abs(pt["slope"]) <= wolfe_c2 * dir_slope

                t_init = 1.0
                if iterations == 0:
                    dn = sp.norm(d)
                    if dn > 0.0:
                        t_init = 1.0 / dn
                have_bracket = False
                lo = {"t": 0.0, "value": f0, "slope": dir_slope, "x": None, "grad": None}
                hi_t = 0.0
                t = t_init
                prev = lo
                for i in range(max_bracket):  # bracketing (lbfgs.hpp:163-183)
                    trial = at(t)
                    if not sufficient(trial) or (i > 0 and trial["value"] <= prev["value"]):
                        lo, hi_t, have_bracket = prev, trial["t"], True
                        break
                    if curvature_ok(trial):
                        accepted = True
                        break
                    if trial["slope"] <= 0.0:
                        lo, hi_t, have_bracket = trial, prev["t"], True
                        break
                    prev = trial
                    t *= 2.0
                if not accepted and have_bracket:  # zoom (lbfgs.hpp:185-225)
                    hi_value = math.nan
                    for _ in range(max_zoom):
                        cand = 0.5 * (lo["t"] + hi_t)
                        if math.isfinite(hi_value):
                            dt = hi_t - lo["t"]
                            denom = 2.0 * (lo["value"] + lo["slope"] * dt - hi_value)
                            if denom != 0.0:
                                interp = lo["t"] + lo["slope"] * dt * dt / denom
                                lg, hg = lo["t"] + 0.1 * dt, hi_t - 0.1 * dt
                                if min(lg, hg) <= interp <= max(lg, hg):
                                    cand = interp
                        if cand == lo["t"] or cand == hi_t:
                            break
                        trial = at(cand)
                        if not sufficient(trial) or trial["value"] <= lo["value"]:
                            hi_t, hi_value = cand, trial["value"]
                            continue
                        if curvature_ok(trial):
                            accepted = True
                            break
                        if trial["slope"] * (hi_t - lo["t"]) <= 0.0:
                            hi_t, hi_value = lo["t"], lo["value"]
                        lo = trial
                    if not accepted and lo["t"] > 0.0:
                        trial, accepted = lo, True
                if not accepted and not have_bracket and prev["t"] > 0.0:
                    trial, accepted = prev, True
            if zero_gradient:
                break
            if not accepted:
                stalled = True
                break
            s = trial["x"] - x  # curvature pair (lbfgs.hpp:243-255)
            y = gx - trial["grad"]
            sy = sp.dot(s, y)
            if sy > 1e-10 * sp.norm(s) * sp.norm(y):
                if len(s_hist) == memory:
                    s_hist.pop(0)
                    y_hist.pop(0)
                    rho_hist.pop(0)
                s_hist.append(s)
                y_hist.append(y)
                rho_hist.append(1.0 / sy)
            x, gx, fx = trial["x"], trial["grad"], trial["value"]
            iterations += 1
        if stalled:
            break
        if screened:  # chunk hook: FastGradDispatcher::refresh (solver.hpp:212-216)
            sp.refresh(x, use_active)
        if sp.inf_norm(gx) <= grad_tol:
            converged = True
            break
    wall = time.perf_counter() - t0
    if not converged:
        converged = sp.inf_norm(gx) <= grad_tol
    return ShardedResult(x, fx, iterations, chunks, converged, stalled and not converged, stats,
                         wall)
