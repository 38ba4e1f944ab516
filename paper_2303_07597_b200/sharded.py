"""Column-sharded solve across GPUs.

Rank p of P owns the column block J_p of the cost and evaluates it on its own
GPU through a shard context (``gsot_create_shard``: cost[:, J_p], a = 0,
b[J_p]). alpha is replicated on every rank, beta is sharded. The evaluation's
one exchange step is a sum all-reduce of m + 1 doubles per call (plus the
counters and the beta part of the line-search slope):

* the shard's ``grad[0, m)`` is minus its plan row sums (a = 0), so
  grad_alpha = a + sum_p (-rowsum_p)                    (dual.hpp:91, :96);
* grad_beta_p is complete on its rank                   (dual.hpp:97-98);
* objective = a.alpha + sum_p (b_p.beta_p - psi_p)      (dual.hpp:51).

The L-BFGS ascent follows the reference's ``maximize`` (lbfgs.hpp:61-274):
t_init, strong-Wolfe bracketing and zoom, the retry from steepest ascent, the
curvature-pair test, chunk hooks and the infinity-norm stop test. Its
direction is the same L-BFGS matrix in the compact representation (Byrd,
Nocedal & Schnabel 1994; the device solver's fast mode):
d = gam g + S p - Y (gam w), w = R^-1 S'g, p = R^-T ((D + gam Y'Y) w - gam Y'g),
R = triu(S'Y), so all the dot products of one direction are independent and
travel in ONE all-reduce; the k x k algebra runs on the host. Every dot is
the alpha part (identical on every rank) plus the all-reduced beta parts and
the infinity norm an all-reduced max, so every rank takes the same decisions.

Vectors live where the evaluations do: device tensors (torch, on the rank's
GPU) for shard contexts, numpy arrays for the test evaluators. Screening is
per rank (the blocks of column shard J_p); the GradStats counters are
all-reduced sums. The collective is ``torch.distributed`` (NCCL on GPU ranks,
gloo for the tests).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
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
    """Sum / max all-reduce over torch.distributed (identical results on every
    rank) of numpy arrays or torch tensors; the result has the input's kind."""

    def __init__(self, pg=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.on = pg is not None and dist.is_initialized() and dist.get_world_size() > 1
        self.nccl = self.on and dist.get_backend() == "nccl"

    def allreduce(self, v, op: str = "sum"):
        torch = self.torch
        is_np = isinstance(v, np.ndarray)
        if not self.on:
            return np.array(v, dtype=np.float64, copy=True) if is_np else v.clone()
        t = torch.from_numpy(np.ascontiguousarray(v, np.float64)) if is_np else v
        if self.nccl and not t.is_cuda:
            t = t.cuda()
        elif not self.nccl and t.is_cuda:
            t = t.cpu()
        else:
            t = t.clone()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX)
        if is_np:
            return t.cpu().numpy()
        return t.to(v.device)


class _Numpy:
    """Vector backend: host numpy arrays (test evaluators)."""

    def zeros(self, n):
        return np.zeros(n)

    def copy(self, v):
        return v.copy()

    def host(self, v):
        return np.asarray(v)

    def stack(self, vs):
        return np.stack(vs)

    def gram(self, A, B):  # (ka, kb) local dot products, to the host
        return A @ B.T

    def combo(self, coef, A):  # sum_i coef_i A_i
        return np.asarray(coef) @ A

    def absmax(self, v):
        return float(np.max(np.abs(v))) if v.size else 0.0


class _Torch:
    """Vector backend: float64 tensors on the rank's GPU."""

    def __init__(self):
        import torch

        self.torch = torch

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device="cuda")

    def copy(self, v):
        return v.clone()

    def host(self, v):
        return v.cpu().numpy()

    def stack(self, vs):
        return self.torch.stack(vs)

    def gram(self, A, B):
        return (A @ B.T).cpu().numpy()

    def combo(self, coef, A):
        return self.torch.from_numpy(np.asarray(coef, np.float64)).to(A.device) @ A

    def absmax(self, v):
        return float(v.abs().max().item()) if v.numel() else 0.0


# ---------------------------------------------------------------------------
# The device-resident sharded solve (gsot_comm_*): the rank's
# shard context runs the library's own solver (CUDA graphs, compact L-BFGS,
# PDL chain) and sums, per device sequence, the gradient head and a 16-double
# scalar tail over the ranks (plus the L-BFGS dots inside each direction
# update) through NCCL on the context stream, or through a host transport.
# The host-driven driver below (solve_sharded) stays as the readable
# restatement the CPU tests check against the oracle.


def shard_context_from_device(d_cost_ptr: int, m: int, n_shard: int, sizes, a, b_block,
                              gamma: float, mu: float, rank: int) -> "G.Context":
    """Rank `rank`'s shard context: a on rank 0, zeros elsewhere, so the sum of
    the shards' gradient heads is a - sum_p rowsum_p and of their objectives
    a.alpha + sum_p (b_p.beta_p - psi_p) (dual.hpp:51, :91-98)."""
    a_p = np.ascontiguousarray(a, np.float64) if rank == 0 else np.zeros(len(a))
    return G.Context.shard_from_device(d_cost_ptr, m, n_shard, sizes, a_p, b_block, gamma, mu)


def shard_context_from_arrays(cost_block, sizes, a, b_block, gamma: float, mu: float,
                              rank: int) -> "G.Context":
    a_p = np.ascontiguousarray(a, np.float64) if rank == 0 else np.zeros(len(a))
    return G.Context.shard_from_arrays(cost_block, sizes, a_p, b_block, gamma, mu)


def attach_comm(ctx: "G.Context", pg=None, transport: str = "auto") -> str:
    """Attach this rank's communicator to its shard context. transport "nccl":
    an NCCL communicator (the unique id broadcast over `pg`, or made locally at
    world size 1); "host": sums through torch.distributed on host memory (gloo);
    "auto": NCCL unless the process group is gloo. Returns the transport used."""
    import torch.distributed as dist

    on = pg is not None and dist.is_initialized()
    world = dist.get_world_size() if on else 1
    rank = dist.get_rank() if on else 0
    if transport == "auto":
        transport = "host" if on and dist.get_backend() == "gloo" else "nccl"
    if transport == "nccl":
        uid = [G.nccl_unique_id() if rank == 0 else None]
        if on and world > 1:
            dist.broadcast_object_list(uid, src=0)
        ctx.attach_nccl(uid[0], world, rank)
        return "nccl"

    import torch

    def allreduce(buf: np.ndarray, op: int) -> None:
        if world == 1:
            return
        t = torch.from_numpy(buf)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM)

    ctx.attach_host(world, rank, allreduce)
    return "host"


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
    """One rank's share of an instance: the shard context (or, in tests, an
    evaluator) and the global marginal a. evaluator(x_local, screened) ->
    (objective_p, grad_local, counters4) on numpy vectors."""

    def __init__(self, cost_block, sizes, a, b_block, gamma: float, mu: float, comm: Comm,
                 evaluator=None, ctx=None):
        self.m = int(np.asarray(a).size)
        self.n_p = int(np.asarray(b_block).size)
        self.comm = comm
        self.evaluator = evaluator
        self.ctx = ctx  # a prebuilt shard context (Context.shard_from_device)
        if evaluator is None and ctx is None:
            self.ctx = G.Context.shard_from_arrays(cost_block, sizes, np.zeros(self.m), b_block,
                                                   gamma, mu)
        self.be = _Numpy() if evaluator is not None else _Torch()
        self.a = np.ascontiguousarray(a, np.float64)
        if evaluator is None:
            import torch

            self.a = torch.from_numpy(self.a).cuda()
            self.grad = torch.empty(self.m + self.n_p, dtype=torch.float64, device="cuda")

    def close(self) -> None:
        if self.ctx is not None:
            self.ctx.close()
            self.ctx = None

    def _dot_a(self, u, v) -> float:
        return float(u[: self.m] @ v[: self.m])

    # ---- evaluation: one all-reduce of m + 1 doubles (+ counters, slope part)
    def eval(self, x, screened: bool, d=None):
        """(objective, gradient, counters, slope g.d or None)."""
        m = self.m
        if self.evaluator is not None:
            obj_p, g, cnt = self.evaluator(x, screened)
            tail = np.array([obj_p, *cnt, float(g[m:] @ d[m:]) if d is not None else 0.0])
            buf = np.concatenate([g[:m], tail])
        else:
            import torch

            torch.cuda.current_stream().synchronize()  # x written on this stream
            obj = C.c_double()
            cs = _lib.CallStats()
            G._raise(_lib.lib().gsot_eval_device(self.ctx.handle, C.c_void_p(x.data_ptr()),
                                                 1 if screened else 0, C.byref(obj),
                                                 C.c_void_p(self.grad.data_ptr()), C.byref(cs)))
            g = self.grad.clone()
            cnt = (cs.in_active, cs.skipped, cs.unskipped, cs.upper_bounds)
            tail = torch.tensor([obj.value, *cnt, 0.0], dtype=torch.float64, device="cuda")
            if d is not None:
                tail[5] = g[m:] @ d[m:]
            buf = torch.cat([g[:m], tail])
        red = self.comm.allreduce(buf, "sum")
        g[:m] = self.a + red[:m]
        # the alpha parts next to the reduced tail: one transfer to the host
        parts = [self.a @ x[:m], (g[:m] @ d[:m]) if d is not None else self.a[:1].sum() * 0.0]
        if self.evaluator is None:
            import torch

            tl = torch.cat([red[m:], torch.stack(parts)]).cpu().numpy()
        else:
            tl = np.concatenate([red[m:], np.array([float(v) for v in parts])])
        obj = float(tl[6] + tl[0])
        slope = None if d is None else float(tl[7] + tl[5])
        return obj, g, tuple(int(v) for v in tl[1:5]), slope

    def init_snapshot(self, x) -> None:
        if self.ctx is not None:
            self.ctx.init_snapshot(self.be.host(x))

    def refresh(self, x, use_active_set: bool) -> None:
        if self.ctx is not None:
            self.ctx.refresh(self.be.host(x), use_active_set)

    # ---- distributed dot products on [alpha; beta_p]
    def dots(self, pairs) -> list:
        """[u . v for (u, v) in pairs] with one all-reduce of the beta parts."""
        m = self.m
        if self.evaluator is None:
            import torch

            loc = torch.stack([u[m:] @ v[m:] for u, v in pairs])
            al = torch.stack([u[:m] @ v[:m] for u, v in pairs])
            red = self.comm.allreduce(loc, "sum")
            return (al + red).cpu().numpy().tolist()
        loc = np.array([float(u[m:] @ v[m:]) for u, v in pairs])
        red = self.comm.allreduce(loc, "sum")
        return [self._dot_a(u, v) + r for (u, v), r in zip(pairs, red)]

    def gram(self, A, B):
        """A B' for stacked vectors (rows), one all-reduce of the beta parts."""
        m = self.m
        red = self.comm.allreduce(self.be.gram(A[:, m:], B[:, m:]), "sum")
        return self.be.gram(A[:, :m], B[:, :m]) + red

    def inf_norm(self, u) -> float:
        m = self.m
        loc = self.be.absmax(u[m:])
        return max(self.be.absmax(u[:m]), float(self.comm.allreduce(np.array([loc]), "max")[0]))


@dataclass
class ShardedResult:
    x: np.ndarray  # this rank's [alpha; beta_p] (host copy)
    objective: float
    iterations: int
    outer_loops: int
    converged: bool
    line_search_failed: bool
    stats: ShardStats
    wall_seconds: float


def _compact_direction(sp: ShardedProblem, s_hist, y_hist, g):
    """H g for the L-BFGS matrix of the pairs (oldest first) in the compact
    form with ONE all-reduce (all the dots of the direction); returns (d, g.d)."""
    be = sp.be
    k = len(s_hist)
    V = be.stack(s_hist + y_hist + [g])  # rows: s_0..s_k-1, y_0..y_k-1, g
    Gm = sp.gram(V, V)
    SY, YY = Gm[:k, k:2 * k], Gm[k:2 * k, k:2 * k]
    u, v, gg = Gm[:k, 2 * k], Gm[k:2 * k, 2 * k], Gm[2 * k, 2 * k]
    gam = SY[k - 1, k - 1] / YY[k - 1, k - 1] if YY[k - 1, k - 1] > 0.0 else 1.0  # lbfgs.hpp:116-119
    R = np.triu(SY)
    w = np.zeros(k)
    for i in range(k - 1, -1, -1):  # back substitution, R w = S'g
        w[i] = (u[i] - R[i, i + 1:] @ w[i + 1:]) / R[i, i]
    z = np.diag(SY) * w + gam * (YY @ w) - gam * v
    p = np.zeros(k)
    for i in range(k):  # forward substitution, R' p = z
        p[i] = (z[i] - R[:i, i] @ p[:i]) / R[i, i]
    d = gam * g + be.combo(p, V[:k]) - be.combo(gam * w, V[k:2 * k])
    slope = gam * gg + float(p @ u) - gam * float(w @ v)  # g.d from the reduced dots
    return d, slope


def solve_sharded(sp: ShardedProblem, mode: int = 1, snapshot_interval: int = 10,
                  grad_tol: float = 1e-6, max_outer_loops: int = 200, memory: int = 10,
                  wolfe_c1: float = 1e-4, wolfe_c2: float = 0.9, max_bracket: int = 40,
                  max_zoom: int = 12) -> ShardedResult:
    """solve_baseline (mode 0) / solve_fast (1) / fast_no_lower_bound (2)
    (solver.hpp:92-258) with maximize (lbfgs.hpp:61-274) over the shards."""
    be = sp.be
    screened = mode in (1, 2)
    use_active = mode == 1
    dim = sp.m + sp.n_p
    stats = ShardStats()

    def evaluate(x, d=None):
        obj, g, cnt, slope = sp.eval(x, screened, d)
        stats.grad_calls += 1
        stats.blocks_in_active_set += cnt[0]
        stats.blocks_skipped += cnt[1]
        stats.blocks_unskipped += cnt[2]
        stats.upper_bounds_evaluated += cnt[3]
        stats.history.append(cnt)
        return obj, g, slope

    x = be.zeros(dim)
    if screened:
        sp.init_snapshot(x)  # FastGradDispatcher::init at the zero state (solver.hpp:143)
    t0 = time.perf_counter()
    fx, gx, _ = evaluate(x)  # gradient, then objective at x0 (lbfgs.hpp:70-71): one call
    s_hist, y_hist = [], []
    iterations = chunks = 0
    stalled = zero_gradient = converged = False
    for _chunk in range(max_outer_loops):
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
                if s_hist:
                    d, dir_slope = _compact_direction(sp, s_hist, y_hist, gx)
                else:
                    d = be.copy(gx)
                    dir_slope = sp.dots([(gx, gx)])[0]
                if not dir_slope > 0.0:  # lbfgs.hpp:126-135
                    s_hist.clear()
                    y_hist.clear()
                    d = be.copy(gx)
                    dir_slope = sp.dots([(gx, gx)])[0]
                    if dir_slope == 0.0:
                        zero_gradient = True
                        break
                f0 = fx
                armijo = wolfe_c1 * dir_slope

                def at(t):
                    xt = x + t * d
                    ft, gt, st = evaluate(xt, d)
                    return {"t": t, "value": ft, "slope": st, "x": xt, "grad": gt}

                def sufficient(pt):
                    return pt["value"] >= f0 + armijo * pt["t"]

                def curvature_ok(pt):
                    return abs(pt["slope"]) <= wolfe_c2 * dir_slope

                t_init = 1.0
                if iterations == 0:
                    dn = math.sqrt(sp.dots([(d, d)])[0])
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
                    for _z in range(max_zoom):
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
            sy, ss, yy = sp.dots([(s, y), (s, s), (y, y)])
            if sy > 1e-10 * math.sqrt(ss) * math.sqrt(yy):
                if len(s_hist) == memory:
                    s_hist.pop(0)
                    y_hist.pop(0)
                s_hist.append(s)
                y_hist.append(y)
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
    return ShardedResult(be.host(x).copy(), fx, iterations, chunks, converged,
                         stalled and not converged, stats, wall)
