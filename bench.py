#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 group-sparse OT dual solver.

Metric (BASELINE.json): dual-grad evals/s inside the L-BFGS solve, achieved
HBM GB/s of the dominant kernel (fraction of the measured peak), and the
L-BFGS solve time for all five configs.

Workload (the largest single-GPU config, BASELINE.json configs[4], "large"):
m = 100,000 source rows in L = 200 classes of 500, n = 50,000 targets,
d = 512, gamma = 0.1, mu = 0.5, 300 L-BFGS iterations (snapshot interval 10,
memory 10, grad_tol 1e-12 so the solve runs to budget), fast mode
(upper-bound skipping + lower-bound active set). The 40 GB cost matrix is
resident in HBM. One step = one complete solve from x0 = 0; value =
objective+gradient evaluations per second over the K timed solves (device
time from CUDA events on the solver stream). The cost exceeds the 126 MB L2,
so no flush is needed between steps.

Also on the same line, timed inside the same clock-sampled region:
  configs   solve ms and evals/s of configs 1-4 (config 3 at mu 0.05, 0.2
            and 1.0) next to the headline config;
  e2e       the same metric through the C ABI with HOST buffers: every step
            uploads C, a, b from pinned host memory (gsot_create: H2D +
            on-device validation + re-layout), solves, downloads x and frees
            the context (warm context cache; one cold step reported apart);
  roofline  the dominant kernel's algorithmic bytes / its mean launch time;
  cpu_baseline  the reference itself (oracle/_ref) on 1 pinned core over a
            column sample of one evaluation at recorded mid-solve states.

    python bench.py [--gpus N --steps K --warmup W] [--config C] [--impl reference]

--gpus N > 1 re-launches itself under torch.distributed.run (one rank per
GPU) unless it already runs under it; at N > 1 the instance is column-sharded
across the ranks (one all-reduce of m + 1 doubles per evaluation, DESIGN.md
§8) and value counts each global evaluation once (strong scaling).

--impl reference: the unmodified reference (oracle/_ref: the reference
headers compiled against the Eigen shim) timed on the host cores on the same
config, every core running its own column sample of one evaluation (the
reference's dense dual_objective + the screened dual_gradient after a
dispatcher refresh, at the recorded mid-solve states of tests/golden/): a
full reference evaluation of config 5 streams 40 GB on one core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(1, os.path.join(ROOT, "tests"))  # CPU checkers (reference arm / cpu_baseline)

CONFIGS = {  # cfg: (gamma, mu, iterations)  -- BASELINE.json configs / SURVEY.md §8(d)
    1: (1.0, 0.1, 100),
    2: (0.1, 0.5, 200),
    3: (0.1, 0.2, 200),
    4: (0.05, 0.3, 200),
    5: (0.1, 0.5, 300),
}
MU_SWEEP3 = (0.05, 0.2, 1.0)  # BASELINE.json configs[2]: mu sweep of config 3
METRIC = "dual-grad evals/s (fused objective+gradient inside L-BFGS, fast mode)"
STATES = os.path.join(ROOT, "tests", "golden", "states_cfg{}.npz")
KIND_NAMES = {0: "k_eval", 1: "k_snapshot", 2: "k_bounds", 3: "k_active", 4: "k_finalize",
              5: "lbfgs", 6: "k_delta", 7: "misc"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    (pynvml, every 5 ms, from a thread; device-wide counters, no CUDA
    interaction), else nvidia-smi every 100 ms. begin()/end() bracket the
    timed region; only samples taken between them are reported."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self.on = False
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.nvml = (N, h, mx, bits)
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _poll_nvml(self):
        N, h, mx, bits = self.nvml
        while not self.stop_ev.is_set():
            if self.on:
                try:
                    sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((float(sm), float(mx),
                                         {nm for nm, b in bits.items() if r & b}))
                except Exception:
                    pass
            time.sleep(0.005)

    def _read_smi(self):
        for ln in self.proc.stdout:
            if not self.on:
                continue
            parts = [p.strip() for p in ln.strip().split(",")]
            if len(parts) < 7:
                continue
            try:
                sm, mx = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            self.samples.append((sm, mx, {nm for nm, v in zip(self.NAMES, parts[3:7])
                                          if v.lower() == "active"}))

    def begin(self):
        self.on = True

    def end(self):
        self.on = False

    def stop(self):
        self.on = False
        self.stop_ev.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.samples:
            return None
        sm = [x[0] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples])
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml else "nvidia-smi"}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        pg = dist
    return world, rank, local, pg


def allreduce(pg, value: float, op: str) -> float:
    if pg is None:
        return value
    import torch

    dev = "cuda" if pg.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX if op == "max" else pg.ReduceOp.SUM)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def ncu_traffic(kernel: str, cfg: int):
    """DRAM bytes per launch of `kernel` from one ncu --set full capture of
    this config's bench command (profiles/ncu_traffic_cfgC.json), or None."""
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{cfg}.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    # the fused evaluation is k_eval or, for instances with tall groups, k_eval_q
    ent = d.get(kernel) or (d.get("k_eval_q") if kernel == "k_eval" else None)
    return None if ent is None else ent.get("dram_bytes_per_launch")


def solve_kw(iters: int) -> dict:
    return dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=iters // 10,
                lbfgs_memory=10, history_cap=0)


# ------------------------------------------------------- CPU timing samples


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_problems(cfg: int, parts: int, threads: int):
    """Column samples of config `cfg` for timing the reference on the host:
    the recorded sample columns (tests/golden/states_cfgC.npz, 512 columns
    evenly spread over n) split into `parts` disjoint sub-instances, each the
    full m rows x its columns, built with the CPU checker (oracle C: the
    config's features, cost_matrix of the sampled columns divided by the
    recorded max C -- bitwise the device instance's entries), with the
    recorded states (x_a, x_s, x) restricted to those columns. Returns
    ([(Problem, x_a, x_s, x)], n, refreshes per evaluation of a device solve)."""
    import ctypes as C

    import numpy as np
    from oracle_bindings import Oracle, Problem

    st = np.load(STATES.format(cfg))
    o = Oracle()
    m, n, L, d = (C.c_int64(), C.c_int64(), C.c_int32(), C.c_int64())
    o.lib.go_config_shape(cfg, C.byref(m), C.byref(n), C.byref(L), C.byref(d))
    m, n, L, d = m.value, n.value, L.value, d.value
    src, tgt = np.empty((m, d)), np.empty((n, d))
    sizes, a, b = np.empty(L, np.int32), np.empty(m), np.empty(n)
    o.lib.go_config_features(C.c_int(cfg), C.c_uint64(cfg),
                             *[v.ctypes.data_as(C.c_void_p) for v in (src, tgt, sizes, a, b)])
    cols, cmax = st["cols"], float(st["cmax"])
    gamma, mu, _ = CONFIGS[cfg]
    out = []
    for idx in np.array_split(np.arange(len(cols)), parts):
        J = cols[idx]
        tj = np.ascontiguousarray(tgt[J])
        cost = np.empty((m, len(J)), order="F")
        o.lib.go_cost_matrix_par(src.ctypes.data_as(C.c_void_p), C.c_int64(m),
                                 tj.ctypes.data_as(C.c_void_p), C.c_int64(len(J)), C.c_int64(d),
                                 cost.ctypes.data_as(C.c_void_p), C.c_int(threads))
        cost /= cmax  # data_io.hpp:162-165
        prob = Problem(cost, sizes, a, b[J], gamma, mu)
        xs = [(st[f"alpha_{k}"], st[f"beta_{k}"][idx]) for k in "asx"]
        out.append((prob, *xs))
    return out, n, float(st["refreshes_per_eval"]) if "refreshes_per_eval" in st else 0.08


def reference_eval_rate(samples, n: int, refresh_per_eval: float, reps: int, cores=None):
    """Every sample timed by the reference (RefLib.time_eval) on its own
    thread (ctypes releases the GIL), thread i pinned to cores[i]. Per
    sample, one evaluation of its columns costs dual_objective + the
    screened dual_gradient + refresh_per_eval x one dispatcher refresh (half
    the timed init + refresh: a snapshot and an active-set build). Returns
    (evals/s of the whole problem at the samples' aggregate column rate,
    wall seconds, details)."""
    from oracle_bindings import RefLib

    lib = RefLib()
    res = [None] * len(samples)

    def run(i):
        if cores is not None:
            os.sched_setaffinity(0, {cores[i]})  # this thread only (Linux)
        prob, xa, xs, x = samples[i]
        res[i] = lib.time_eval(prob, xa, xs, x, reps)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=run, args=(i,)) for i in range(len(samples))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    cols_per_s, t_obj, t_grad, t_ref = 0.0, 0.0, 0.0, 0.0
    for (prob, *_), (times, cnt, obj) in zip(samples, res):
        per_eval = (times[0] + times[1] + refresh_per_eval * 0.5 * times[2]) / reps
        cols_per_s += prob.n / per_eval
        t_obj, t_grad, t_ref = t_obj + times[0], t_grad + times[1], t_ref + times[2]
    return cols_per_s / n, wall, {"objective_s": t_obj, "gradient_s": t_grad,
                                  "init_refresh_s": t_ref,
                                  "columns": int(sum(p.n for p, *_ in samples))}


def run_reference(args, world, rank, pg):
    if rank != 0:
        return 0
    from oracle_bindings import ref_available

    if not ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libgroupot_ref.so not built"}))
        return 0
    if not os.path.exists(STATES.format(args.config)):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no recorded states for config {args.config} (tools/record_states.py)"}))
        return 0
    cores = sorted(os.sched_getaffinity(0))
    samples, n, rpe = sample_problems(args.config, len(cores), len(cores))
    reps = args.ref_reps
    for _ in range(args.warmup):
        reference_eval_rate(samples, n, rpe, reps, cores)
    vals, walls, det = [], [], None
    for _ in range(args.steps):
        v, w, det = reference_eval_rate(samples, n, rpe, reps, cores)
        vals.append(v)
        walls.append(w)
    value = statistics.mean(vals)
    unit = "evals/s"
    cfg = args.config
    sample = (f"{len(cores)} threads (one pinned per core, {cpu_model()}), each timing the "
              f"reference on its own column sample ({det['columns']} of n = {n} columns in all, "
              f"all m rows) x {reps} rep(s) per step: dual_objective (dense, solver.hpp:161-164) "
              f"+ screened dual_gradient after FastGradDispatcher init + refresh at recorded "
              f"mid-solve states (iterations 190 / 200 / 210 of a device solve), plus "
              f"{rpe:.3f} refreshes per evaluation; evals/s = aggregate column rate / n")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": unit,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(walls),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY.md §8(d) recipe, seed = config id)",
        "config": {"workload": f"config {cfg}: reference per-evaluation column sample "
                               f"(partial: the reference's full solve of this config takes hours "
                               f"on the host)",
                   "m": samples[0][0].m, "n": n, "L": samples[0][0].L,
                   "gamma": CONFIGS[cfg][0], "mu": CONFIGS[cfg][1]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": len(cores), "kind": "reference",
                         "cpu": cpu_model(), "sample": sample, "partial": True},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cfg: int):
    """The reference (oracle/_ref) on ONE pinned core over all 512 sample
    columns of one evaluation at the recorded states, repeated to ~10 s."""
    from oracle_bindings import ref_available

    if not ref_available() or not os.path.exists(STATES.format(cfg)):
        return None
    cores = sorted(os.sched_getaffinity(0))
    core = cores[-1]
    samples, n, rpe = sample_problems(cfg, 1, len(cores))
    v1, w1, _ = reference_eval_rate(samples, n, rpe, 1, [core])
    reps = max(1, min(20, int(10.0 / max(w1, 1e-3))))
    v, w, det = reference_eval_rate(samples, n, rpe, reps, [core])
    return {"value": v, "unit": "evals/s", "cores": 1, "kind": "reference", "cpu": cpu_model(),
            "pinned_core": core, "partial": True,
            "sample": f"reference dual_objective + screened dual_gradient (after dispatcher "
                      f"init + refresh) at recorded mid-solve states over {det['columns']} of "
                      f"{n} columns (all rows), {reps} reps, {w:.1f} s on 1 pinned core; "
                      f"plus {rpe:.3f} refreshes per evaluation; evals/s = column rate / n"}


# ---------------------------------------------------------------- ours


def timed_solves(ctx, kw: dict, steps: int) -> dict:
    ctx.timer_start()
    out = {"calls": 0, "iters": 0, "blocks": 0, "tasks": 0, "solve_ms": [], "refreshes": 0}
    for _ in range(steps):
        t0 = time.perf_counter()
        r = ctx.solve(**kw)
        out["solve_ms"].append(1e3 * (time.perf_counter() - t0))
        out["calls"] += r["grad_calls"]
        out["iters"] += r["iterations"]
        out["blocks"] += r["eval_blocks"]
        out["tasks"] += r["eval_tasks"]
        out["refreshes"] += r["outer_loops"]
        out["objective"] = r["objective"]
        out["x"] = r["x"]
    out["ms"] = ctx.timer_stop()
    return out


def configs_table(args, head_cfg: int, head: dict, clocks) -> dict:
    """Solve time and evals/s of every BASELINE config on this GPU (the
    headline config from its own K timed solves; config 3 at each mu of the
    sweep), each timed with CUDA events inside the clock-sampled region."""
    import paper_2303_07597_b200 as G

    table = {}
    for cfg in (1, 2, 3, 4, 5):
        gamma, mu0, iters = CONFIGS[cfg]
        mus = MU_SWEEP3 if cfg == 3 else (mu0,)
        if cfg == head_cfg and len(mus) == 1:
            table[f"config{cfg}"] = {
                "mu": mu0, "solve_ms": head["ms"] / args.steps, "solves": args.steps,
                "evals_per_solve": head["calls"] / args.steps,
                "evals_per_s": head["calls"] / (head["ms"] / 1e3),
                "iterations": head["iters"] / args.steps}
            continue
        if cfg == 5 and head_cfg != 5 and args.skip_large:
            continue
        reps = 5 if cfg <= 2 else 2
        ctx = G.Context.from_config(cfg, cfg, gamma, mus[0])
        for mu in mus:
            ctx.set_params(gamma, mu)
            kw = solve_kw(iters)
            ctx.solve(**kw)  # warm-up (graph capture)
            clocks.begin()
            r = timed_solves(ctx, kw, reps)
            clocks.end()
            key = f"config{cfg}" + (f"_mu{mu:g}" if len(mus) > 1 else "")
            table[key] = {"mu": mu, "solve_ms": r["ms"] / reps, "solves": reps,
                          "evals_per_solve": r["calls"] / reps,
                          "evals_per_s": r["calls"] / (r["ms"] / 1e3),
                          "iterations": r["iters"] / reps,
                          "blocks_computed_frac": r["blocks"] / (r["calls"] * ctx.L * ctx.n)}
            if cfg in args.exact_configs:
                table[key]["exact"] = exact_solve(ctx, iters, clocks)
        ctx.close()
        G.cache_clear()
    return table


def exact_solve(ctx, iters: int, clocks) -> dict:
    """Exact-order mode (GSOT_SOLVE_EXACT: every sum in the reference's own
    order, so the trajectory is bitwise the reference's -- tests/
    test_gpu_exact.py): one warm-up and one timed solve on the context."""
    kw = dict(solve_kw(iters), exact=True)
    ctx.solve(**kw)
    clocks.begin()
    r = timed_solves(ctx, kw, 1)
    clocks.end()
    return {"solve_ms": r["ms"], "evals_per_s": r["calls"] / (r["ms"] / 1e3),
            "evals_per_solve": r["calls"], "iterations": r["iters"]}


def run_ours(args, world, rank, local, pg):
    if world > 1:
        return run_sharded(args, world, rank, local, pg)
    import paper_2303_07597_b200 as G

    G.set_device(local)
    cfg = args.config
    gamma, mu, iters = CONFIGS[cfg]
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    kw = solve_kw(iters)
    for _ in range(args.warmup):
        ctx.solve(**kw)

    # ---- timed region: K solves on the resident instance, no instrumentation
    # (event nodes between kernels would break the programmatic launch chain)
    ctx.profile(False)
    launches0 = ctx.kernel_launches()
    clocks = ClockSampler(local)
    clocks.start()
    clocks.begin()
    head = timed_solves(ctx, kw, args.steps)
    clocks.end()
    launches = ctx.kernel_launches() - launches0
    value = head["calls"] / (head["ms"] / 1e3)

    # ---- roofline pass: the same solves again with CUDA events around the
    # two HBM-streaming kernels (eval, snapshot) on the solver stream
    nprof = min(args.steps, 5)
    ctx.profile((1 << 0) | (1 << 1))
    ctx.solve(**kw)  # capture the profiled graphs outside the measured pass
    ctx.profile_reset()
    ctx.profile((1 << 0) | (1 << 1))
    clocks.begin()
    ctx.timer_start()
    for _ in range(nprof):
        ctx.solve(**kw)
    ms_prof = ctx.timer_stop()
    clocks.end()
    ctx.profile(False)
    kinds = {}
    for k, name in KIND_NAMES.items():
        kms, kbytes, kn = ctx.profile_read(k)
        if kn:
            kinds[name] = {"ms": kms, "bytes": kbytes, "launches": kn}
    peak, peak_kind = peaks()
    cand = {k: v for k, v in kinds.items() if v["bytes"] > 0}
    dom = max(cand, key=lambda k: cand[k]["ms"])
    d = cand[dom]
    achieved = (d["bytes"] / d["launches"]) / (d["ms"] / d["launches"] / 1e3) / 1e9
    regimes = None
    if dom == "k_eval":
        nms, nbytes, nn = ctx.profile_read(8)
        tot = kinds["k_eval"]
        regimes = {}
        for name, (rms, rbytes, rn) in (("near_dense", (nms, nbytes, nn)),
                                         ("screened", (tot["ms"] - nms, tot["bytes"] - nbytes,
                                                       tot["launches"] - nn))):
            if rn > 0 and rms > 0:
                a = rbytes / (rms / 1e3) / 1e9
                regimes[name] = {"launches": rn, "bytes_per_launch": rbytes / rn,
                                 "us_per_launch": 1e3 * rms / rn, "achieved": a,
                                 "frac": a / peak, "share_of_eval_time": rms / tot["ms"]}
    fetched = None
    if dom == "k_eval":  # cost bytes actually fetched (8-column quarters) vs the minimum
        _, fbytes, fn = ctx.profile_read(9)
        if fn:
            fetched = {"cost_bytes_per_launch": fbytes / fn,
                       "vs_algorithmic": fbytes / d["bytes"],
                       "what": "64-byte quarter rows the evaluation's TMA copies moved, "
                               "counted by the producer warps (tiles streamed twice count "
                               "twice), over the algorithmic bytes"}
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_kind,
                "traffic": ncu_traffic(dom, cfg),
                "bytes_per_launch": d["bytes"] / d["launches"],
                "ms_per_launch": d["ms"] / d["launches"],
                "share_of_step": d["ms"] / ms_prof,
                "regimes": regimes,
                "fetched": fetched,
                "measured": f"CUDA events around every launch of the kernel on the solver "
                            f"stream, over a second pass of {nprof} solves (the value pass "
                            f"runs uninstrumented)"}
    m_, n_, L_ = ctx.m, ctx.n, ctx.L
    # ---- the parity-pinned (exact-order, bitwise-reference) mode on this config
    exact = exact_solve(ctx, iters, clocks) if cfg in args.exact_configs else None
    ctx.close()
    G.cache_clear()

    # ---- the column-sharded (multi-GPU) code path at N = 1, same config
    shard1 = None
    if not args.no_sharded_n1:
        clocks.begin()
        shard1 = sharded_n1(cfg, head["ms"] / args.steps, head["x"], min(args.steps, 3))
        clocks.end()

    # ---- all five configs (fast and exact-order mode)
    table = configs_table(args, cfg, head, clocks)
    if exact is not None and f"config{cfg}" in table:
        table[f"config{cfg}"]["exact"] = exact
    clk = clocks.stop()

    # ---- e2e through the C ABI with host buffers
    e2e = run_e2e(args, cfg, gamma, mu, kw)

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None if args.no_cpu_baseline else cpu_baseline(cfg)

    steps = args.steps
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "evals/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms"] / steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY.md §8(d) recipe, seed = config id), generated on device",
        "config": {"workload": f"config {cfg}: one fast-mode L-BFGS solve per step "
                               f"({iters} iterations, r=10, memory 10)",
                   "m": m_, "n": n_, "L": L_, "gamma": gamma, "mu": mu,
                   "l2": f"inputs larger than L2 (cost {8 * m_ * n_ / 1e9:.1f} GB > 126 MB), "
                         "no flush",
                   "parallelism": "single GPU"},
        "solve_ms": statistics.median(head["solve_ms"]),
        "evals_per_solve": head["calls"] / steps,
        "iterations_per_solve": head["iters"] / steps,
        "screening": {"blocks_computed_frac": head["blocks"] / (head["calls"] * L_ * n_),
                      "active_lanes_per_task": head["blocks"] / max(head["tasks"], 1)},
        "roofline": roofline,
        "kernels": kinds,
        "gpu_launches": launches,
        "configs": table,
        "sharded_n1": shard1,
        "parity_pinned": None if exact is None else dict(
            exact, mode="exact-order (GSOT_SOLVE_EXACT): the reference's own order of every "
                        "floating-point operation; the solve is bitwise the reference's "
                        "trajectory (tests/test_gpu_exact.py), unlike fast mode whose "
                        "re-associated sums diverge on these unconverged solves"),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def run_e2e(args, cfg, gamma, mu, kw):
    """The bench metric through the public C ABI from pinned host memory:
    per step gsot_create (H2D + device validation + re-layout) + gsot_solve
    + x download + gsot_destroy. Steps reuse the device state parked by the
    previous step's destroy (the warm context cache); one cold step (cache
    cleared first: allocation + graph capture) is reported apart."""
    import ctypes as C

    import torch

    import paper_2303_07597_b200 as G

    m, n, L, d = G.config_shape(cfg)
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    host = torch.empty((n, m), dtype=torch.float64, pin_memory=torch.cuda.is_available())
    cost = host.numpy().T  # (m, n) Fortran view: column-major as the ABI expects
    dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
    G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(
        src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 1,
        C.c_void_p(dev.data_ptr())))
    host.copy_(dev)
    del dev
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    def step():
        t0 = time.perf_counter()
        c2 = G.Context.from_arrays(cost, sizes, a, b, gamma, mu)
        r = c2.solve(**kw)
        _ = r["x"].sum()  # x is downloaded by gsot_solve into host memory
        c2.close()
        return time.perf_counter() - t0, r["grad_calls"]

    G.cache_clear()
    cold_s, cold_calls = step()  # allocation + graph capture included
    steps = max(2, args.steps // 4)
    times, calls = [], 0
    for _ in range(steps):
        t, c = step()
        times.append(t)
        calls += c
    G.cache_clear()
    del host, cost
    tot = sum(times)
    return {"value": calls / tot, "unit": "evals/s",
            "h2d_bytes_per_step": 8 * m * n + 8 * (m + n) + 4 * L,
            "d2h_bytes_per_step": 8 * (m + n),
            "ms_per_step": 1e3 * tot / steps, "steps": steps,
            "cold_ms": 1e3 * cold_s, "cold_evals_per_s": cold_calls / cold_s,
            "what": "gsot_create from pinned host cost (H2D + device validation + re-layout) "
                    "+ gsot_solve + x download + gsot_destroy; warm context cache (each "
                    "destroy parks the device buffers and captured graphs, the next create of "
                    "the same shape reuses them); cold_ms: one step after gsot_cache_clear"}


# ------------------------------------------------------- column-sharded (N > 1)


def shard_block(cfg: int, world: int, rank: int, pg):
    """This rank's column block of config cfg's normalised cost, on the device
    (column-major m x n_p), with the global maximum all-reduced: the same bits
    as the unsharded C / max C (data_io.hpp:162-165)."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2303_07597_b200 as G
    from paper_2303_07597_b200 import sharded as S

    m, n, L, d = G.config_shape(cfg)
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    j0, j1 = S.shard_columns(n, world, rank)
    npc = j1 - j0
    block = torch.empty((npc, m), dtype=torch.float64, device="cuda")
    tb = np.ascontiguousarray(tgt[j0:j1])
    G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(
        src.ctypes.data_as(C.c_void_p), m, tb.ctypes.data_as(C.c_void_p), npc, d, 0,
        C.c_void_p(block.data_ptr())))
    gmax = torch.tensor([block.max().item()], dtype=torch.float64)
    if pg is not None:
        import torch.distributed as dist

        gmax = gmax.cuda() if dist.get_backend() == "nccl" else gmax
        dist.all_reduce(gmax, op=dist.ReduceOp.MAX)
    # true division by a device tensor (a CPU-scalar divisor makes torch multiply by
    # the reciprocal: other bits than cost_matrix's C / max C)
    block.div_(gmax.to(device=block.device))
    torch.cuda.synchronize()
    return block, (m, n, L, sizes, a, b, j0, j1)


def sharded_solves(ctx, kw: dict, steps: int) -> dict:
    ctx.timer_start()
    calls = iters = 0
    for _ in range(steps):
        r = ctx.solve(**kw)
        calls += r["grad_calls"]
        iters += r["iterations"]
    return {"ms": ctx.timer_stop(), "calls": calls, "iters": iters, "x": r["x"],
            "objective": r["objective"]}


def sharded_n1(cfg: int, single_ms: float, single_x, steps: int) -> dict:
    """The column-sharded path at N = 1 on this GPU: the shard context (every
    column, a on rank 0) with an NCCL communicator attached runs the split
    direction update and the per-sequence all-reduces inside its graphs.
    Compared with the single-context solve of the same config (speed, and the
    final state bit for bit)."""
    import numpy as np

    import paper_2303_07597_b200 as G
    from paper_2303_07597_b200 import sharded as S

    gamma, mu, iters = CONFIGS[cfg]
    block, (m, n, L, sizes, a, b, j0, j1) = shard_block(cfg, 1, 0, None)
    ctx = S.shard_context_from_device(block.data_ptr(), m, j1 - j0, sizes, a, b[j0:j1], gamma,
                                      mu, 0)
    del block
    S.attach_comm(ctx, None, "nccl")
    kw = solve_kw(iters)
    ctx.solve(**kw)
    r = sharded_solves(ctx, kw, steps)
    ctx.close()
    G.cache_clear()
    ms = r["ms"] / steps
    return {"solve_ms": ms, "evals_per_s": r["calls"] / (r["ms"] / 1e3),
            "vs_single_context": single_ms / ms,
            "x_bitwise_equal_single_context": bool(np.array_equal(r["x"], single_x)),
            "what": "config %d as ONE column shard (gsot_create_shard_device, a on rank 0) with "
                    "an NCCL communicator attached (world 1): the N>1 code path -- split "
                    "direction update, shard pack / NCCL all-reduce / unpack per sequence -- "
                    "on one GPU, %d timed solves" % (cfg, steps)}


def run_sharded(args, world, rank, local, pg):
    """N > 1: the config's instance column-sharded across the ranks (each
    rank's shard context holds cost[:, J_p]); the library's device-resident
    solve with an NCCL communicator attached (gsot_comm_attach_nccl): per
    device sequence one sum all-reduce of the gradient head (m doubles) and a
    16-double tail, plus the L-BFGS dots of each direction update, all on the
    context stream inside its CUDA graphs. value counts every global
    evaluation once: strong scaling."""
    import numpy as np
    import torch

    import paper_2303_07597_b200 as G
    from paper_2303_07597_b200 import sharded as S

    G.set_device(local)
    cfg = args.config
    gamma, mu, iters = CONFIGS[cfg]
    block, (m, n, L, sizes, a, b, j0, j1) = shard_block(cfg, world, rank, pg)
    npc = j1 - j0
    ctx = S.shard_context_from_device(block.data_ptr(), m, npc, sizes, a, b[j0:j1], gamma, mu,
                                      rank)
    host = torch.empty((npc, m), dtype=torch.float64, pin_memory=True)
    host.copy_(block)  # for the e2e leg
    del block
    torch.cuda.synchronize()
    transport = S.attach_comm(ctx, pg, "nccl")
    kw = solve_kw(iters)
    for _ in range(args.warmup):
        ctx.solve(**kw)
    clocks = ClockSampler(local)
    clocks.start()
    barrier(pg)
    clocks.begin()
    launches0 = ctx.kernel_launches()
    r = sharded_solves(ctx, kw, args.steps)
    launches = ctx.kernel_launches() - launches0
    clocks.end()
    barrier(pg)
    clk = clocks.stop()
    ms = allreduce(pg, r["ms"], "max")
    value = r["calls"] / (ms / 1e3)
    ctx.close()
    # e2e: each rank uploads its pinned host column block through the C ABI,
    # attaches its communicator, solves, downloads its [alpha; beta_p]
    tsteps, ecalls = max(1, args.steps // 4), 0
    barrier(pg)
    t0 = time.perf_counter()
    for _ in range(tsteps):
        c2 = S.shard_context_from_arrays(host.numpy().T, sizes, a, b[j0:j1], gamma, mu, rank)
        S.attach_comm(c2, pg, "nccl")
        ecalls += c2.solve(**kw)["grad_calls"]
        c2.close()
    et = allreduce(pg, time.perf_counter() - t0, "max")
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY.md §8(d) recipe, seed = config id), generated on device",
            "config": {"workload": f"config {cfg}: one fast-mode L-BFGS solve per step, "
                                   f"column-sharded over {world} GPUs ({iters} iterations)",
                       "m": m, "n": n, "L": L, "gamma": gamma, "mu": mu,
                       "l2": "inputs larger than L2, no flush",
                       "parallelism": f"column shards x{world}: device-resident solve per rank, "
                                      f"{transport} all-reduce of m+16 doubles per sequence "
                                      f"and of the L-BFGS dots per direction"},
            "evals_per_solve": r["calls"] / args.steps,
            "iterations_per_solve": r["iters"] / args.steps,
            "gpu_launches": launches,
            "e2e": {"value": ecalls / et, "unit": "evals/s",
                    "h2d_bytes_per_step": 8 * m * n + 8 * (m + n),
                    "d2h_bytes_per_step": 8 * (m + n),
                    "what": "per rank gsot_create_shard from its pinned host column block + "
                            "communicator attach + the sharded solve + x download"},
            "clocks": clk}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--ref-reps", type=int, default=1)
    ap.add_argument("--exact-configs", type=lambda s: [int(c) for c in s.split(",") if c],
                    default=[1, 2, 3, 4, 5])
    ap.add_argument("--skip-large", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded-n1", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "RANK" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    world, rank, local, pg = dist_init()
    try:
        if args.impl == "reference":
            return run_reference(args, world, rank, pg)
        return run_ours(args, world, rank, local, pg)
    finally:
        if pg is not None:
            pg.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
