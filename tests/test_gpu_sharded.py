"""GPU: the column-sharded solve (paper_2303_07597_b200/sharded.py) through
gsot_create_shard contexts, against the single-context device solve and the
oracle. Two ranks share the one GPU of the test box over gloo: a functional
check of the sharding (each rank's kernels are independent; the all-reduce is
a host collective), not a multi-GPU performance claim."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2303_07597_b200 as G
from oracle_bindings import Oracle, Problem
from paper_2303_07597_b200 import sharded as S

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def instance():
    rng = np.random.default_rng(11)
    sizes = np.array([40, 9, 130, 25, 60], np.int32)
    m, n = int(sizes.sum()), 150
    cost = rng.uniform(0, 2, (m, n))
    a = rng.uniform(0.5, 1.5, m)
    return Problem(cost, sizes, a / a.sum(), np.full(n, 1 / n), 0.3, 0.6)


KW = dict(mode=1, snapshot_interval=10, grad_tol=1e-12, max_outer_loops=3)


def test_shard_context_terms():
    """With a = 0 a shard's gradient head is minus its plan row sums and its
    objective b_p.beta_p - psi_p: the shards' terms add up to the full eval."""
    o = Oracle()
    p = instance()
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.uniform(0, 0.02, p.m), rng.uniform(0, 1.2, p.n)])
    obj_o = o.objective(p, x[: p.m], x[p.m:])
    ga_o, gb_o = o.gradient(p, x[: p.m], x[p.m:])
    ga, obj, gb = p.a.copy(), float(np.dot(p.a, x[: p.m])), []
    for r in range(3):
        j0, j1 = S.shard_columns(p.n, 3, r)
        ctx = G.Context.shard_from_arrays(p.cost[:, j0:j1], p.sizes, np.zeros(p.m), p.b[j0:j1],
                                          p.gamma, p.mu)
        ob, g, _ = ctx.eval(np.concatenate([x[: p.m], x[p.m + j0: p.m + j1]]))
        ctx.close()
        ga += g[: p.m]
        obj += ob
        gb.append(g[p.m:])
    assert abs(obj - obj_o) <= 1e-12 * abs(obj_o)
    assert np.max(np.abs(ga - ga_o)) <= 1e-12 and np.max(np.abs(np.concatenate(gb) - gb_o)) <= 1e-12
    # shard marginals are not required to sum to one; entries are still checked
    with pytest.raises(G.MarginalNotNormalized):
        G.Context.shard_from_arrays(p.cost[:, :32], p.sizes, np.zeros(p.m), -p.b[:32], 1.0, 1.0)


def test_sharded_world1_matches_device_solve():
    p = instance()
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    rd = ctx.solve(**KW)
    ctx.close()
    sp = S.ShardedProblem(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu, S.Comm(None))
    r = S.solve_sharded(sp, mode=1, max_outer_loops=3, grad_tol=1e-12)
    sp.close()
    assert r.iterations == rd["iterations"] and r.stats.grad_calls == rd["grad_calls"]
    assert (r.stats.blocks_in_active_set, r.stats.blocks_skipped, r.stats.blocks_unskipped) == \
        (rd["blocks_in_active_set"], rd["blocks_skipped"], rd["blocks_unskipped"])
    assert np.max(np.abs(r.x - rd["x"])) <= 1e-9 * np.max(np.abs(rd["x"]))
    assert abs(r.objective - rd["objective"]) <= 1e-10 * abs(rd["objective"])


WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch.distributed as dist
dist.init_process_group("gloo")
from test_gpu_sharded import instance
from paper_2303_07597_b200 import sharded as S
p = instance()
rank, world = dist.get_rank(), dist.get_world_size()
j0, j1 = S.shard_columns(p.n, world, rank)
sp = S.ShardedProblem(p.cost[:, j0:j1], p.sizes, p.a, p.b[j0:j1], p.gamma, p.mu, S.Comm(dist.group.WORLD))
r = S.solve_sharded(sp, mode=1, max_outer_loops=3, grad_tol=1e-12)
sp.close()
st = r.stats
print(json.dumps({"rank": rank, "j0": j0, "j1": j1, "iters": r.iterations, "calls": st.grad_calls,
                  "cnt": [st.blocks_in_active_set, st.blocks_skipped, st.blocks_unskipped],
                  "obj": r.objective, "x": r.x.tolist()}))
dist.destroy_process_group()
"""


@pytest.mark.timeout(600)
def test_sharded_world2_on_one_gpu_matches_device_solve():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for rank in range(2):
        env = dict(os.environ, ROOT=ROOT, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for pr in procs:
        out, err = pr.communicate(timeout=500)
        assert pr.returncode == 0, err
        outs.append(json.loads(out.strip().splitlines()[-1]))
    p = instance()
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    rd = ctx.solve(**KW)
    ctx.close()
    r0, r1 = sorted(outs, key=lambda d: d["rank"])
    assert r0["iters"] == r1["iters"] == rd["iterations"]
    assert r0["calls"] == r1["calls"] == rd["grad_calls"]
    assert r0["cnt"] == [rd["blocks_in_active_set"], rd["blocks_skipped"], rd["blocks_unskipped"]]
    assert r0["obj"] == r1["obj"]
    x0, x1 = np.array(r0["x"]), np.array(r1["x"])
    assert np.array_equal(x0[: p.m], x1[: p.m])
    x = np.concatenate([x0, x1[p.m:]])
    assert np.max(np.abs(x - rd["x"])) <= 1e-9 * np.max(np.abs(rd["x"]))
    assert abs(r0["obj"] - rd["objective"]) <= 1e-10 * abs(rd["objective"])


# ---- the device-resident sharded solve (gsot_comm_*) ----------

def _single(p, **kw):
    ctx = G.Context.from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu)
    r = ctx.solve(**kw)
    ctx.close()
    return r


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_device_sharded_world1_nccl_bitwise(mode):
    """One rank over NCCL: the shard context (all columns, a on rank 0) with its
    communicator attached runs the same graphs plus the split direction update
    and the all-reduces, and reproduces the single-context solve bit for bit."""
    p = instance()
    kw = dict(KW, mode=mode, history_cap=4096)
    rd = _single(p, **kw)
    ctx = S.shard_context_from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu, rank=0)
    assert S.attach_comm(ctx, None, "nccl") == "nccl"
    r = ctx.solve(**kw)
    r2 = ctx.solve(**kw)  # replayed graphs
    ctx.close()
    for rr in (r, r2):
        for f in ("iterations", "grad_calls", "blocks_in_active_set", "blocks_skipped",
                  "blocks_unskipped", "upper_bounds_evaluated", "converged"):
            assert rr[f] == rd[f], f
        assert rr["objective"] == rd["objective"]
        assert np.array_equal(rr["x"], rd["x"])
        assert np.array_equal(rr["history"], rd["history"])


def test_device_sharded_rejects_exact_and_audit():
    p = instance()
    ctx = S.shard_context_from_arrays(p.cost, p.sizes, p.a, p.b, p.gamma, p.mu, rank=0)
    S.attach_comm(ctx, None, "nccl")
    with pytest.raises(G.Error):
        ctx.solve(**dict(KW, exact=True))
    with pytest.raises(G.Error):
        ctx.solve(**dict(KW, mode=3))
    ctx.detach_comm()
    ctx.solve(**KW)  # alone again
    ctx.close()


DEVICE_WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch.distributed as dist
dist.init_process_group("gloo")
from test_gpu_sharded import instance, KW
from paper_2303_07597_b200 import sharded as S
p = instance()
rank, world = dist.get_rank(), dist.get_world_size()
mode = int(os.environ["MODE"])
j0, j1 = S.shard_columns(p.n, world, rank)
ctx = S.shard_context_from_arrays(p.cost[:, j0:j1], p.sizes, p.a, p.b[j0:j1], p.gamma, p.mu, rank)
assert S.attach_comm(ctx, dist.group.WORLD, "host") == "host"
r = ctx.solve(**dict(KW, mode=mode, history_cap=4096))
ctx.close()
print(json.dumps({"rank": rank, "j0": j0, "j1": j1, "iters": r["iterations"],
                  "calls": r["grad_calls"], "hist": r["history"].tolist(),
                  "cnt": [r["blocks_in_active_set"], r["blocks_skipped"], r["blocks_unskipped"],
                          r["upper_bounds_evaluated"]],
                  "obj": r["objective"], "x": r["x"].tolist()}))
dist.destroy_process_group()
"""


def _run_ranks(world, env_extra):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for rank in range(world):
        env = dict(os.environ, ROOT=ROOT, RANK=str(rank), WORLD_SIZE=str(world),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **env_extra)
        procs.append(subprocess.Popen([sys.executable, "-c", DEVICE_WORKER], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for pr in procs:
        out, err = pr.communicate(timeout=500)
        assert pr.returncode == 0, err
        outs.append(json.loads(out.strip().splitlines()[-1]))
    return sorted(outs, key=lambda d: d["rank"])


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,mode", [(2, 1), (3, 1), (2, 0)])
def test_device_sharded_host_transport_matches_single_context(world, mode):
    """world ranks share the test box's one GPU, summing through gloo (the host
    transport: each rank's kernels are independent, the host does the exchange).
    Every rank takes the same decisions; the assembled state matches the
    single-context device solve; counters are the global GradStats."""
    outs = _run_ranks(world, {"MODE": str(mode)})
    p = instance()
    rd = _single(p, **dict(KW, mode=mode, history_cap=4096))
    m = p.m
    for o in outs:
        assert o["iters"] == rd["iterations"] and o["calls"] == rd["grad_calls"]
        assert o["obj"] == outs[0]["obj"] and o["hist"] == outs[0]["hist"]
        assert o["cnt"] == [rd["blocks_in_active_set"], rd["blocks_skipped"],
                            rd["blocks_unskipped"], rd["upper_bounds_evaluated"]]
        assert np.array_equal(np.array(o["x"][:m]), np.array(outs[0]["x"][:m]))
    assert outs[0]["hist"] == rd["history"].tolist()
    x = np.concatenate([np.array(outs[0]["x"][:m])] + [np.array(o["x"][m:]) for o in outs])
    assert np.max(np.abs(x - rd["x"])) <= 1e-9 * np.max(np.abs(rd["x"]))
    assert abs(outs[0]["obj"] - rd["objective"]) <= 1e-10 * abs(rd["objective"])
