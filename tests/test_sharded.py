"""CPU, world_size 1, 2 and 3 over gloo: the column-sharded solve
(paper_2303_07597_b200/sharded.py).

The device evaluation is replaced by the oracle (test infrastructure) on each
rank's column shard (a = 0, b_p): what is under test is the sharding, the one
all-reduce per evaluation, and the distributed restatement of the reference's
maximize (lbfgs.hpp:61-274). Against the oracle's unsharded solve_baseline:
the same accepted-iteration and call counts, the iterate within 1e-9 of its
scale, the objective within 1e-10 relative (the sums are re-associated
across shards, so not bitwise)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle_bindings import Oracle, Problem  # noqa: E402

from paper_2303_07597_b200 import sharded as S  # noqa: E402


def instance(seed=5):
    rng = np.random.default_rng(seed)
    sizes = np.array([7, 12, 3, 20], np.int32)
    m, n = int(sizes.sum()), 75
    cost = rng.uniform(0, 2, (m, n))
    a = rng.uniform(0.5, 1.5, m)
    return Problem(cost, sizes, a / a.sum(), np.full(n, 1 / n), 0.4, 0.7)


def oracle_evaluator(o, p, j0, j1):
    q = Problem(p.cost[:, j0:j1], p.sizes, np.zeros(p.m), p.b[j0:j1], p.gamma, p.mu)

    def ev(x, screened):
        al, be = x[: p.m], x[p.m:]
        ga, gb = o.gradient(q, al, be)
        return o.objective(q, al, be), np.concatenate([ga, gb]), (0, 0, q.L * q.n, 0)

    return ev


def test_shard_columns_cover_in_whole_chunks():
    for n in (1, 31, 32, 45, 1000, 50000):
        for world in (1, 2, 3, 8):
            bounds = [S.shard_columns(n, world, r) for r in range(world)]
            assert bounds[0][0] == 0 and bounds[-1][1] == n
            assert all(bounds[r][1] == bounds[r + 1][0] for r in range(world - 1))
            assert all(b0 % 32 == 0 for b0, _ in bounds)


def test_sharded_world1_matches_oracle_baseline():
    o = Oracle()
    p = instance()
    comm = S.Comm(None)
    sp = S.ShardedProblem(None, p.sizes, p.a, p.b, p.gamma, p.mu, comm,
                          evaluator=oracle_evaluator(o, p, 0, p.n))
    r = S.solve_sharded(sp, mode=0, max_outer_loops=4, grad_tol=1e-12)
    ro = o.solve(p, mode=0, max_outer_loops=4, grad_tol=1e-12)
    assert r.iterations == ro["iterations"] and r.stats.grad_calls == ro["grad_calls"]
    assert np.max(np.abs(r.x - ro["x"])) <= 1e-9 * np.max(np.abs(ro["x"]))
    assert abs(r.objective - ro["objective"]) <= 1e-10 * abs(ro["objective"])


WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch.distributed as dist
dist.init_process_group("gloo")
from test_sharded import instance, oracle_evaluator
from oracle_bindings import Oracle
from paper_2303_07597_b200 import sharded as S
o = Oracle(); p = instance()
rank, world = dist.get_rank(), dist.get_world_size()
j0, j1 = S.shard_columns(p.n, world, rank)
sp = S.ShardedProblem(None, p.sizes, p.a, p.b[j0:j1], p.gamma, p.mu, S.Comm(dist.group.WORLD),
                      evaluator=oracle_evaluator(o, p, j0, j1))
r = S.solve_sharded(sp, mode=0, max_outer_loops=4, grad_tol=1e-12)
print(json.dumps({"rank": rank, "j0": j0, "j1": j1, "iters": r.iterations,
                  "calls": r.stats.grad_calls, "unskipped": r.stats.blocks_unskipped,
                  "obj": r.objective, "x": r.x.tolist()}))
dist.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gloo_matches_oracle_baseline(world):
    port = free_port()
    procs = []
    for rank in range(world):
        env = dict(os.environ, ROOT=ROOT, RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for pr in procs:
        out, err = pr.communicate(timeout=240)
        assert pr.returncode == 0, err
        outs.append(json.loads(out.strip().splitlines()[-1]))
    o = Oracle()
    p = instance()
    ro = o.solve(p, mode=0, max_outer_loops=4, grad_tol=1e-12)
    rs = sorted(outs, key=lambda d: d["rank"])
    assert rs[0]["j0"] == 0 and rs[-1]["j1"] == p.n
    assert all(rs[i]["j1"] == rs[i + 1]["j0"] for i in range(world - 1))
    # every rank takes the same decisions: counts, objective, replicated alpha
    for r in rs:
        assert (r["iters"], r["calls"]) == (ro["iterations"], ro["grad_calls"])
        assert r["unskipped"] == ro["grad_calls"] * p.L * p.n  # counters summed over ranks
        assert r["obj"] == rs[0]["obj"]
        assert np.array_equal(np.array(r["x"])[: p.m], np.array(rs[0]["x"])[: p.m])
    x = np.concatenate([np.array(rs[0]["x"])[: p.m]] + [np.array(r["x"])[p.m:] for r in rs])
    assert np.max(np.abs(x - ro["x"])) <= 1e-9 * np.max(np.abs(ro["x"]))
    assert abs(rs[0]["obj"] - ro["objective"]) <= 1e-10 * abs(ro["objective"])
