"""CPU, world_size 2 over gloo: the N > 1 path of bench.py.

The solve does not shard for the BASELINE configs that fit one GPU
(configs 1-2 are replicas), so `bench.py --gpus N` runs one
independent replica per rank with no data-path collective. What crosses
ranks is the measurement: a barrier around the timed region, the MAX of the
per-rank device times and the SUM of the per-rank evaluation counts. These
tests run that exact code (bench.dist_init / allreduce / barrier) in two gloo
processes, and check that the reference arm's non-zero ranks exit without
work."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import bench
world, rank, local, pg = bench.dist_init()
assert pg is not None and pg.get_backend() == "gloo" and world == 2
# per-rank "device time" and evaluation counts of a replica run
ms = [30.0, 45.0][rank]
calls = [270, 268][rank]
bench.barrier(pg)
ms_max = bench.allreduce(pg, ms, "max")
calls_tot = bench.allreduce(pg, float(calls), "sum")
value = calls_tot / (ms_max / 1e3)
class A: pass
a = A(); a.config = 2; a.steps = 1; a.warmup = 0; a.ref_iters = 1; a.ref_replicas = 1
ref_rc = bench.run_reference(a, world, rank, pg) if rank == 1 else 0
print(json.dumps({"rank": rank, "ms_max": ms_max, "calls": calls_tot, "value": value,
                  "ref_rc": ref_rc}))
pg.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_replica_measurement_over_gloo():
    import json

    port = free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, ROOT=ROOT, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=240)
        assert p.returncode == 0, e
        outs.append(json.loads(o.strip().splitlines()[-1]))
    for o in outs:
        assert o["ms_max"] == 45.0  # time = max over ranks
        assert o["calls"] == 538.0  # work = sum over ranks
        assert abs(o["value"] - 538.0 / 0.045) < 1e-6
        assert o["ref_rc"] == 0  # reference arm: rank != 0 exits 0 without work
