"""Column-sharded solve of a BASELINE config across the GPUs of one node.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/sharded_solve.py --config 5
    python tools/sharded_solve.py --config 5            # N = 1

Every rank builds the config's features (SURVEY.md §8(d) recipe, seed = config
id), computes the cost of its column block J_p on its own GPU
(gsot_cost_matrix_device), divides by the global max (all-reduce max: the same
bits as the unsharded C / max C, data_io.hpp:162-165), creates its shard
context on the device (gsot_create_shard_device) and runs the sharded fast
solve (paper_2303_07597_b200/sharded.py). Rank 0 prints one JSON line; the
solve time is the max over ranks.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
           5: (0.1, 0.5, 300)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--outer-loops", type=int, default=0)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2303_07597_b200 as G
    from paper_2303_07597_b200 import sharded as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    G.set_device(local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl")
        pg = dist.group.WORLD
    comm = S.Comm(pg)
    cfg = args.config
    gamma, mu, iters = CONFIGS[cfg]
    m, n, L, d = G.config_shape(cfg)
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    j0, j1 = S.shard_columns(n, world, rank)
    npc = j1 - j0
    block = torch.empty((npc, m), dtype=torch.float64, device="cuda")  # column-major m x npc
    tb = np.ascontiguousarray(tgt[j0:j1])
    G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(
        src.ctypes.data_as(C.c_void_p), m, tb.ctypes.data_as(C.c_void_p), npc, d, 0,
        C.c_void_p(block.data_ptr())))
    gmax = comm.allreduce(np.array([block.max().item()]), "max")[0]
    block /= gmax
    torch.cuda.synchronize()
    ctx = G.Context.shard_from_device(block.data_ptr(), m, npc, sizes, np.zeros(m), b[j0:j1],
                                      gamma, mu)
    del block
    sp = S.ShardedProblem(None, sizes, a, b[j0:j1], gamma, mu, comm, ctx=ctx)
    outer = args.outer_loops or iters // 10
    if pg is not None:
        dist.barrier()
    r = S.solve_sharded(sp, mode=1, max_outer_loops=outer, grad_tol=1e-12)
    wall = comm.allreduce(np.array([r.wall_seconds]), "max")[0]
    sp.close()
    if rank == 0:
        st = r.stats
        print(json.dumps({"config": cfg, "world": world, "m": m, "n": n, "columns_rank0": npc,
                          "solve_s": wall, "evals": st.grad_calls,
                          "evals_per_s": st.grad_calls / wall, "iterations": r.iterations,
                          "objective": r.objective,
                          "blocks": [st.blocks_in_active_set, st.blocks_skipped,
                                     st.blocks_unskipped]}), flush=True)
    if pg is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
