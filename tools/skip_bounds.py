"""Diagnostic: how much of the cost a (group, 32-column) task must read under
read-free block tests, at the states of a fast-mode solve (dense estimate: every
task, before the screen).

  zero      max_{i in l} alpha_i + beta_j <= min_{i in l} c_ij    (z = 0: k_eval today)
  subthr    g_l * M^2 <= tau^2 (1 - 1e-9), M = amax_l + beta_j - cmin_lj
            (z <= sqrt(g_l) M <= tau: the block's plan, psi and gradient terms are 0)
  needed    z > tau (the block is nonzero: gsot_block_mask)

For each test: the fraction of tasks with a column that fails it (whole-tile
reads), of 8-column quarters (sector-granular reads), and the bytes.

    python tools/skip_bounds.py [--config 5]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = {1: (1.0, 0.1, 100), 2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200),
           5: (0.1, 0.5, 300)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2303_07597_b200 as G

    cfg = args.config
    gamma, mu, iters = CONFIGS[cfg]
    tau = gamma * mu
    m, n, L, d = G.config_shape(cfg)
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
    G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(
        src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 1,
        C.c_void_p(dev.data_ptr())))
    off = np.concatenate([[0], np.cumsum(sizes)])
    cmin = torch.empty((L, n), dtype=torch.float64, device="cuda")
    for l in range(L):
        cmin[l] = dev[:, off[l]:off[l + 1]].min(dim=1).values
    torch.cuda.empty_cache()
    g = torch.tensor(sizes, dtype=torch.float64, device="cuda")
    nw = (n + 31) // 32
    pad = nw * 32 - n
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    out = []

    def frac(fail):  # fail: (L, n) bool -> task / quarter fractions, bytes
        f = torch.nn.functional.pad(fail, (0, pad)).view(L, nw, 4, 8)
        q = f.any(dim=3)  # (L, nw, 4)
        t = q.any(dim=2)  # (L, nw)
        gb = g[:, None]
        tile_bytes = float((t.double() * gb * 256).sum())
        quarter_bytes = float((q.double().sum(dim=2) * gb * 64).sum())
        return {"tasks": float(t.double().mean()), "quarters": float(q.double().mean()),
                "tile_GB": tile_bytes / 1e9, "quarter_GB": quarter_bytes / 1e9}

    def hmax(xa):  # H[l, j] = max_{i in l} (alpha_i - c_ij)
        H = torch.empty((L, n), dtype=torch.float64, device="cuda")
        for l in range(L):
            H[l] = (xa[None, off[l]:off[l + 1]] - dev[:, off[l]:off[l + 1]]).max(dim=1).values
        return H

    def state(outer, interval):
        x = ctx.solve(mode=1, max_outer_loops=outer, snapshot_interval=interval,
                      grad_tol=1e-12)["x"]
        return torch.from_numpy(x[:m]).cuda(), torch.from_numpy(x[m:]).cuda(), x

    for k in (1, 2, 5, 10, iters // 20, iters // 10 - 1):
        sa, sb, _ = state(k, 10)  # the snapshot state (a refresh point)
        xa, xb, x = state(2 * k + 1, 5)  # five iterations later (same trajectory)
        amax = torch.stack([xa[off[l]:off[l + 1]].max() for l in range(L)])
        samax = torch.stack([sa[off[l]:off[l + 1]].max() for l in range(L)])
        dmax = torch.stack([(xa - sa)[off[l]:off[l + 1]].max() for l in range(L)])
        M = (amax[:, None] + xb[None, :]) - cmin
        zero_fail = M > 0
        sub_fail = (g[:, None] * M * M > tau * tau * (1 - 1e-9)) & zero_fail
        Hs = hmax(sa)
        snap_fail = ((Hs + dmax[:, None] + xb[None, :]) > 0) & zero_fail
        # the snapshot is lazy: exact H only where it reads (the zero test fails at the snapshot)
        lazy_read = (samax[:, None] + sb[None, :]) - cmin > 0
        Hl = torch.where(lazy_read, Hs, samax[:, None] - cmin)
        snapl_fail = ((Hl + dmax[:, None] + xb[None, :]) > 0) & zero_fail
        pos = (hmax(xa) + xb[None, :]) > 0  # z > 0: the best any z = 0 test can do
        needed = torch.from_numpy(ctx.block_mask(x)).cuda()
        out.append({"snapshot_outer_loops": k, "iterations": 10 * k + 5,
                    "dense_GB": 8.0 * m * nw * 32 / 1e9,
                    "zero": frac(zero_fail), "subthr": frac(sub_fail), "snapH": frac(snap_fail),
                    "snapH_lazy": frac(snapl_fail), "z_pos": frac(pos), "needed": frac(needed)})
        print(json.dumps(out[-1]), flush=True)
    ctx.close()
    print(json.dumps({"config": cfg, "states": out}))


if __name__ == "__main__":
    main()
