"""Diagnostic: how many blocks a TIGHTER valid upper bound on z would skip.

The paper's bound (screening.hpp:63-86) is z <= z~ + |[dalpha_l]+| + sqrt(g_l) [dbeta_j]+.
Since [a + b]+ <= [a]+ + [b]+ elementwise, z <= z~ + phi_l(dbeta_j) with
phi_l(d) = |[dalpha_l + d]+|_2 also holds, and it is tighter when dbeta_j < 0
(a falling beta_j cancels rising alphas). Any proof of z <= tau lets the
evaluation skip a block with bitwise-identical results (its plan entries, psi
and sums are exact zeros), after the reference's own decisions are counted.

At refresh states of a fast config solve and five iterations later: the
fraction of blocks (and of 8-column quarters, what the evaluation fetches)
left to compute under each test.

    python tools/tight_bound_study.py [--config 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CONFIGS = {2: (0.1, 0.5, 200), 3: (0.1, 0.2, 200), 4: (0.05, 0.3, 200), 5: (0.1, 0.5, 300)}


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
    import ctypes as C
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    dev = torch.empty((n, m), dtype=torch.float64, device="cuda")  # cost, column-major
    G.groupot._raise(G._lib.lib().gsot_cost_matrix_device(
        src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 1,
        C.c_void_p(dev.data_ptr())))
    sizes = np.asarray(sizes)
    off = np.concatenate([[0], np.cumsum(sizes)])
    cmin = torch.empty((L, n), dtype=torch.float64, device="cuda")
    for l in range(L):
        cmin[l] = dev[:, off[l]:off[l + 1]].min(dim=1).values
    del dev
    torch.cuda.empty_cache()
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    g = torch.tensor(sizes, dtype=torch.float64, device="cuda")
    nw = (n + 31) // 32
    pad = nw * 32 - n

    def state(outer, interval):
        return ctx.solve(mode=1, max_outer_loops=outer, snapshot_interval=interval,
                         grad_tol=1e-12)["x"]

    def quarters(keep):  # keep: (L, n) bool -> fraction of blocks, of quarters with a kept block
        q = torch.nn.functional.pad(keep, (0, pad)).view(L, nw, 4, 8).any(dim=3)
        gb = g[:, None, None]
        return {"blocks": float(keep.double().mean()),
                "quarter_GB": float((q.double() * gb * 64).sum()) / 1e9}

    out = []
    for k in (2, 5, 10, iters // 20, iters // 10 - 1):
        xs = state(k, 10)            # a refresh point: the snapshot state
        x = state(2 * k + 1, 5)      # five iterations later on the same trajectory
        ctx.init_snapshot(xs)
        zt = torch.from_numpy(ctx.snapshot_norms()[0]).cuda()      # exact z~ (L, n)
        da = torch.from_numpy(x[:m] - xs[:m]).cuda()
        db = torch.from_numpy(x[m:] - xs[m:]).cuda()
        dpos = torch.stack([da[off[l]:off[l + 1]].clamp(min=0).norm() for l in range(L)])
        paper = zt + dpos[:, None] + torch.sqrt(g)[:, None] * db.clamp(min=0)[None, :]
        tight = torch.empty_like(paper)
        for l in range(L):
            tight[l] = zt[l] + (da[None, off[l]:off[l + 1]] + db[:, None]).clamp(min=0).norm(dim=1)
        needed = torch.from_numpy(ctx.block_mask(x)).cuda()
        xa = torch.from_numpy(x[:m]).cuda()
        xb = torch.from_numpy(x[m:]).cuda()
        amax = torch.stack([xa[off[l]:off[l + 1]].max() for l in range(L)])
        pz = (amax[:, None] + xb[None, :]) > cmin  # not provably zero
        keep_paper = (paper > tau) & pz
        keep_tight = (tight > tau) & pz
        assert not bool((needed & ~keep_tight).any()), "the tight bound skipped a nonzero block"
        row = {"snapshot_outer_loops": k, "zero_test_only": quarters(pz),
               "paper": quarters(keep_paper),
               "tight": quarters(keep_tight), "needed": quarters(needed),
               "dbeta_negative_frac": float((db < 0).double().mean())}
        out.append(row)
        print(json.dumps(row), flush=True)
    ctx.close()
    print(json.dumps({"config": cfg, "states": out}))


if __name__ == "__main__":
    main()
