"""(f)1 study: generating the cost from the features on the device (the
reference's k-sequential, FMA-free definition, data_io.hpp:101-123) against
streaming the stored 8 m n bytes, on one config.

    python tools/cost_gen_vs_stream.py [--config 5]

Times gsot_cost_matrix_device (every c_ij = sum_k (x_ik - y_jk)^2 in fp64,
bitwise the reference) and one dense fused evaluation of the stored cost,
with CUDA events on the current stream; prints one JSON line."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {1: (1.0, 0.1), 2: (0.1, 0.5), 3: (0.1, 0.2), 4: (0.05, 0.3), 5: (0.1, 0.5)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2303_07597_b200 as G

    cfg = args.config
    m, n, L, d = G.config_shape(cfg)
    src, tgt, sizes, a, b = G.config_features(cfg, cfg)
    # cost generation (column-major m x n output in HBM)
    dev = torch.empty((n, m), dtype=torch.float64, device="cuda")
    lib = G._lib.lib()

    def gen():
        G.groupot._raise(lib.gsot_cost_matrix_device(
            src.ctypes.data_as(C.c_void_p), m, tgt.ctypes.data_as(C.c_void_p), n, d, 0,
            C.c_void_p(dev.data_ptr())))

    gen()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        gen()
    e1.record()
    torch.cuda.synchronize()
    gen_ms = e0.elapsed_time(e1) / args.reps
    del dev
    torch.cuda.empty_cache()
    # one dense fused evaluation of the stored cost
    gamma, mu = CONFIGS[cfg]
    ctx = G.Context.from_config(cfg, cfg, gamma, mu)
    x = np.zeros(m + n)
    r = ctx.solve(mode=1, max_outer_loops=2, grad_tol=1e-12)
    x = r["x"]
    ctx.eval(x)
    ctx.timer_start()
    for _ in range(args.reps):
        ctx.eval(x)
    eval_ms = ctx.timer_stop() / args.reps
    ctx.close()
    flops = 3.0 * m * n * d  # one sub, one mul, one add per (i, j, k): no FMA (parity)
    print(json.dumps({
        "config": cfg, "m": m, "n": n, "d": d,
        "cost_generation_ms": gen_ms,
        "cost_generation_tflops": flops / (gen_ms * 1e-3) / 1e12,
        "dense_eval_of_stored_cost_ms": eval_ms,
        "stored_cost_bytes": 8 * m * n,
        "ratio_generation_over_stream": gen_ms / eval_ms,
        "note": "generation is a lower bound for a fused variant (the eval's own work comes on top)"}))


if __name__ == "__main__":
    main()
