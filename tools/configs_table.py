"""Render profiles/configs_r1.md from a tools/solve_configs.py JSON.

    python tools/configs_table.py gpurun_out/configs.json profiles/configs_r1
"""
import json
import shutil
import sys

src, dst = sys.argv[1], sys.argv[2]
d = json.load(open(src))
shutil.copy(src, dst + ".json")
L = ["# L-BFGS solve times, all five configs", "",
     "Command: `python tools/solve_configs.py --e2e --reps 2` on one B200 (gpurun). Synthetic",
     "instances per SURVEY.md §8(d) (seed = config id), cost generated on device; snapshot",
     "interval 10, memory 10, grad_tol 1e-12 (runs to the iteration budget). `solve ms` is the",
     "maximize span (the reference's `Solution::wall_time`), best of 2; `e2e` is",
     "`gsot_create` from a pinned host cost matrix (H2D + validation + re-layout) + the solve +",
     "`gsot_destroy`, best of 2 (the second create reuses the parked device state).", "",
     "| cfg | m x n, L | budget | fast solve ms | evals | evals/s | blocks computed | baseline solve ms | baseline evals/s | fast / baseline | e2e ms (create ms) |",
     "|---|---|---|---|---|---|---|---|---|---|---|"]
for r in d:
    f, b, e = r["fast"], r["baseline"], r.get("e2e_fast", {})
    L.append(f"| {r['config']} | {r['m']} x {r['n']}, {r['L']} | {r['iteration_budget']} | "
             f"{f['solve_ms']:.1f} | {f['grad_calls']} | {f['evals_per_s']:.0f} | "
             f"{100 * f['blocks_computed_frac']:.1f} % | {b['solve_ms']:.1f} | {b['evals_per_s']:.0f} | "
             f"{r['fast_vs_baseline_speedup']:.2f}x | {e.get('total_ms', 0):.0f} ({e.get('create_ms', 0):.0f}) |")
L += ["", "`baseline` = every block on every call (the reference's solve_baseline on the GPU);",
      "`fast` = upper-bound skipping + lower-bound active set (solve_fast). Dense HBM bytes per",
      "baseline evaluation are 8·m·n: cfg2 0.8 GB, cfg3 8 GB, cfg4 9.6 GB, cfg5 40 GB."]
open(dst + ".md", "w").write("\n".join(L) + "\n")
print("\n".join(L))
