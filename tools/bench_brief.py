"""Prints the main figures of a bench.py JSON line (log file argument)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        r = d["roofline"]
        print(path, "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 2), "frac",
              round(r["frac"], 3), "e2e", round(d["e2e"]["value"], 1), d["clocks"]["sm_mhz"],
              d["clocks"]["reasons"], "launches", d.get("gpu_launches"))
        print("  k_eval: bytes/launch", round(r["bytes_per_launch"] / 1e6, 1), "MB, ms/launch",
              round(r["ms_per_launch"], 4), "share", round(r["share_of_step"], 3), "fetched",
              r.get("fetched"))
        for k, v in (r.get("regimes") or {}).items():
            print("  ", k, {a: (round(b, 3) if isinstance(b, float) else b) for a, b in v.items()})
        print("  configs", {k: (round(v["solve_ms"], 2), round(v["exact"]["solve_ms"], 1))
                            for k, v in d["configs"].items()})
        print("  kernels", {k: (round(v["ms"], 1), v["launches"]) for k, v in d["kernels"].items()})
        if d.get("sharded_n1"):
            print("  sharded_n1", d["sharded_n1"]["solve_ms"], d["sharded_n1"]["vs_single_context"])
