"""Per-kernel duration stats from a gpurun_out/launches_TAG.csv launch list.

    python tools/launch_stats.py TAG [KERNEL]
"""
import collections
import csv
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rows = list(csv.reader(open(os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv"))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] in ("nsecond", "ns") else v * 1000 if r[ui] in ("msecond", "ms") else v
    per[r[ki].split("(")[0]].append(v)
tot = sum(sum(v) for v in per.values())
print(f"total {tot:.0f} us")
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:22s} n={len(v):4d} mean={sum(v) / len(v):8.2f} median={statistics.median(v):8.2f} tot={sum(v):8.0f}")
if len(sys.argv) > 2:
    v = per[sys.argv[2]]
    print("first 12:", [round(x, 1) for x in v[:12]])
    print("every 20th:", [round(x, 1) for x in v[::20]])
