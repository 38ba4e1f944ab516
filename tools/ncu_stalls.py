"""Top warp-stall SASS lines of one kernel in an ncu report.

    python tools/ncu_stalls.py REPORT.ncu-rep KERNEL_REGEX [N] [LAUNCH_SKIP]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", sys.argv[4] if len(sys.argv) > 4 else "0", "--launch-count", "1", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))[1:]
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
body = [r for r in rows[1:] if len(r) > si and r[si].replace(".", "").isdigit()]
tot = sum(float(r[si] or 0) for r in body) or 1.0
idx = {id(r): i for i, r in enumerate(body)}
for r in sorted(body, key=lambda r: -float(r[si] or 0))[:n]:
    print(f"{idx[id(r)]:5d} {float(r[si]) / tot:6.3f} ex={r[ex]:>8s}  {r[1].strip()[:70]}")
