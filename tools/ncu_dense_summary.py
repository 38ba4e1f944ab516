"""Summarise the dense k_eval captures of tools/ncu_dense.sh into profiles/.

    python tools/ncu_dense_summary.py TAG

Reads gpurun_out/prof_TAG_c{2,4,5}.ncu-rep (--set full, dense / near-dense
evaluations of configs 2, 4, 5) and writes profiles/ncu_dense_TAG.md.
"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size"]
CFG = {"c2": "config 2 (g = 100), baseline mode", "c4": "config 4 (Zipf 9..4000 rows), fast mode, early call",
       "c5": "config 5 (g = 500), fast mode, early call"}


def main():
    tag = sys.argv[1]
    out = [f"# Dense k_eval captures `{tag}` (ncu --set full, one launch each)", "",
           "`bash tools/ncu_dense.sh` on one B200; per-launch, cold L2 between replays.", "",
           "| capture | kernel | " + " | ".join(METRICS) + " | DRAM GB/s |",
           "|---" * (len(METRICS) + 3) + "|"]
    for c, what in CFG.items():
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{c}.ncu-rep")
        if not os.path.exists(rep):
            continue
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                              ",".join(METRICS)], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        h, units = rows[0], rows[1]
        for r in rows[2:3]:
            vals = {m: (r[h.index(m)], units[h.index(m)]) for m in METRICS if m in h}
            t = float(vals["gpu__time_duration.sum"][0].replace(",", ""))
            tu = vals["gpu__time_duration.sum"][1]
            t_s = t * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
                       "msecond": 1e-3}[tu]
            def gb(m):
                v, u = vals[m]
                return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                    "Gbyte": 1e9}[u]
            bw = (gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")) / t_s / 1e9
            name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
            out.append(f"| {what} | {name} | " + " | ".join(f"{v} {u}".strip() for v, u in vals.values())
                       + f" | {bw:.0f} |")
    path = os.path.join(ROOT, "profiles", f"ncu_dense_{tag}.md")
    open(path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
