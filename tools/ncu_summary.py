"""Summarise ncu captures from gpurun_out/ into profiles/ (committed evidence).

    python tools/ncu_summary.py TAG [--cmd "..."] [--full PROF_TAG ...] [--traffic-cfg C]

Reads gpurun_out/launches_TAG.csv (gpu__time_duration + dram bytes per launch,
cold-cache, serialised) and gpurun_out/prof_<PROF_TAG>.ncu-rep (--set full
captures), writes profiles/ncu_TAG.md and, with --traffic-cfg C,
profiles/ncu_traffic_cfgC.json (per-kernel DRAM bytes per launch of the full
captures, read by bench.py's roofline.traffic).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name: str) -> str:
    # template arguments dropped (k_eval<0> and k_eval<1> are both "k_eval")
    return name.split("(")[0].split("<")[0].replace("gsot::", "").replace("void ", "").strip()


def launches(tag: str):
    path = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    idi = h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        per[r[idi]][r[mi]] = v
        names[r[idi]] = short(r[ki])
    agg = collections.defaultdict(lambda: {"n": 0, "us": 0.0, "read": 0.0, "write": 0.0})
    for lid, ms in per.items():
        a = agg[names[lid]]
        a["n"] += 1
        a["us"] += ms.get("gpu__time_duration.sum", 0.0)
        a["read"] += ms.get("dram__bytes_read.sum", 0.0)
        a["write"] += ms.get("dram__bytes_write.sum", 0.0)
    return agg


def full(tag: str):
    path = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    if not os.path.exists(path):
        return []
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "l1tex__t_sector_hit_rate.pct", "launch__grid_size",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for w in want:
            if w in h:
                i = h.index(w)
                d[w] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--cmd", default="python bench.py --steps 1 --warmup 1 --no-cpu-baseline")
    ap.add_argument("--full", nargs="*", default=None)
    ap.add_argument("--traffic-cfg", type=int, default=None)
    args = ap.parse_args()
    tag = args.tag
    agg = launches(tag)
    tot = sum(a["us"] for a in agg.values())
    lines = [f"# ncu summary `{tag}`", "",
             f"Command: `{args.cmd}` (per-launch times are cold-cache and serialised under ncu: "
             "compare shares, not absolutes).", "",
             "| kernel | launches | total us | mean us | share | DRAM read MB/launch | DRAM write MB/launch |",
             "|---|---|---|---|---|---|---|"]
    traffic = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        n = a["n"]
        lines.append(f"| {k} | {n} | {a['us']:.1f} | {a['us'] / n:.2f} | {a['us'] / tot:.3f} | "
                     f"{a['read'] / n / 1e6:.3f} | {a['write'] / n / 1e6:.3f} |")
        traffic[k] = {"dram_bytes_per_launch": (a["read"] + a["write"]) / n, "launches": n,
                      "mean_us": a["us"] / n, "source": f"profiles/ncu_{tag}.md"}
    fl = []
    for ft in (args.full if args.full is not None else [tag]):
        fl += [dict(d, capture=ft) for d in full(ft)]
    if fl:
        lines += ["", "## `--set full` captures", "",
                  "| kernel | " + " | ".join(k for k in fl[0] if k != "kernel") + " |",
                  "|---" * len(fl[0]) + "|"]
        for d in fl:
            lines.append(f"| {d['kernel']} | " + " | ".join(v for k, v in d.items()
                                                          if k != "kernel") + " |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if args.traffic_cfg is not None:
        with open(os.path.join(ROOT, "profiles", f"ncu_traffic_cfg{args.traffic_cfg}.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
