"""Summaries of one round's ncu evidence for profiles/ (run here, on the files gpurun brought
back):

python tools/ncu_summaries.py <tag>     reads gpurun_out/<tag>_ncu_launches.csv and
                                        gpurun_out/<tag>_full.ncu-rep, writes
                                        profiles/<tag>_ncu_launches{.csv,_summary.txt},
                                        profiles/<tag>_ncu_full_summary.txt,
                                        profiles/<tag>_ncu_hot_lines.txt
"""
import collections
import csv
import io
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(tag):
    src = os.path.join(ROOT, "gpurun_out", f"{tag}_ncu_launches.csv")
    shutil.copy(src, os.path.join(ROOT, "profiles", f"{tag}_ncu_launches.csv"))
    lines = [ln for ln in open(src) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        key = (r["Kernel Name"][:60], r["Grid Size"], r["Block Size"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        agg.setdefault(key, []).append(us)
    out = [f"ncu --metrics gpu__time_duration.sum --clock-control none -c 400 of "
           f"`python bench.py --steps 2 --warmup 3 --no-cpu-baseline`",
           "(serialised, cold cache; absolute times are not bench values, the kernel's share of the step is).", ""]
    for (name, grid, block), ts in agg.items():
        out.append(f"{name:60s} grid {grid:>14s} block {block:>12s} launches {len(ts):3d}  mean {sum(ts) / len(ts):9.1f} us")
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_launches_summary.txt"), "w").write("\n".join(out) + "\n")


def full(tag):
    rep = os.path.join(ROOT, "gpurun_out", f"{tag}_full.ncu-rep")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True, check=True).stdout
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_summary.txt"), "w").write(txt)
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "60"],
                         capture_output=True, text=True, check=True).stdout
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_hot_lines.txt"), "w").write(hot)


if __name__ == "__main__":
    t = sys.argv[1]
    launches(t)
    full(t)
