"""Summarise ncu captures (gpurun_out/) into a markdown table for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches_c2.csv \
        --reports gpurun_out/prof_*.ncu-rep --out profiles/r01_ncu_summary.md

Launch list: per-kernel launch count, summed gpu__time_duration and share
(cold-cache, serialised replay: compare SHARES).  Full captures: duration,
DRAM bytes, DRAM % of peak, achieved occupancy, warp execution efficiency
(threads per executed instruction / 32), registers.
"""
from __future__ import annotations

import argparse
import collections
import csv
import glob
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst (of 32)"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0}


def launch_table(path: str):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"Launch list `{path}`: {sum(v[0] for v in agg.values())} launches, "
           f"{tot * 1e3:.3f} ms summed kernel time (cold-cache, serialised).", "",
           "| kernel | launches | sum (ms) | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1] * 1e3:.3f} | {100 * v[1] / tot:.1f}% |")
    return out


def report_table(paths):
    out = ["| kernel | " + " | ".join(n for _, n in METRICS) + " |",
           "|---|" + "---:|" * len(METRICS)]
    for p in paths:
        txt = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 3:
            continue
        h, u = rows[0], rows[1]
        for v in rows[2:]:
            name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
            cells = []
            for key, _ in METRICS:
                if key not in h:
                    cells.append("-")
                    continue
                i = h.index(key)
                cells.append(f"{v[i]} {u[i]}".strip())
            out.append(f"| `{name}` | " + " | ".join(cells) + " |")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--reports", nargs="*", default=[])
    ap.add_argument("--out")
    ap.add_argument("--title", default="ncu summary")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.launches:
        lines += launch_table(a.launches) + [""]
    reps = sorted(p for g in a.reports for p in glob.glob(g))
    if reps:
        lines += ["Full captures (`ncu --set full --clock-control none`):", ""]
        lines += report_table(reps) + [""]
    text = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
