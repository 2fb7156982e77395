"""Average ncu DRAM traffic per launch for the engine kernels -> profiles/traffic.json.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        -k regex:'k_collect_flags|k_batch_split|k_batch_rollback' --csv \
        --log-file gpurun_out/traffic_c2.csv python tools/probe.py --n 1000000 --reps 1
    python tools/traffic.py gpurun_out/traffic_c2.csv config2
"""
import collections
import csv
import json
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    path, key = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, ii = h.index("Kernel Name"), h.index("ID")
    mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    per = collections.defaultdict(float)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[mi].startswith("dram__bytes"):
            continue
        per[r[ii]] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
    agg = collections.defaultdict(list)
    for i, b in per.items():
        agg[names[i]].append(b)
    out_p = Path(__file__).resolve().parent.parent / "profiles" / "traffic.json"
    db = json.loads(out_p.read_text()) if out_p.exists() else {}
    db[key] = {k: sum(v) / len(v) for k, v in agg.items()}
    db[key + "_launches"] = {k: len(v) for k, v in agg.items()}
    out_p.write_text(json.dumps(db, indent=1) + "\n")
    print(json.dumps(db[key], indent=1))


if __name__ == "__main__":
    main()
