"""Per-CUDA-line warp-stall samples of an ncu report (source page, cuda,sass).

    python tools/ncu_lines.py report.ncu-rep [--top 40] [--kernel REGEX]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--skip", type=int, default=-1, help="result index in the report")
    a = ap.parse_args()
    extra = ["--launch-skip", str(a.skip), "--launch-count", "1"] if a.skip >= 0 else []
    txt = subprocess.run(["ncu", "-i", a.report] + extra + [ "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    agg = collections.Counter()
    src = {}
    fname, line, hdr = None, None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 5:
            continue
        if r[0]:
            line = (fname, int(r[0]))
            src[line] = r[1].strip()[:100]
            continue
        try:
            agg[line] += int(r[4] or 0)
        except ValueError:
            pass
    tot = sum(agg.values())
    print(f"total samples {tot}")
    for (f, ln), s in agg.most_common(a.top):
        print(f"{100 * s / max(tot, 1):5.1f}% {s:7d} {f}:{ln}  {src.get((f, ln), '')}")


if __name__ == "__main__":
    main()
