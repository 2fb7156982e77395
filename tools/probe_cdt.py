"""Time the device CDT builder (k_cdt.cu) against the reference build_cdt.

    python tools/probe_cdt.py --n 1000000 --dist uniform [--ref]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--m", type=int, default=-1)
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref", action="store_true")
    a = ap.parse_args()
    from paper_2007_00324_b200 import Engine, host
    m = a.m if a.m >= 0 else a.n // 10
    pts, segs = host.generate_pslg(a.n, m, a.dist, 20261017)
    closed = host.close_hull(pts, segs, check=False)
    with Engine(0) as eng:
        for r in range(a.reps):
            t0 = time.perf_counter()
            rep = eng.build_cdt(pts, closed)
            dt = time.perf_counter() - t0
            print(f"rep {r}: wall {dt * 1e3:.1f} ms device {rep['seconds'] * 1e3:.1f} ms "
                  f"(delaunay {rep['delaunay_seconds'] * 1e3:.1f} recover "
                  f"{rep['recover_seconds'] * 1e3:.1f} finish {rep['finish_seconds'] * 1e3:.1f}) "
                  f"T={rep['n_triangles']} S={rep['n_subsegments']} rounds={rep['insert_rounds']} "
                  f"flip_rounds={rep['flip_rounds']} flips={rep['flips']} "
                  f"present={rep['segments_present']} pipes={rep['pipes_recovered']} "
                  f"rec_rounds={rep['recover_rounds']} max_pipe={rep['max_pipe']} "
                  f"final_rounds={rep['final_flip_rounds']}", flush=True)
    if a.ref:
        t0 = time.perf_counter()
        ref, _ = host.build_cdt(pts, segs)
        print(f"reference build_cdt: {time.perf_counter() - t0:.2f} s, T={int(ref.tri_alive.sum())}")


if __name__ == "__main__":
    main()
