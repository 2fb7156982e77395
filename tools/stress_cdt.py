"""Randomised device-CDT sweep: random PSLGs (generator, 500-500K points),
device build_cdt against the reference build_cdt as triangle sets and
subsegment sets.  GPU box only.   python tools/stress_cdt.py [--count 50]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2007_00324_b200 import build_cdt, host  # noqa: E402


def canon_tris(m):
    t = np.sort(m.tri_v[m.tri_alive.astype(bool)], axis=1)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def canon_segs(m):
    a = m.seg_alive.astype(bool)
    r = np.column_stack([np.sort(m.seg_v[a], axis=1), m.seg_parent[a]])
    return r[np.lexsort((r[:, 2], r[:, 1], r[:, 0]))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=50)
    a = ap.parse_args()
    rng = np.random.default_rng(7)
    fails = 0
    t0 = time.time()
    for k in range(a.count):
        n = int(rng.integers(500, 500_000))
        m = int(n * rng.choice([0.0, 0.02, 0.1, 0.25]))
        dist = str(rng.choice(["uniform", "gaussian"]))
        seed = int(rng.integers(1, 1 << 30))
        pts, segs = host.generate_pslg(n, m, dist, seed)
        closed = host.close_hull(pts, segs, check=False)
        dev, rep = build_cdt(pts, closed)
        ref, _ = host.build_cdt(pts, segs)
        ok = (np.array_equal(canon_tris(dev), canon_tris(ref)) and
              np.array_equal(canon_segs(dev), canon_segs(ref)))
        fails += not ok
        print(f"{k:3d} n={n:6d} m={len(segs):6d} {dist:8s} seed={seed:10d} -> {'ok' if ok else 'FAIL'} "
              f"T={rep['n_triangles']} pipes={rep['pipes_recovered']} rounds={rep['insert_rounds']} "
              f"{rep['seconds'] * 1e3:.1f} ms", flush=True)
    print(f"stress_cdt: {a.count - fails}/{a.count} ok in {time.time() - t0:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
