"""Randomised robustness sweep: PSLGs of several sizes / distributions / seeds,
refined under several criteria, each result checked by the device validators
(structure, exact local CDT, quality, conformity).  GPU box only.

    python tools/stress.py [--count 40] [--max-n 300000]
"""
import argparse
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2007_00324_b200 import CHEW, RUPPERT, Engine, QualityCriteria, host  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=40)
    ap.add_argument("--max-n", type=int, default=300_000)
    a = ap.parse_args()
    rng = np.random.default_rng(2026)
    fails = 0
    t0 = time.time()
    with Engine(0) as eng:
        for k in range(a.count):
            n = int(rng.integers(1_000, a.max_n))
            m = int(n * rng.choice([0.01, 0.05, 0.1, 0.2]))
            dist = str(rng.choice(["uniform", "gaussian"]))
            seed = int(rng.integers(1, 1 << 30))
            theta = float(rng.choice([15.0, 20.704811054635428, 25.0, 28.0, 30.0]))
            mode = int(rng.choice([RUPPERT, CHEW]))
            ell = float(rng.choice([math.inf, math.inf, 4.0 / math.sqrt(n)]))
            device_cdt = bool(rng.integers(0, 2))
            pts, segs = host.generate_pslg(n, m, dist, seed)
            if device_cdt:
                eng.build_cdt(pts, host.close_hull(pts, segs, check=False))
            else:
                mesh, _ = host.build_cdt(pts, segs)
                eng.upload(mesh)
            q = QualityCriteria(theta, ell, mode)
            try:
                rep = eng.refine(q)
                v = eng.validate(q)
                ok = (v["structure_failure"] == 0 and v["cdt_violations"] == 0 and
                      v["bad_triangles"] == 0 and v["conformity_failures"] == 0 and
                      rep.bad_triangles == 0 and not rep.iteration_cap_hit)
            except Exception as e:  # noqa: BLE001
                ok, rep, v = False, None, {"error": str(e)[:200]}
            fails += not ok
            print(f"{k:3d} n={n:7d} m={m:6d} {dist:8s} seed={seed:10d} theta={theta:6.2f} "
                  f"mode={mode} ell={ell:.4g} devcdt={int(device_cdt)} -> "
                  f"{'ok' if ok else 'FAIL'} steiner={rep.steiner_points if rep else '-'} "
                  f"batches={len(rep.batches) if rep else '-'} {'' if ok else v}", flush=True)
    print(f"stress: {a.count - fails}/{a.count} ok in {time.time() - t0:.0f} s")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
