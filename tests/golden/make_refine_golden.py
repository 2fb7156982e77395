#!/usr/bin/env python
"""TEST INFRASTRUCTURE: full-refinement golden records from the reference.

For each BASELINE config (SURVEY 8(d) generator, seed 20261017) this runs,
entirely inside oracle/_ref (the unmodified cdtref headers + the generator):

    generate -> close_hull (cdt.hpp:447) -> build_cdt (cdt.hpp:483)
    -> cdtref::refine(m, q, EngineConfig{})        (refine.hpp:651-713)

and records the reference's Steiner count, batch count, wall time, its
quality summary (refine.hpp:614-645) and the histogram of per-triangle
minimum angles (0.5-degree bins over [0, 60], the corner formula of
verify.hpp:186-200).  The GPU test tests/test_gpu_refine_golden.py refines
the same PSLGs on the device and compares against these records; the PSLG
and initial-mesh digests let it prove the input is identical.

    python tests/golden/make_refine_golden.py [cfg ...]     (default: 1 2 3 4)

cfg3 and cfg4 each take ~6 min of one core; configs run in parallel
processes and the file is merged, so re-running one config keeps the others.
"""
from __future__ import annotations

import hashlib
import json
import math
import multiprocessing as mp
import os
import platform
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
OUT = HERE / "refine_cfg.json"
SEED = 20261017
B_THETA = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))
CFGS = {
    1: dict(n=100_000, m=1_000, dist="uniform", theta=B_THETA),
    2: dict(n=1_000_000, m=100_000, dist="uniform", theta=B_THETA),
    3: dict(n=5_000_000, m=500_000, dist="gaussian", theta=B_THETA),
    4: dict(n=1_000_000, m=100_000, dist="uniform", theta=30.0),
}


def pslg_digest(pts, segs) -> str:
    import numpy as np
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pts, np.float64).tobytes())
    h.update(np.ascontiguousarray(segs, np.uint32).tobytes())
    return h.hexdigest()[:32]


def run_one(k: int) -> dict:
    from oracle.ref import HIST_BIN_DEG, HIST_BINS, ref_workload
    from paper_2007_00324_b200.gdp2d import QualityCriteria
    c = CFGS[k]
    t0 = time.perf_counter()
    pts, closed, m = ref_workload(c["n"], c["m"], c["dist"], SEED)
    setup = time.perf_counter() - t0
    V, T, S = m.sizes()
    q = QualityCriteria(c["theta"])
    rep = m.refine(q)
    hist, mean = m.min_angle_hist()
    m.check_structure()
    return {
        "config": k, **c, "seed": SEED,
        "pslg_sha": pslg_digest(pts, closed), "n_segments_closed": int(len(closed)),
        "initial": {"vertices": V, "triangles": T, "subsegments": S},
        "steiner_points": rep.steiner_points, "output_points": rep.output_points,
        "batches": len(rep.batches), "wall_seconds": rep.wall_seconds,
        "bad_triangles": rep.bad_triangles, "min_angle_deg": rep.min_angle_deg,
        "max_edge": rep.max_edge, "mean_min_angle_deg": mean,
        "hist_bin_deg": HIST_BIN_DEG, "min_angle_hist": [int(x) for x in hist],
        "conforming": bool(m.conformity_ok(pts, closed)), "euler": m.euler_holds(),
        "cdt_violations": m.cdt_violations(),
        "setup_seconds": setup,
        "host": {"cpu": platform.processor() or platform.machine(), "nproc": os.cpu_count()},
        "engine": "cdtref::refine EngineConfig{} (sequential), oracle/_ref g++ -O3",
    }


def main(argv):
    ks = [int(a) for a in argv] or sorted(CFGS)
    old = json.loads(OUT.read_text()) if OUT.exists() else {}
    with mp.get_context("spawn").Pool(len(ks)) as pool:
        for r in pool.imap_unordered(run_one, ks):
            old[f"cfg{r['config']}"] = r
            OUT.write_text(json.dumps(old, indent=1, sort_keys=True) + "\n")
            print(f"cfg{r['config']}: {r['steiner_points']} Steiner, {r['batches']} batches, "
                  f"{r['wall_seconds']:.1f} s, mean min angle {r['mean_min_angle_deg']:.3f}",
                  flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
