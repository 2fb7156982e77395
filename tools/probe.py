"""Ad-hoc GPU probe: refine one BASELINE config, print per-batch counters and
validity checks against the reference validators.  Not part of the product."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host  # noqa: E402
import os  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--theta", type=float, default=20.704811054635428)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    m_segs = a.m or a.n // 10
    t = time.time()
    pts, segs = host.generate_pslg(a.n, m_segs, a.dist)
    mesh, closed = host.build_cdt(pts, segs)
    print(f"input: {a.n} pts {len(closed)} segs  T={mesh.n_triangles}  build {time.time()-t:.2f}s",
          flush=True)
    q = QualityCriteria(a.theta)
    with Engine(0) as eng:
        eng.upload(mesh)
        for r in range(a.reps):
            eng.reset()
            t = time.time()
            rep = eng.refine(q, EngineConfig(insert_mode=int(os.environ.get('GDP2D_MODE', '1'))))
            dt = time.time() - t
            print(f"rep {r}: wall {rep.wall_seconds*1e3:.1f} ms device {rep.device_seconds*1e3:.1f} ms "
                  f"py {dt*1e3:.1f} ms steiner {rep.steiner_points} batches {len(rep.batches)} "
                  f"bad {rep.bad_triangles} minang {rep.min_angle_deg:.4f} "
                  f"bytes_alg {rep.algorithmic_bytes()/1e9:.3f} GB", flush=True)
        if a.verbose:
            for b in rep.batches:
                c = b.counters
                ph = " ".join(f"{k[:4]}={v*1e3:.2f}" for k, v in b.phase_breakdown.items())
                print(f"  b{b.batch_index:3d} C={b.attempted:8d} ret={b.concurrency:7d} "
                      f"T={c['tris_alive']:9d} surv={c['survivors_claim']}/{c['survivors_cavity']} "
                      f"mid={c['inserted_midpoints']} cc={c['inserted_circumcenters']} "
                      f"red={c['removed_redundant']} dep={c['removed_dependent']} "
                      f"mark={c['marked_encroached']} drop={c['dropped']} flips={c['flips']} "
                      f"fr={c['flip_rounds']} rr={c['removal_rounds']} kept={c['removals_kept']} | {ph}", flush=True)
        tot = {}
        for b in rep.batches:
            for k, v in b.phase_breakdown.items():
                tot[k] = tot.get(k, 0.0) + v
        print("phase totals (ms): " + " ".join(f"{k}={v*1e3:.2f}" for k, v in tot.items()),
              f"sum={sum(tot.values())*1e3:.2f}", flush=True)
        print("totals: " + " ".join(f"{k}={v}" for k, v in rep.totals.items()), flush=True)
        out = eng.download()
    if a.check or a.ref:
        from oracle.ref import RefMesh
        if a.check:
            chk = RefMesh.from_mesh(out)
            t = time.time()
            chk.check_structure()
            print("check_structure ok; euler", chk.euler_holds(), "conform",
                  chk.conformity_ok(pts, closed), "bad", chk.count_bad(q),
                  f"({time.time()-t:.1f}s)", flush=True)
            if out.n_vertices <= 300_000:
                print("cdt violations", chk.cdt_violations(), flush=True)
        if a.ref:
            ref = RefMesh.from_mesh(mesh)
            t = time.time()
            rr = ref.refine(q)
            print(f"reference: {rr.wall_seconds:.2f}s steiner {rr.steiner_points} batches "
                  f"{len(rr.batches)} (py {time.time()-t:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
