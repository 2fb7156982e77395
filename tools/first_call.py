"""First-call cost of a one-shot refine in a fresh process (1M-point PSLG):
device seconds of the first and second call and the slowest batches of each.
GPU box only.  Usage: first_call.py THETA [THETA ...]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2007_00324_b200 import QualityCriteria, host  # noqa: E402
from paper_2007_00324_b200.gdp2d import refine_c  # noqa: E402


def main():
    thetas = [float(t) for t in sys.argv[1:]] or [30.0, 30.0]
    pts, segs = host.generate_pslg(1_000_000, 100_000, "uniform", 20261017)
    mesh0, _ = host.build_cdt(pts, segs)
    for th in thetas:
        m = mesh0.copy()
        t0 = time.perf_counter()
        r = refine_c(m, QualityCriteria(th))
        wall = time.perf_counter() - t0
        per = sorted(((sum(b.phase_breakdown.values()), b.batch_index, b.attempted)
                      for b in r.batches), reverse=True)[:5]
        print(f"theta {th}: wall {wall * 1e3:.0f} ms  device {r.device_seconds * 1e3:.0f} ms  "
              f"refine-wall {r.wall_seconds * 1e3:.0f} ms  batches {len(r.batches)}  "
              f"steiner {r.steiner_points}", flush=True)
        for s, i, a in per:
            print(f"    batch {i}: {s * 1e3:.1f} ms  attempted {a}")


if __name__ == "__main__":
    main()
