"""Per-batch device time of a warm refinement, bucketed by batch size
(where the time goes: big batches vs the latency-bound tail).  GPU box only.

    python tools/batch_profile.py [theta] [n] [m] [uniform|gaussian]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2007_00324_b200 import Engine, QualityCriteria, host  # noqa: E402


def main():
    theta = float(sys.argv[1]) if len(sys.argv) > 1 else 20.704811054635428
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    m = int(sys.argv[3]) if len(sys.argv) > 3 else n // 10
    dist = sys.argv[4] if len(sys.argv) > 4 else "uniform"
    pts, segs = host.generate_pslg(n, m, dist, 20261017)
    mesh0, _ = host.build_cdt(pts, segs)
    with Engine(0) as eng:
        for _ in range(3):
            eng.upload(mesh0)
            r = eng.refine(QualityCriteria(theta))
    buckets = {}
    for b in r.batches:
        t = sum(b.phase_breakdown.values())
        k = next(lim for lim in (1_000, 4_000, 30_000, 100_000, 10**9) if b.attempted <= lim)
        n, s = buckets.get(k, (0, 0.0))
        buckets[k] = (n + 1, s + t)
    print(f"device {r.device_seconds * 1e3:.1f} ms, batches {len(r.batches)}, "
          f"sum of batch phases {sum(s for _, s in buckets.values()) * 1e3:.1f} ms")
    for k in sorted(buckets):
        n, s = buckets[k]
        print(f"  attempted <= {k:>10}: {n:3d} batches, {s * 1e3:6.2f} ms, {s / n * 1e6:6.0f} us/batch")
    for b in r.batches:
        print("   ", b.batch_index, b.attempted,
              {k: round(v * 1e6) for k, v in b.phase_breakdown.items() if v},
              {k: b.counters[k] for k in ("inserted_midpoints", "inserted_circumcenters",
                                          "flips", "flip_rounds", "removal_rounds",
                                          "removed_redundant", "removed_dependent")})


if __name__ == "__main__":
    main()
