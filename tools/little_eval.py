"""Little's-law batch sizing on vs off (EngineConfig.little_batch_sizing):
per-batch attempted A, concurrency U (retained insertions), latency L,
throughput T = U / L and waste 1 - U / A (record_batch, ruleskit.hpp:128-142),
plus the device time and Steiner count of each whole refinement.  GPU box only.

    python tools/little_eval.py [configs ...]  > profiles/rXX_little.md
"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host  # noqa: E402

B = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))
CFG = {1: (100_000, 1_000, "uniform", B), 2: (1_000_000, 100_000, "uniform", B),
       3: (5_000_000, 500_000, "gaussian", B), 4: (1_000_000, 100_000, "uniform", 30.0)}


def run(eng, q, little):
    best = None
    for _ in range(3):
        eng.reset()
        r = eng.refine(q, EngineConfig(little_batch_sizing=little))
        if best is None or r.device_seconds < best.device_seconds:
            best = r
    return best


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]
    for c in cfgs:
        n, m, dist, theta = CFG[c]
        pts, segs = host.generate_pslg(n, m, dist, 20261017)
        mesh, _ = host.build_cdt(pts, segs)
        q = QualityCriteria(theta)
        with Engine(0) as eng:
            eng.upload(mesh)
            eng.refine(q)
            off = run(eng, q, False)
            on = run(eng, q, True)
        print(f"## cfg{c}: {n} {dist} points, theta {theta:.3f}\n")
        for name, r in (("off", off), ("on", on)):
            print(f"- little_batch_sizing {name}: device {r.device_seconds * 1e3:.2f} ms, "
                  f"{len(r.batches)} batches, {r.steiner_points} Steiner")
        print("\n| batch | A (off) | U | L ms | T (M/s) | waste | A (on) | U | L ms | T (M/s) | waste |")
        print("|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
        for i in range(max(len(off.batches), len(on.batches))):
            cells = [str(i)]
            for r in (off, on):
                if i < len(r.batches):
                    b = r.batches[i]
                    cells += [str(b.attempted), str(b.concurrency), f"{b.latency * 1e3:.3f}",
                              f"{b.throughput / 1e6:.2f}", f"{b.waste_fraction:.3f}"]
                else:
                    cells += [""] * 5
            print("| " + " | ".join(cells) + " |")
        print()


if __name__ == "__main__":
    main()
