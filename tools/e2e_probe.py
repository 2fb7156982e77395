"""e2e timing of one config through the Engine API: upload + refine + download_to
vs upload + refine_to (overlapped download).  GPU box only."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2007_00324_b200 import Engine, PinnedPool, QualityCriteria, host  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    theta = float(sys.argv[2]) if len(sys.argv) > 2 else 20.704811054635428
    pts, segs = host.generate_pslg(n, n // 10, "uniform", 20261017)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(theta)
    pin_in = PinnedPool(m.n_vertices, m.n_triangles, m.n_subsegments)
    src = pin_in.load(m)
    pool = PinnedPool(6 * m.n_vertices, 6 * m.n_triangles, 6 * m.n_subsegments)
    with Engine(0) as eng:
        for mode in ("download_to", "refine_to", "download_to", "refine_to"):
            ts = []
            for _ in range(4):
                t = time.perf_counter()
                eng.upload(src)
                if mode == "refine_to":
                    rep, out = eng.refine_to(q, pool)
                else:
                    rep = eng.refine(q)
                    out = eng.download_to(pool)
                ts.append(time.perf_counter() - t)
            print(f"{mode:12s} e2e {min(ts[1:]) * 1e3:.1f} ms (device {rep.device_seconds * 1e3:.1f} ms, "
                  f"steiner {rep.steiner_points})", flush=True)


if __name__ == "__main__":
    main()
