"""One warm refinement under GDP2D_TRACE (set by the caller) of a BASELINE
config; the engine prints per-batch host events and device step traces to
stderr.  GPU box only.   GDP2D_TRACE=2 python tools/trace_run.py 3 2> t.txt"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2007_00324_b200 import Engine, QualityCriteria, host  # noqa: E402

B = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))
CFG = {1: (100_000, 1_000, "uniform", B), 2: (1_000_000, 100_000, "uniform", B),
       3: (5_000_000, 500_000, "gaussian", B), 4: (1_000_000, 100_000, "uniform", 30.0)}

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n, m, dist, theta = CFG[c]
pts, segs = host.generate_pslg(n, m, dist, 20261017)
mesh, _ = host.build_cdt(pts, segs)
with Engine(0) as eng:
    eng.upload(mesh)
    eng.refine(QualityCriteria(theta))      # warm-up run (also traced)
    print("=== second run ===", file=sys.stderr, flush=True)
    eng.upload(mesh)
    r = eng.refine(QualityCriteria(theta))
print(f"device {r.device_seconds * 1e3:.2f} ms, {len(r.batches)} batches")
