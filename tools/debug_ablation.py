import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from paper_2007_00324_b200 import EngineConfig, QualityCriteria, RuleFlags, host, refine
from oracle.ref import RefMesh
from test_gpu_refine import batch_safety_holds

q = QualityCriteria(20.0)
pts, segs = host.generate_pslg(10_000, 1_000, "uniform", 2)
m, closed = host.build_cdt(pts, segs)
for name, rules in (("default", RuleFlags()), ("rule2off", RuleFlags(rule2_filtering_enabled=False)),
                    ("rule4off", RuleFlags(rule4_unified_collection=False)),
                    ("rule1=0", RuleFlags(rule1_compaction_threshold=0))):
    g = m.copy()
    rep = refine(g, q, EngineConfig(rules=rules))
    kept = sum(b.counters["removals_kept"] for b in rep.batches)
    print(name, "steiner", rep.steiner_points, "batches", len(rep.batches), "bad", rep.bad_triangles,
          "kept", kept, "safety", batch_safety_holds(g))
    if not batch_safety_holds(g):
        t = g.tri_v[g.tri_alive.astype(bool)]
        for i in range(3):
            x, y = t[:, (i + 1) % 3], t[:, (i + 2) % 3]
            bad = (g.vert_kind[x] == 2) & (g.vert_kind[y] == 2) & (g.vert_birth[x] == g.vert_birth[y]) & (g.vert_birth[x] > 0)
            for xx, yy in zip(x[bad][:3], y[bad][:3]):
                print("   pair", xx, yy, g.xy[xx], g.xy[yy], "birth", g.vert_birth[xx],
                      "dist", np.linalg.norm(g.xy[xx] - g.xy[yy]))
