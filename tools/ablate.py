"""Debug: run each rule-ablation variant and report which invariant fails."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from paper_2007_00324_b200 import EngineConfig, QualityCriteria, RuleFlags, host, refine
from oracle.ref import RefMesh
q = QualityCriteria(20.0)
pts, segs = host.generate_pslg(10_000, 1_000, "uniform", 2)
m, closed = host.build_cdt(pts, segs)
for name, rules in (("no-rule2", RuleFlags(rule2_filtering_enabled=False)),
                    ("no-rule4", RuleFlags(rule4_unified_collection=False)),
                    ("rule1=0", RuleFlags(rule1_compaction_threshold=0))):
    out = m.copy()
    rep = refine(out, q, EngineConfig(rules=rules))
    rm = RefMesh.from_mesh(out)
    print(name, "batches", len(rep.batches), "cap", rep.iteration_cap_hit, "steiner", rep.steiner_points,
          "bad", rep.bad_triangles, "collect", len(rm.collect(q)),
          "cdt", rm.cdt_violations(), flush=True)
    for b in rep.batches[-3:]:
        print("   ", b)
