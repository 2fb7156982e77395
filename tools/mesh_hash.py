"""Hash of the refined mesh (every output array) for A/B identity checks
between engine builds (GDP2D_ENGINE_LIB).  GPU box only.
    python tools/mesh_hash.py N M DIST THETA [insert_mode]"""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host  # noqa: E402

n, m, dist, theta = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], float(sys.argv[4])
mode = int(sys.argv[5]) if len(sys.argv) > 5 else 0
pts, segs = host.generate_pslg(n, m, dist, 20261017)
mesh, _ = host.build_cdt(pts, segs)
with Engine(0) as eng:
    eng.upload(mesh)
    rep = eng.refine(QualityCriteria(theta), EngineConfig(insert_mode=mode))
    out = eng.download()
h = hashlib.sha256()
for name in ("xy", "tri_v", "tri_n", "tri_seg", "tri_alive", "seg_v", "seg_alive", "vert_tri", "seg_tri"):
    h.update(getattr(out, name).tobytes())
print(f"{n} {dist} {theta:.3f} mode={mode}: steiner={rep.steiner_points} batches={len(rep.batches)} sha={h.hexdigest()[:16]}")
