"""Compare the refined mesh after `cap` batches between two engine modes as a
set of triangles by coordinates (vertex ids differ between modes)."""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2007_00324_b200 import Engine, QualityCriteria, EngineConfig, host

mode, cap, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
pts, segs = host.generate_pslg(n, n // 10, "uniform", 20261017)
mesh, closed = host.build_cdt(pts, segs)
q = QualityCriteria(20.704811054635428)
with Engine(0) as eng:
    eng.upload(mesh)
    rep = eng.refine(q, EngineConfig(iteration_cap=cap))
    out = eng.download()
a = out.tri_alive.astype(bool)
P = out.xy[out.tri_v[a]]                     # (T, 3, 2)
order = np.lexsort((P[:, :, 1], P[:, :, 0]), axis=1) if False else None
# sort the 3 corners of each triangle lexicographically by (x, y)
key = P[:, :, 0] * 0  # placeholder
idx = np.argsort(P[:, :, 0] + 0 * P[:, :, 1], axis=1, kind="stable")
Ps = np.take_along_axis(P, idx[:, :, None], axis=1)
flat = Ps.reshape(len(Ps), 6)
flat = flat[np.lexsort(flat.T[::-1])]
np.save(f"/tmp/tris_{mode}_{cap}.npy", flat)
b = rep.batches[-1]
print(mode, cap, "T", int(a.sum()), "V", int(out.vert_alive.sum()), "last batch C", b.attempted,
      "ret", b.concurrency, "steiner", rep.steiner_points, flush=True)
