"""Debug: refine until a device error, download the working mesh, dump the
neighbourhood of the reported vertex."""
import re
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2007_00324_b200 import Engine, QualityCriteria, host
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
pts, segs = host.generate_pslg(n, n // 10, "uniform")
mesh, closed = host.build_cdt(pts, segs)
q = QualityCriteria(20.704811054635428)
with Engine(0) as eng:
    eng.upload(mesh)
    try:
        rep = eng.refine(q)
        print("no error", rep.steiner_points)
        sys.exit(0)
    except Exception as e:
        msg = str(e)
        print(msg)
    out = eng.download()
v = int(re.search(r"info (\d+)", msg).group(1))
alive = out.tri_alive.astype(bool)
tv = out.tri_v
inc = np.where(alive & ((tv == v).any(axis=1)))[0]
print("vertex", v, "xy", out.xy[v], "kind", out.vert_kind[v], "birth", out.vert_birth[v], "alive", out.vert_alive[v])
print("incident alive triangles:", len(inc))
nb = set()
for t in inc:
    for u in tv[t]:
        if u != v:
            nb.add(int(u))
nb = sorted(nb)
print("neighbours", len(nb))
kinds = out.vert_kind[nb]; births = out.vert_birth[nb]; al = out.vert_alive[nb]
print("neighbour kinds", np.bincount(kinds, minlength=3), "alive", al.sum(), "births", np.unique(births, return_counts=True))
d = np.linalg.norm(out.xy[nb] - out.xy[v], axis=1)
print("neighbour dist min/median/max", d.min(), np.median(d), d.max())
for t in inc[:10]:
    a, b, c = out.xy[tv[t]]
    area = 0.5 * ((b[0]-a[0])*(c[1]-a[1]) - (b[1]-a[1])*(c[0]-a[0]))
    print(" tri", t, tv[t], "area", area, "kinds", out.vert_kind[tv[t]], "births", out.vert_birth[tv[t]])
