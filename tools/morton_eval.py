"""Spatial order of the uploaded mesh vs refinement time (VERDICT r1 'next' 4).

Permutes the initial CDT host-side before upload -- triangles by the Morton
key of their centroid, optionally vertices by the Morton key of their point --
and refines each variant.  GPU box only.

    python tools/morton_eval.py [configs ...]
"""
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2007_00324_b200 import Engine, QualityCriteria, host  # noqa: E402
from paper_2007_00324_b200.gdp2d import Mesh, _FIELDS  # noqa: E402

NONE = np.uint32(0xFFFFFFFF)
B = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))
CFG = {1: (100_000, 1_000, "uniform", B), 2: (1_000_000, 100_000, "uniform", B),
       3: (5_000_000, 500_000, "gaussian", B), 4: (1_000_000, 100_000, "uniform", 30.0)}


def morton(xy):
    lo, hi = xy.min(0), xy.max(0)
    q = ((xy - lo) / np.maximum(hi - lo, 1e-300) * 65535.0).astype(np.uint64)

    def spread(v):
        v = (v | (v << 8)) & 0x00FF00FF
        v = (v | (v << 4)) & 0x0F0F0F0F
        v = (v | (v << 2)) & 0x33333333
        v = (v | (v << 1)) & 0x55555555
        return v
    return spread(q[:, 0]) | (spread(q[:, 1]) << 1)


def remap(a, inv):
    out = a.copy()
    m = a != NONE
    out[m] = inv[a[m]]
    return out


def permute(m: Mesh, tris: bool, verts: bool) -> Mesh:
    d = {name: getattr(m, name).copy() for name, _, _ in _FIELDS}
    if verts:
        order = np.argsort(morton(d["xy"]), kind="stable")
        inv = np.empty_like(order, dtype=np.uint32)
        inv[order] = np.arange(order.size, dtype=np.uint32)
        for k in ("xy", "vert_kind", "vert_birth", "vert_alive", "vert_tri"):
            d[k] = d[k][order]
        d["tri_v"] = remap(d["tri_v"], inv)
        d["seg_v"] = remap(d["seg_v"], inv)
    if tris:
        c = d["xy"][d["tri_v"]].mean(axis=1)
        order = np.argsort(morton(c), kind="stable")
        inv = np.empty_like(order, dtype=np.uint32)
        inv[order] = np.arange(order.size, dtype=np.uint32)
        for k in ("tri_v", "tri_n", "tri_seg", "tri_alive"):
            d[k] = d[k][order]
        d["tri_n"] = remap(d["tri_n"], inv)
        d["vert_tri"] = remap(d["vert_tri"], inv)
        d["seg_tri"] = remap(d["seg_tri"], inv)
    d["batch_epoch"] = m.batch_epoch
    return Mesh(**d)


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [2, 3]
    for c in cfgs:
        n, mm, dist, theta = CFG[c]
        pts, segs = host.generate_pslg(n, mm, dist, 20261017)
        mesh, _ = host.build_cdt(pts, segs)
        q = QualityCriteria(theta)
        for name, t, v in (("as built", False, False), ("tris morton", True, False),
                           ("verts morton", False, True), ("both morton", True, True)):
            pm = permute(mesh, t, v)
            best = None
            with Engine(0) as eng:
                for _ in range(4):
                    eng.upload(pm)
                    r = eng.refine(q)
                    if best is None or r.device_seconds < best.device_seconds:
                        best = r
                val = eng.validate(q)
            print(f"cfg{c} {name:13s}: device {best.device_seconds * 1e3:7.2f} ms, "
                  f"{len(best.batches)} batches, {best.steiner_points} Steiner, "
                  f"bad {val['bad_triangles']} cdt {val['cdt_violations']} "
                  f"struct {val['structure_failure']}", flush=True)


if __name__ == "__main__":
    main()
