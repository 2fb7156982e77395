"""Regenerate the golden fixtures from the REFERENCE itself (oracle/_ref,
compiled from the unmodified /root/reference/proj/include headers).  Run in
the build container: python tests/golden/make_golden.py

  pred_<kind>.npz : seeded predicate inputs + the reference's outputs
  phase_<name>.npz: a small initial CDT (reference build_cdt) with the
                    reference's collect / locate / claim / cavity lists
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

import gdp2d_cases as G  # noqa: E402
from gdp2d_testlib import B_SQRT2_THETA, small_corpus  # noqa: E402
from oracle import ref as R  # noqa: E402
from paper_2007_00324_b200 import QualityCriteria  # noqa: E402


def main():
    preds = {
        "orient": (0, np.concatenate([G.near_collinear(2000, 101), G.grid_degenerate(1000, 3, 102),
                                      G.mesh_scale_collinear(1000, 103)]), 20.0),
        "incircle": (1, np.concatenate([G.near_cocircular(1000, 104), G.grid_degenerate(1000, 4, 105),
                                        G.mesh_scale_cocircular(1000, 106)]), 20.0),
        "diametric": (2, G.diametric_cases(2000, 107), 20.0),
        "lens": (3, G.diametric_cases(2000, 108), 20.0),
        "bad": (4, G.triangles_near_bound(B_SQRT2_THETA, 2000, 109), B_SQRT2_THETA),
    }
    for name, (kind, pts, theta) in preds.items():
        out = R.ref_predicates(kind, pts, QualityCriteria(theta))
        np.savez_compressed(HERE / f"pred_{name}.npz", kind=kind, pts=pts, out=out, theta=theta)
    cases = []
    corpus = small_corpus()
    inputs = {"square-100": corpus["square-100"], "hexagon-200": corpus["hexagon-200"]}
    for name, (pts, segs) in inputs.items():
        closed_n = R.ref_lib().ref_close_hull
        import ctypes as C
        segs = np.ascontiguousarray(segs, np.uint32)
        out = np.zeros((len(segs) + len(pts)) * 2, np.uint32)
        m_out = closed_n(np.ascontiguousarray(pts).ctypes.data, len(pts), segs.ctypes.data,
                         len(segs), out.ctypes.data)
        closed = out[: 2 * m_out].reshape(-1, 2)
        rm = R.RefMesh.build_cdt(pts, closed)
        mesh = rm.to_mesh()
        for theta in (B_SQRT2_THETA, 30.0):
            q = QualityCriteria(theta)
            col = rm.collect(q)
            loc = rm.locate(col)
            clm = rm.claim_filter(loc)
            cav = rm.cavity_filter(clm, 32)
            fname = f"phase_{name}_{int(theta)}.npz"
            arrays = {f"m_{k}": getattr(mesh, k) for k in (
                "xy", "vert_kind", "vert_birth", "vert_alive", "vert_tri", "tri_v", "tri_n",
                "tri_seg", "tri_alive", "seg_v", "seg_parent", "seg_encroached", "seg_alive",
                "seg_tri")}
            np.savez_compressed(HERE / fname, collect=col, locate=loc, claim=clm, cavity=cav,
                                **arrays)
            cases.append({"file": fname, "theta": theta, "candidates": int(len(col))})
    (HERE / "phases.json").write_text(json.dumps({"cases": cases}, indent=1))
    print("golden fixtures written:", [c["file"] for c in cases])


if __name__ == "__main__":
    main()
