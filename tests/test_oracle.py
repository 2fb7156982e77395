"""The C restatement (oracle/cdt_oracle.c) pinned against the compiled
reference: predicate known answers (test_predicates.cpp:52-181), seeded
near-degenerate vectors, the committed golden fixtures, and the hot-path
phases (collect / locate / claim / cavity) on identical meshes."""
import json
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import gdp2d_cases as G
from gdp2d_testlib import B_SQRT2_THETA, small_corpus

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def R(built):
    from oracle import ref
    return ref


def _both(R, kind, pts, q=None):
    a = R.orc_predicates(kind, pts, q)
    b = R.ref_predicates(kind, pts, q)
    assert np.array_equal(a, b), np.nonzero(a != b)[0][:5]
    return a


def test_known_answers(R):
    # test_predicates.cpp:52-63, 126-140
    o = np.array([[[0, 0], [1, 0], [0, 1]], [[0, 0], [1, 1], [2, 2]], [[0, 0], [0, 1], [1, 0]]], float)
    assert _both(R, 0, o).tolist() == [1, 0, -1]
    a, b, c = [1, 0], [0, 1], [-1, 0]
    ic = np.array([[a, b, c, [0, 0]], [a, b, c, [0, -1]], [a, b, c, [0, -2]]], float)
    assert _both(R, 1, ic).tolist() == [1, 0, -1]
    sa, sb = [0, 0], [2, 0]
    d = np.array([[sa, sb, [1, 0.5]], [sa, sb, [3, 0]], [sa, sb, [0, 0]], [sa, sb, [1, 1]],
                  [sa, sb, [1, 0.99]]], float)
    assert _both(R, 2, d).tolist() == [1, 0, 0, 0, 1]
    assert _both(R, 3, d).tolist() == [1, 0, 0, 0, 0]


def _frac_orient(p):
    (ax, ay), (bx, by), (cx, cy) = [(Fraction(x), Fraction(y)) for x, y in p]
    d = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    return (d > 0) - (d < 0)


def _frac_incircle(p):
    q = [(Fraction(x), Fraction(y)) for x, y in p]
    (dx, dy) = q[3]
    rows = [(x - dx, y - dy, (x - dx) ** 2 + (y - dy) ** 2) for x, y in q[:3]]
    (ax, ay, al), (bx, by, bl), (cx, cy, cl) = rows
    det = ax * (by * cl - bl * cy) - ay * (bx * cl - bl * cx) + al * (bx * cy - by * cx)
    return (det > 0) - (det < 0)


def test_exactness_vs_rational_oracle(R):
    """test_predicates.cpp:90-124 with Python Fractions instead of Boost cpp_int."""
    pts = G.near_collinear(3000)
    got = _both(R, 0, pts)
    assert got.tolist() == [_frac_orient(p) for p in pts]
    pts = G.near_cocircular(1500)
    got = _both(R, 1, pts)
    assert got.tolist() == [_frac_incircle(p) for p in pts]
    pts = G.mesh_scale_cocircular(1500)
    got = _both(R, 1, pts)
    assert got.tolist() == [_frac_incircle(p) for p in pts]


def test_seeded_vectors(R):
    _both(R, 0, G.random_points(20_000, 3))
    _both(R, 0, G.grid_degenerate(20_000, 3))
    _both(R, 1, G.random_points(20_000, 4))
    _both(R, 1, G.grid_degenerate(20_000, 4))
    _both(R, 1, G.mesh_scale_cocircular(20_000))
    _both(R, 2, G.diametric_cases(20_000))
    _both(R, 3, G.diametric_cases(20_000))
    from paper_2007_00324_b200 import QualityCriteria
    for th in (20.0, B_SQRT2_THETA, 30.0):
        _both(R, 4, G.triangles_near_bound(th, 5000), QualityCriteria(th))


def test_golden_fixtures(R):
    """tests/golden/*.npz were produced by tests/golden/make_golden.py from the
    reference itself; the C restatement must reproduce them exactly."""
    from paper_2007_00324_b200 import QualityCriteria
    for f in sorted(GOLDEN.glob("pred_*.npz")):
        z = np.load(f)
        q = QualityCriteria(float(z["theta"]))
        assert np.array_equal(R.orc_predicates(int(z["kind"]), z["pts"], q), z["out"]), f.name
    meta = json.loads((GOLDEN / "phases.json").read_text())
    for case in meta["cases"]:
        z = np.load(GOLDEN / case["file"])
        from paper_2007_00324_b200.gdp2d import Mesh
        m = Mesh(**{k[2:]: z[k] for k in z.files if k.startswith("m_")}, batch_epoch=0)
        q = QualityCriteria(case["theta"])
        c = R.orc_collect(m, q)
        assert np.array_equal(c, z["collect"]), case["file"]
        c = R.orc_locate(m, c)
        assert np.array_equal(c, z["locate"])
        c = R.orc_claim(m, c)
        assert np.array_equal(c, z["claim"])
        c = R.orc_cavity(m, c, 32)
        assert np.array_equal(c, z["cavity"])


def test_phases_match_reference(R):
    from paper_2007_00324_b200 import QualityCriteria, host
    meshes = []
    pts, segs = host.generate_pslg(20_000, 2_000, "gaussian", 3)
    meshes.append(host.build_cdt(pts, segs)[0])
    for name, (p, s) in list(small_corpus().items())[:2]:
        meshes.append(host.build_cdt(p, s)[0])
    for m in meshes:
        rm = R.RefMesh.from_mesh(m)
        for theta in (B_SQRT2_THETA, 30.0):
            q = QualityCriteria(theta)
            a, b = R.orc_collect(m, q), rm.collect(q)
            assert np.array_equal(a, b)
            a, b = R.orc_locate(m, b), rm.locate(b)
            assert np.array_equal(a, b)
            a, b = R.orc_claim(m, b), rm.claim_filter(b)
            assert np.array_equal(a, b)
            for n in (32, 3):
                assert np.array_equal(R.orc_cavity(m, b, n), rm.cavity_filter(b, n))


def test_refine_golden_cfg1_reproduces():
    """tests/golden/refine_cfg.json is the reference's own output: re-running
    the committed recipe (make_refine_golden.run_one) for config 1 gives the
    same PSLG digest, Steiner count, batch count and min-angle histogram."""
    import json
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(here))
    import make_refine_golden as mk
    gold = json.loads((here / "refine_cfg.json").read_text())
    r = mk.run_one(1)
    g = gold["cfg1"]
    for k in ("pslg_sha", "steiner_points", "batches", "min_angle_hist", "initial",
              "bad_triangles", "conforming"):
        assert r[k] == g[k], k
    assert abs(r["mean_min_angle_deg"] - g["mean_min_angle_deg"]) < 1e-12
    for k in ("cfg2", "cfg3", "cfg4"):
        assert gold[k]["conforming"] and sum(gold[k]["min_angle_hist"]) > 0
    for k in ("cfg2", "cfg4"):
        assert gold[k]["bad_triangles"] == 0 and gold[k]["cdt_violations"] == 0
    # recorded as found: the reference's own config-3 output keeps one bad
    # triangle and fails its own constrained-Delaunay check
    # (constrained_delaunay_violations, verify.hpp:92, capped at 32) on 22
    assert gold["cfg3"]["bad_triangles"] == 1 and gold["cfg3"]["cdt_violations"] == 22
