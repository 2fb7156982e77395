"""Device validators (k_verify.cu) agree with the
reference's host validators (mesh.hpp:505-557, verify.hpp:92-200) on valid
refined meshes, on unrefined CDTs, and on deliberately broken meshes; and
validate a BASELINE-size output in milliseconds."""
import numpy as np
import pytest

from gdp2d_testlib import B_SQRT2_THETA

pytestmark = pytest.mark.gpu


def _refined(n, m, dist, seed, theta=B_SQRT2_THETA):
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    pts, segs = host.generate_pslg(n, m, dist, seed)
    mesh, closed = host.build_cdt(pts, segs)
    return mesh, pts, closed, QualityCriteria(theta)


def test_valid_refinement_passes(built):
    from paper_2007_00324_b200 import Engine
    from oracle.ref import RefMesh
    mesh, pts, closed, q = _refined(20_000, 2_000, "uniform", 41)
    with Engine(0) as eng:
        eng.upload(mesh)
        before = eng.validate(q)
        eng.refine(q)
        after = eng.validate(q)
        out = eng.download()
    ref0 = RefMesh.from_mesh(mesh)
    assert before["structure_failure"] == 0 and before["cdt_violations"] == 0
    assert before["conformity_failures"] == 0
    assert before["bad_triangles"] == len(ref0.collect(q)) - int((ref0.collect(q)["kind"] == 0).sum())
    rm = RefMesh.from_mesh(out)
    assert after == {**after, "structure_failure": 0, "cdt_violations": 0, "bad_triangles": 0,
                     "conformity_failures": 0}
    assert rm.cdt_violations() == 0 and rm.conformity_ok(pts, closed) and rm.count_bad(q) == 0
    assert after["min_angle_deg"] >= q.theta - 1e-9


def test_broken_meshes_are_caught(built):
    from paper_2007_00324_b200 import Engine, Mesh
    from oracle.ref import RefMesh
    mesh, pts, closed, q = _refined(5_000, 500, "uniform", 42)
    with Engine(0) as eng:
        eng.upload(mesh)
        eng.refine(q)
        good = eng.download()
    # (1) move an interior Steiner vertex a little: breaks local Delaunay
    bad = good.copy()
    steiner = np.nonzero((bad.vert_kind == 2) & (bad.vert_alive == 1))[0]
    v = int(steiner[len(steiner) // 2])
    tris = np.nonzero(bad.tri_alive.astype(bool) & (bad.tri_v == v).any(1))[0]
    nb = [u for u in np.unique(bad.tri_v[tris]) if u != v]
    bad.xy[v] = 0.6 * bad.xy[v] + 0.4 * bad.xy[nb[0]]
    with Engine(0) as eng:
        eng.upload(bad)
        res = eng.validate(q)
    rm = RefMesh.from_mesh(bad)
    assert (res["cdt_violations"] > 0) == (rm.cdt_violations() > 0)
    # (2) drop a subsegment: the input segment is no longer covered
    cut = good.copy()
    s = int(np.nonzero(cut.seg_alive)[0][0])
    cut.seg_alive[s] = 0
    cut.tri_seg[cut.tri_seg == s] = 0xFFFFFFFF
    with Engine(0) as eng:
        eng.upload(cut)
        res = eng.validate(q)
    assert res["conformity_failures"] > 0
    assert not RefMesh.from_mesh(cut).conformity_ok(pts, closed)


def test_baseline_size_validation(built):
    """cfg 2 (1M points): refine and validate on the device."""
    import time
    from paper_2007_00324_b200 import Engine
    mesh, pts, closed, q = _refined(1_000_000, 100_000, "uniform", 20261017)
    with Engine(0) as eng:
        eng.upload(mesh)
        eng.refine(q)
        t = time.perf_counter()
        res = eng.validate(q)
        dt = time.perf_counter() - t
    assert res["structure_failure"] == 0 and res["cdt_violations"] == 0
    assert res["bad_triangles"] == 0 and res["conformity_failures"] == 0
    assert res["min_angle_deg"] >= q.theta - 1e-9
    assert dt < 5.0


def test_compacted_export_matches_write_node_ele(built):
    """the device-compacted export formats to exactly the
    reference's write_node_ele text (pslg_io.hpp:294-319) of the same mesh,
    while moving only the alive elements."""
    from paper_2007_00324_b200 import Engine, host
    mesh, pts, closed, q = _refined(20_000, 2_000, "gaussian", 43)
    with Engine(0) as eng:
        eng.upload(mesh)
        eng.refine(q)
        xy, marker, tri = eng.export_node_ele()
        full = eng.download()
    node, ele = host.format_node_ele(xy, marker, tri)
    rnode, rele = host.write_node_ele(full)
    assert node == rnode
    assert ele == rele
    assert len(xy) == full.alive_vertex_count() and len(tri) == full.alive_triangle_count()
