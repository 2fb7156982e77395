"""Device Line-1 CDT (k_cdt.cu) against the reference's
build_cdt (cdt.hpp:483 = build_delaunay :198 + recover_segments :437).

The CDT of a PSLG in general position is unique, so the device mesh must
equal the reference's as a SET of triangles (ids differ) and carry the same
subsegments with the same parents; the reference's check_structure must pass
on it; refinement from it must behave like refinement from the host CDT.
Error behaviour mirrors CdtError (duplicate points, all collinear, crossing
segments)."""
import numpy as np
import pytest

from gdp2d_testlib import B_SQRT2_THETA, small_corpus, unit_square

pytestmark = pytest.mark.gpu


def _tris(mesh):
    t = mesh.tri_v[mesh.tri_alive.astype(bool)]
    t = np.sort(t, axis=1)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))]


def _segs(mesh):
    a = mesh.seg_alive.astype(bool)
    s = np.sort(mesh.seg_v[a], axis=1)
    rows = np.column_stack([s, mesh.seg_parent[a]])
    return rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]


def _check_against_reference(pts, segs):
    from paper_2007_00324_b200 import build_cdt, host
    from oracle.ref import RefMesh
    closed = host.close_hull(pts, segs)
    dev, rep = build_cdt(pts, closed)
    ref, _ = host.build_cdt(pts, segs)
    assert rep["n_triangles"] == int(ref.tri_alive.sum())
    np.testing.assert_array_equal(_tris(dev), _tris(ref))
    np.testing.assert_array_equal(_segs(dev), _segs(ref))
    # subsegment ids follow the reference's numbering (segment order)
    np.testing.assert_array_equal(dev.seg_parent, ref.seg_parent)
    np.testing.assert_array_equal(np.sort(dev.seg_v, axis=1), np.sort(ref.seg_v, axis=1))
    assert (dev.vert_kind == 0).all() and (dev.vert_alive == 1).all()
    np.testing.assert_array_equal(dev.xy, ref.xy)
    rm = RefMesh.from_mesh(dev)
    rm.check_structure()
    assert rm.euler_holds()
    assert rm.cdt_violations() == 0
    assert rm.conformity_ok(pts, closed)
    return dev, rep


@pytest.mark.parametrize("dist,n,m,seed", [("uniform", 20_000, 2_000, 3),
                                          ("gaussian", 20_000, 2_000, 4),
                                          ("uniform", 2_000, 1_000, 5)])
def test_generator_pslg_equals_reference(built, dist, n, m, seed):
    from paper_2007_00324_b200 import host
    pts, segs = host.generate_pslg(n, m, dist, seed)
    _, rep = _check_against_reference(pts, segs)
    assert rep["insert_rounds"] > 0 and rep["segments_present"] + rep["pipes_recovered"] >= len(segs)


@pytest.mark.parametrize("name", sorted(small_corpus()))
def test_polygon_corpus_equals_reference(built, name):
    pts, segs = small_corpus()[name]
    _check_against_reference(pts, segs)


def test_unit_square(built):
    pts, segs = unit_square()
    dev, rep = _check_against_reference(pts, segs)
    assert rep["n_triangles"] == 2


def test_long_segments_through_point_cloud(built):
    """Long segments cross many Delaunay edges: multi-triangle pipes, several
    recovery rounds (segments sharing triangles)."""
    rng = np.random.default_rng(11)
    inner = rng.uniform(0.02, 0.98, size=(3000, 2))
    corners = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], np.float64)
    ends = np.array([[0.01, 0.2], [0.99, 0.25], [0.01, 0.45], [0.99, 0.4],
                     [0.01, 0.6], [0.99, 0.65], [0.01, 0.85], [0.99, 0.8]], np.float64)
    pts = np.vstack([corners, ends, inner])
    # drop interior points lying too close to the long segments (no collinear hits)
    segs = np.array([[4, 5], [6, 7], [8, 9], [10, 11]], np.uint32)
    keep = np.ones(len(pts), bool)
    for a, b in segs:
        pa, pb = pts[a], pts[b]
        d = pb - pa
        t = np.clip(((pts - pa) @ d) / (d @ d), 0, 1)
        dist = np.linalg.norm(pts - (pa + t[:, None] * d), axis=1)
        keep &= (dist > 1e-4) | (np.arange(len(pts)) < 12)
    pts = pts[keep]
    _, rep = _check_against_reference(pts, segs)
    assert rep["max_pipe"] > 10
    assert rep["pipes_recovered"] >= 4


def test_segment_through_vertex_splits_like_recover_chain(built):
    """A vertex exactly on a segment splits it (recover_chain cdt.hpp:386-389):
    two subsegments with the same parent, numbered along the segment."""
    rng = np.random.default_rng(5)
    inner = rng.uniform(0.05, 0.95, size=(400, 2))
    inner = inner[np.abs(inner[:, 1] - 0.5) > 0.02]
    fixed = np.array([[0, 0], [1, 0], [1, 1], [0, 1], [0.125, 0.5], [0.875, 0.5], [0.5, 0.5],
                      [0.25, 0.5]], np.float64)
    pts = np.vstack([fixed, inner])
    segs = np.array([[4, 5]], np.uint32)
    dev, rep = _check_against_reference(pts, segs)
    assert rep["collinear_splits"] >= 1


def test_determinism(built):
    from paper_2007_00324_b200 import build_cdt, host
    pts, segs = host.generate_pslg(30_000, 3_000, "gaussian", 9)
    closed = host.close_hull(pts, segs)
    a, _ = build_cdt(pts, closed)
    b, _ = build_cdt(pts, closed)
    for name in ("tri_v", "tri_n", "tri_seg", "seg_v", "seg_parent", "vert_tri", "seg_tri"):
        np.testing.assert_array_equal(getattr(a, name), getattr(b, name), err_msg=name)


def test_errors_match_cdterror(built):
    from paper_2007_00324_b200 import CdtError, Engine
    with Engine(0) as eng:
        pts = np.array([[0, 0], [1, 0], [0, 1], [1, 0]], np.float64)     # duplicate
        with pytest.raises(CdtError, match="duplicate"):
            eng.build_cdt(pts, np.array([[0, 1], [1, 2], [2, 0]], np.uint32))
        pts = np.array([[0, 0], [1, 1], [2, 2], [3, 3]], np.float64)     # all collinear
        with pytest.raises(CdtError, match="collinear"):
            eng.build_cdt(pts, np.array([[0, 1], [1, 2], [2, 3]], np.uint32))
        pts = np.array([[0, 0], [4, 0], [4, 4], [0, 4], [1, 1], [3, 3], [1, 3], [3, 1]],
                       np.float64)                                        # crossing segments
        segs = np.array([[0, 1], [1, 2], [2, 3], [3, 0], [4, 5], [6, 7]], np.uint32)
        with pytest.raises(CdtError, match="cross"):
            eng.build_cdt(pts, segs)
        pts = np.array([[0, 0], [1, 0], [np.nan, 1]], np.float64)
        with pytest.raises(CdtError, match="finite"):
            eng.build_cdt(pts, np.zeros((0, 2), np.uint32))
        # the context is still usable after an error
        pts, segs = unit_square()
        assert eng.build_cdt(pts, segs)["n_triangles"] == 2


def test_refine_from_device_cdt(built):
    """Lines 1-9 on the device: build, refine, validate; Steiner count close to
    refining the host CDT (triangle ids differ, so the batches differ slightly)."""
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    from oracle.ref import RefMesh
    pts, segs = host.generate_pslg(50_000, 5_000, "uniform", 21)
    closed = host.close_hull(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    with Engine(0) as eng:
        eng.build_cdt(pts, closed)
        v0 = eng.validate(q)
        assert v0["structure_failure"] == 0 and v0["cdt_violations"] == 0
        r_dev = eng.refine(q)
        v1 = eng.validate(q)
        out = eng.download()
        ref_mesh, _ = host.build_cdt(pts, segs)
        eng.upload(ref_mesh)
        r_host = eng.refine(q)
    assert v1["structure_failure"] == 0 and v1["cdt_violations"] == 0
    assert v1["bad_triangles"] == 0 and v1["conformity_failures"] == 0
    rm = RefMesh.from_mesh(out)
    rm.check_structure()
    assert rm.conformity_ok(pts, closed) and rm.count_bad(q) == 0
    assert abs(r_dev.steiner_points - r_host.steiner_points) <= 0.01 * r_host.steiner_points


def test_million_points_equals_reference(built):
    """BASELINE config 2 input (1M points, 100K segments): identical triangle set."""
    from paper_2007_00324_b200 import build_cdt, host
    pts, segs = host.generate_pslg(1_000_000, 100_000, "uniform", 20261017)
    closed = host.close_hull(pts, segs, check=False)
    dev, rep = build_cdt(pts, closed)
    ref, _ = host.build_cdt(pts, segs)
    np.testing.assert_array_equal(_tris(dev), _tris(ref))
    np.testing.assert_array_equal(_segs(dev), _segs(ref))
    from paper_2007_00324_b200 import Engine
    with Engine(0) as eng:   # warm context: device time of the build itself
        eng.build_cdt(pts, closed)
        assert eng.build_cdt(pts, closed)["seconds"] < 0.5


def test_cocircular_grid_is_a_valid_cdt(built):
    """A lattice is maximally cocircular: the CDT is not unique, so the device
    result is checked by the reference's validators (structure, local CDT with
    ties allowed, conformity) and by the triangle count every triangulation of
    the same points and hull shares."""
    from paper_2007_00324_b200 import build_cdt, host
    from oracle.ref import RefMesh
    k = 60
    g = np.linspace(0.0, 1.0, k)
    pts = np.array([(x, y) for y in g for x in g], np.float64)
    segs = np.array([[k * 10 + 10, k * 10 + 40], [k * 30 + 5, k * 50 + 5]], np.uint32)
    closed = host.close_hull(pts, segs)
    dev, rep = build_cdt(pts, closed)
    ref, _ = host.build_cdt(pts, segs)
    assert rep["n_triangles"] == int(ref.tri_alive.sum())
    assert rep["collinear_splits"] >= 2          # both segments pass through lattice points
    np.testing.assert_array_equal(_segs(dev), _segs(ref))
    rm = RefMesh.from_mesh(dev)
    rm.check_structure()
    assert rm.euler_holds() and rm.cdt_violations() == 0 and rm.conformity_ok(pts, closed)
