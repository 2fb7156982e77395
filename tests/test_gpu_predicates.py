"""GPU predicates vs the reference, bit for bit (predicates.hpp:63-185,
refine.hpp:192).  Inputs follow test_predicates.cpp's generators."""
import numpy as np
import pytest

from gdp2d_testlib import B_SQRT2_THETA
import gdp2d_cases as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def libs(built):
    from paper_2007_00324_b200 import gdp2d
    from oracle import ref
    return gdp2d, ref


def _cmp(libs, kind, pts, q=None):
    gdp2d, ref = libs
    g = gdp2d.predicates(kind, pts, q)
    r = ref.ref_predicates(kind, pts, q)
    bad = np.nonzero(g != r)[0]
    assert bad.size == 0, f"kind {kind}: {bad.size} mismatches, first {pts[bad[0]].tolist()}"
    return g


def test_orient2d_known_answers(libs):
    # test_predicates.cpp:52-56
    pts = np.array([[[0, 0], [1, 0], [0, 1]], [[0, 0], [1, 1], [2, 2]], [[0, 0], [0, 1], [1, 0]]],
                   dtype=np.float64)
    assert _cmp(libs, 0, pts).tolist() == [1, 0, -1]


def test_incircle_known_answers(libs):
    # test_predicates.cpp:58-63
    a, b, c = [1, 0], [0, 1], [-1, 0]
    pts = np.array([[a, b, c, [0, 0]], [a, b, c, [0, -1]], [a, b, c, [0, -2]]], dtype=np.float64)
    assert _cmp(libs, 1, pts).tolist() == [1, 0, -1]


def test_orient2d_near_collinear(libs):
    pts = G.near_collinear(100_000)
    s = _cmp(libs, 0, pts)
    assert (s == 0).sum() > 0 and (s != 0).sum() > 0


def test_orient2d_random_and_grid(libs):
    _cmp(libs, 0, G.random_points(50_000, 3))
    _cmp(libs, 0, G.grid_degenerate(50_000, 3))


def test_incircle_near_cocircular(libs):
    _cmp(libs, 1, G.near_cocircular(20_000))


def test_incircle_random_and_grid(libs):
    _cmp(libs, 1, G.random_points(50_000, 4))
    _cmp(libs, 1, G.grid_degenerate(50_000, 4))


def test_diametric_and_lens(libs):
    # test_predicates.cpp:126-140 known answers, then boundary cases
    sa, sb = [0, 0], [2, 0]
    pts = np.array([[sa, sb, [1, 0.5]], [sa, sb, [3, 0]], [sa, sb, [0, 0]], [sa, sb, [1, 1]],
                    [sa, sb, [1, 0.99]]], dtype=np.float64)
    assert _cmp(libs, 2, pts).tolist() == [1, 0, 0, 0, 1]
    assert _cmp(libs, 3, pts).tolist() == [1, 0, 0, 0, 0]
    cases = G.diametric_cases(50_000)
    _cmp(libs, 2, cases)
    _cmp(libs, 3, cases)
    _cmp(libs, 2, G.grid_degenerate(20_000, 3))
    _cmp(libs, 3, G.grid_degenerate(20_000, 3))


def test_is_bad_triangle(libs):
    from paper_2007_00324_b200 import QualityCriteria
    for theta in (20.0, B_SQRT2_THETA, 30.0):
        _cmp(libs, 4, G.triangles_near_bound(theta, 20_000), QualityCriteria(theta=theta))
    _cmp(libs, 4, G.random_points(20_000, 3, 0, 1), QualityCriteria(theta=20.0, ell=0.3))


def test_circumcenter_bits(libs):
    gdp2d, ref = libs
    pts = np.concatenate([G.random_points(50_000, 3), G.near_collinear(10_000)])
    g, gok = gdp2d.circumcenters(pts)
    r, rok = ref.ref_circumcenters(pts)
    assert np.array_equal(gok, rok)
    ok = rok.astype(bool)
    assert np.array_equal(g[ok].view(np.uint64), r[ok].view(np.uint64))


def test_mesh_scale_near_degenerate(libs):
    pts4 = G.mesh_scale_cocircular(200_000)
    _cmp(libs, 1, pts4)
    _cmp(libs, 0, pts4[:, :3])
    _cmp(libs, 0, G.mesh_scale_collinear(200_000))
