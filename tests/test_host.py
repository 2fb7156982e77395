"""Host side (reference I/O + generator) and the CPU oracle restatement,
checked against the compiled reference (no GPU needed)."""
import numpy as np
import pytest

from gdp2d_testlib import B_SQRT2_THETA, small_corpus, unit_square


def test_generator_deterministic_and_valid(built):
    from paper_2007_00324_b200 import host
    a = host.generate_pslg(20_000, 2_000, "uniform", 5)
    b = host.generate_pslg(20_000, 2_000, "uniform", 5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    pts, segs = a
    assert pts.shape == (20_000, 2) and len(segs) > 1500
    assert ((pts >= 0) & (pts <= 1)).all()
    assert len(np.unique(pts, axis=0)) == len(pts)
    used = segs.ravel()
    assert len(np.unique(used)) == len(used), "segments must be vertex-disjoint"
    g = host.generate_pslg(20_000, 2_000, "gaussian", 5)[0]
    assert len(np.unique(g, axis=0)) == len(g)


def test_build_cdt_is_valid_cdt(built):
    from paper_2007_00324_b200 import host
    from oracle.ref import RefMesh
    pts, segs = host.generate_pslg(5_000, 500, "uniform", 1)
    m, closed = host.build_cdt(pts, segs)
    assert len(closed) == len(segs) + 4   # close_hull adds the square
    rm = RefMesh.from_mesh(m)
    rm.check_structure()
    assert rm.euler_holds()
    assert rm.cdt_violations() == 0
    assert rm.conformity_ok(pts, closed)


def test_poly_roundtrip(built):
    from paper_2007_00324_b200 import host
    text = "4 2 0 0\n0 0 0\n1 1 0\n2 1 1\n3 0 1\n4 0\n0 0 1\n1 1 2\n2 2 3\n3 3 0\n0\n"
    pts, segs = host.read_poly(text)
    assert pts.shape == (4, 2) and len(segs) == 4
    m, closed = host.build_cdt(pts, segs, close_hull=False)
    node, ele = host.write_node_ele(m)
    assert node.splitlines()[0].split()[0] == "4"
    assert ele.splitlines()[0].split()[0] == "2"
    with pytest.raises(ValueError):
        host.read_poly("4 2 0 0\n0 0 0\n1 1 0\n2 1 1\n3 1 1\n0 0\n0\n")  # duplicate point


def test_reference_refine_small(built):
    """The checker itself: the reference refines the unit square to quality."""
    from paper_2007_00324_b200 import QualityCriteria, host
    from oracle.ref import RefMesh
    pts, segs = unit_square()
    m, closed = host.build_cdt(pts, segs)
    rm = RefMesh.from_mesh(m)
    rep = rm.refine(QualityCriteria(20.0, 0.2))
    rm.check_structure()
    assert rep.bad_triangles == 0 and rep.max_edge <= 0.2
    assert rm.cdt_violations() == 0


def test_close_hull_matches_build_cdt_segments():
    """host.close_hull (the device CDT builder's input) returns exactly the
    segment list the reference's build path closes (cdt.hpp:447)."""
    import numpy as np
    from paper_2007_00324_b200 import host
    pts, segs = host.generate_pslg(3000, 300, "gaussian", 2)
    closed = host.close_hull(pts, segs)
    _, closed_ref = host.build_cdt(pts, segs)
    np.testing.assert_array_equal(closed, closed_ref)
    assert len(closed) > len(segs)


def test_parallel_node_ele_formatting_is_byte_identical(monkeypatch):
    """format_node_ele renders blocks of lines on several threads and joins
    them in order: the text must not depend on the thread count."""
    import numpy as np
    from paper_2007_00324_b200 import host
    rng = np.random.default_rng(3)
    n, m = 50_000, 90_000
    xy = rng.uniform(-1e3, 1e3, size=(n, 2))
    xy[::7] = np.round(xy[::7], 2)
    marker = (rng.random(n) < 0.1).astype(np.uint8)
    tri = rng.integers(0, n, size=(m, 3)).astype(np.uint32)
    monkeypatch.setenv("GDP2D_IO_THREADS", "1")
    a = host.format_node_ele(xy, marker, tri)
    monkeypatch.setenv("GDP2D_IO_THREADS", "7")
    b = host.format_node_ele(xy, marker, tri)
    assert a == b
    node, ele = a
    assert node.startswith(f"{n} 2 0 1\n") and ele.startswith(f"{m} 3 0\n")
    assert node.count("\n") == n + 1 and ele.count("\n") == m + 1
