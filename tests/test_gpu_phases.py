"""Bit-exact parity of each hot-path phase on identical uploaded meshes:
collect + splitting points (refine.hpp:226-296), locate (:301-335), claim
(:367-376), cavity (:382-429) and the Lawson flip fixpoint (cdt.hpp:111-123)."""
import numpy as np
import pytest

from gdp2d_testlib import B_SQRT2_THETA, small_corpus, unit_square

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def meshes(built):
    from paper_2007_00324_b200 import host
    out = {}
    pts, segs = host.generate_pslg(20_000, 2_000, "uniform", 7)
    out["uniform-20k"] = host.build_cdt(pts, segs)
    pts, segs = host.generate_pslg(20_000, 2_000, "gaussian", 11)
    out["gauss-20k"] = host.build_cdt(pts, segs)
    for name, (p, s) in list(small_corpus().items())[:3]:
        out[name] = host.build_cdt(p, s)
    return out


def _same(a, b, what):
    assert a.dtype == b.dtype and len(a) == len(b), f"{what}: length {len(a)} vs {len(b)}"
    diff = np.nonzero(a.view(np.uint8).reshape(len(a), -1).any(axis=1) !=
                      b.view(np.uint8).reshape(len(b), -1).any(axis=1))[0]
    eq = (a.view(np.uint8).reshape(len(a), -1) == b.view(np.uint8).reshape(len(b), -1)).all(axis=1)
    bad = np.nonzero(~eq)[0]
    assert bad.size == 0, f"{what}: {bad.size} records differ; first gpu={a[bad[0]]} ref={b[bad[0]]}"


@pytest.mark.parametrize("theta", [B_SQRT2_THETA, 30.0])
def test_phases_bit_exact(meshes, theta):
    from paper_2007_00324_b200 import Engine, QualityCriteria
    from oracle.ref import RefMesh
    q = QualityCriteria(theta=theta)
    with Engine() as eng:
        for name, (m, _) in meshes.items():
            rm = RefMesh.from_mesh(m)
            eng.upload(m)
            g = eng.collect(q)
            r = rm.collect(q)
            _same(g, r, f"{name} collect")
            g = eng.locate(r)
            r = rm.locate(r)
            _same(g, r, f"{name} locate")
            g = eng.claim_filter(r)
            r = rm.claim_filter(r)
            _same(g, r, f"{name} claim")
            for n in (32, 4, 0):
                g = eng.cavity_filter(r, n)
                rr = rm.cavity_filter(r, n)
                _same(g, rr, f"{name} cavity n={n}")


def test_cavity_regions_match_oracle(meshes):
    from paper_2007_00324_b200 import Engine, QualityCriteria
    from oracle import ref
    q = QualityCriteria(theta=B_SQRT2_THETA)
    m, _ = meshes["uniform-20k"]
    rm = ref.RefMesh.from_mesh(m)
    c = rm.claim_filter(rm.locate(rm.collect(q)))
    with Engine() as eng:
        eng.upload(m)
        g, greg = eng.cavity_filter(c, 32, with_regions=True)
    o, oreg = ref.orc_cavity(m, c, 32, with_regions=True)
    assert np.array_equal(g["alive"], o["alive"])
    for i in range(len(c)):
        assert np.array_equal(greg[i], oreg[i]), i


def test_claim_exact_ties():
    """Identical priorities: the first claimer wins (refine.hpp:349-354, sequential)."""
    from paper_2007_00324_b200 import Engine, host
    from paper_2007_00324_b200 import _abi as A
    from oracle.ref import RefMesh
    pts, segs = unit_square()
    m, _ = host.build_cdt(pts, segs)
    c = np.zeros(3, dtype=A.candidate_dtype())
    c["located"] = [0, 0, 1]
    c["alive"] = 1
    c["kind"] = 1
    with Engine() as eng:
        eng.upload(m)
        g = eng.claim_filter(c)
    r = RefMesh.from_mesh(m).claim_filter(c)
    assert g["alive"].tolist() == r["alive"].tolist() == [1, 0, 1]


def test_flip_fixpoint_matches_reference(meshes):
    """Insert the cavity survivors with the reference's own split primitives,
    then run Lawson on both sides from the same seeds: identical CDT."""
    from paper_2007_00324_b200 import Engine, QualityCriteria
    from oracle.ref import RefMesh
    q = QualityCriteria(theta=B_SQRT2_THETA)
    for name in ("uniform-20k", "gauss-20k"):
        m, _ = meshes[name]
        rm = RefMesh.from_mesh(m)
        c = rm.cavity_filter(rm.claim_filter(rm.locate(rm.collect(q))))
        fresh = rm.split_only(c)
        assert len(fresh) > 100
        split_mesh = rm.to_mesh()
        tris, edges = [], []
        for v in fresh:
            for t in rm.incident(int(v)):
                for e in range(3):
                    tris.append(t)
                    edges.append(e)
        with Engine() as eng:
            eng.upload(split_mesh)
            flips = eng.lawson_fixpoint(tris, edges)
            out = eng.download()
        rm.lawson(tris, edges)
        a = np.unique(out.canonical_triangles(), axis=0)
        b = np.unique(rm.canonical_triangles(), axis=0)
        assert flips > 0
        assert a.shape == b.shape and np.array_equal(a, b), name
        RefMesh.from_mesh(out).check_structure()


def test_split_points_bit_exact(meshes):
    """gdp2d_split_points == compute_splitting_points (refine.hpp:267-296) on the
    reference's own candidate list with the points wiped."""
    from paper_2007_00324_b200 import Engine, QualityCriteria
    from oracle.ref import RefMesh
    q = QualityCriteria(theta=B_SQRT2_THETA)
    with Engine() as eng:
        for name, (m, _) in meshes.items():
            rm = RefMesh.from_mesh(m)
            eng.upload(m)
            c = rm.collect(q)
            c["x"] = 0.0
            c["y"] = 0.0
            _same(eng.split_points(c), rm.split_points(c), f"{name} split points")


@pytest.mark.parametrize("cap_frac", [0.0, 0.01, 0.33, 0.999])
def test_batch_size_cap_bit_exact(meshes, cap_frac):
    """batch_size_cap keeps the highest priorities in list order with the
    original tiebreaks (refine.hpp:252-261); device radix select vs the
    reference's sort."""
    from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria
    from oracle.ref import RefMesh
    q = QualityCriteria(theta=B_SQRT2_THETA)
    with Engine() as eng:
        for name, (m, _) in meshes.items():
            rm = RefMesh.from_mesh(m)
            eng.upload(m)
            full = rm.collect(q)
            cap = max(1, int(len(full) * cap_frac))
            cfg = EngineConfig(batch_size_cap=cap)
            g = eng.collect(q, cfg)
            r = rm.collect(q, cfg)
            assert len(r) == min(cap, len(full))
            _same(g, r, f"{name} collect cap={cap}")
