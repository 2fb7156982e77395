"""Full refinement on the GPU, invariant-checked against the reference's own
validators (mesh.hpp:505-557, verify.hpp:92-200) and its Steiner count."""
import math

import numpy as np
import pytest

from gdp2d_testlib import B_SQRT2_THETA, small_corpus, unit_square

pytestmark = pytest.mark.gpu


def batch_safety_holds(m):
    """test_refine.cpp:30-44: no edge joins two same-batch circumcenters."""
    t = m.tri_v[m.tri_alive.astype(bool)]
    for i in range(3):
        x, y = t[:, (i + 1) % 3], t[:, (i + 2) % 3]
        cc = (m.vert_kind[x] == 2) & (m.vert_kind[y] == 2)
        same = (m.vert_birth[x] == m.vert_birth[y]) & (m.vert_birth[x] > 0)
        if np.any(cc & same):
            return False
    return True


def check_invariants(out, pts, closed, q, cdt_check=True, strict_quality=True):
    from oracle.ref import RefMesh
    rm = RefMesh.from_mesh(out)
    rm.check_structure()
    assert rm.euler_holds()
    assert rm.conformity_ok(pts, closed)
    if strict_quality:
        assert rm.count_bad(q) == 0
    else:
        # the reference's own stopping criterion: nothing left to collect
        # (bad triangles below the precision floor are unresolvable, refine.hpp:169)
        assert len(rm.collect(q)) == 0
    if cdt_check:
        assert rm.cdt_violations() == 0
    assert batch_safety_holds(out)
    return rm


def _run(pts, segs, q, cfg=None):
    from paper_2007_00324_b200 import host, refine
    from oracle.ref import RefMesh
    m, closed = host.build_cdt(pts, segs)
    ref = RefMesh.from_mesh(m)
    gpu = m.copy()
    rep = refine(gpu, q, cfg)
    rref = ref.refine(q)
    return gpu, closed, rep, rref


def test_unit_square(built):
    from paper_2007_00324_b200 import QualityCriteria
    pts, segs = unit_square()
    for q in (QualityCriteria(20.0), QualityCriteria(20.0, 0.2), QualityCriteria(22.0, 0.3),
              QualityCriteria(30.0)):
        out, closed, rep, rref = _run(pts, segs, q)
        assert not rep.iteration_cap_hit
        assert rep.bad_triangles == 0 and rep.bad_area_percent == 0.0
        check_invariants(out, pts, closed, q)
        assert rep.steiner_points <= 1.3 * rref.steiner_points + 8


def test_already_quality_runs_zero_batches(built):
    from paper_2007_00324_b200 import QualityCriteria, refine
    pts, segs = unit_square()
    q = QualityCriteria(20.0)
    out, _, _, _ = _run(pts, segs, q)
    again = out.copy()
    r2 = refine(again, q)
    assert len(r2.batches) == 0
    assert again.alive_vertex_count() == out.alive_vertex_count()


def test_corpus(built):
    from paper_2007_00324_b200 import QualityCriteria
    q = QualityCriteria(20.0)
    for name, (pts, segs) in small_corpus().items():
        out, closed, rep, rref = _run(pts, segs, q)
        check_invariants(out, pts, closed, q)
        assert rep.steiner_points <= 1.10 * rref.steiner_points + 8, (name, rep.steiner_points,
                                                                     rref.steiner_points)


@pytest.mark.parametrize("insert_mode", [0, 1, 2])
@pytest.mark.parametrize("theta", [B_SQRT2_THETA, 30.0])
def test_uniform_50k(built, theta, insert_mode):
    from paper_2007_00324_b200 import EngineConfig, QualityCriteria, host
    q = QualityCriteria(theta)
    pts, segs = host.generate_pslg(50_000, 5_000, "uniform", 3)
    out, closed, rep, rref = _run(pts, segs, q, EngineConfig(insert_mode=insert_mode))
    check_invariants(out, pts, closed, q, cdt_check=True)
    assert abs(rep.steiner_points - rref.steiner_points) <= 0.10 * rref.steiner_points, \
        (rep.steiner_points, rref.steiner_points)
    assert rep.min_angle_deg >= theta - 1e-9


def test_gaussian_50k(built):
    from paper_2007_00324_b200 import QualityCriteria, host
    q = QualityCriteria(B_SQRT2_THETA)
    pts, segs = host.generate_pslg(50_000, 5_000, "gaussian", 5)
    out, closed, rep, rref = _run(pts, segs, q)
    check_invariants(out, pts, closed, q)
    assert abs(rep.steiner_points - rref.steiner_points) <= 0.10 * rref.steiner_points


def test_deterministic(built):
    from paper_2007_00324_b200 import QualityCriteria, host, refine
    pts, segs = host.generate_pslg(20_000, 2_000, "uniform", 9)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    a, b = m.copy(), m.copy()
    refine(a, q)
    refine(b, q)
    assert np.array_equal(a.xy[a.vert_alive.astype(bool)], b.xy[b.vert_alive.astype(bool)])
    assert np.array_equal(a.tri_v, b.tri_v)


def test_rule_ablations(built):
    from paper_2007_00324_b200 import EngineConfig, QualityCriteria, RuleFlags, host
    q = QualityCriteria(20.0)
    pts, segs = host.generate_pslg(10_000, 1_000, "uniform", 2)
    for rules in (RuleFlags(rule2_filtering_enabled=False), RuleFlags(rule4_unified_collection=False),
                  RuleFlags(rule1_compaction_threshold=0)):
        out, closed, rep, rref = _run(pts, segs, q, EngineConfig(rules=rules))
        check_invariants(out, pts, closed, q, strict_quality=False)


def test_chew_mode(built):
    from paper_2007_00324_b200 import CHEW, QualityCriteria
    pts, segs = unit_square()
    q = QualityCriteria(20.0, math.inf, CHEW)
    out, closed, rep, _ = _run(pts, segs, q)
    check_invariants(out, pts, closed, q)


def test_growth_paths_identical(built, monkeypatch):
    """Headroom 1.0 forces device-side INS_GROW + host growth + relaunch on
    almost every batch; the result must be bit-identical to the default run."""
    from paper_2007_00324_b200 import QualityCriteria, host, refine
    pts, segs = host.generate_pslg(30_000, 3_000, "uniform", 11)
    m, closed = host.build_cdt(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    a = m.copy()
    refine(a, q)
    monkeypatch.setenv("GDP2D_HEADROOM", "1.0")
    b = m.copy()
    rep = refine(b, q)
    assert rep.bad_triangles == 0
    for name in ("xy", "tri_v", "tri_n", "tri_seg", "tri_alive", "seg_v", "seg_alive"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    check_invariants(b, pts, closed, q, cdt_check=False)


def test_collect_round_trip_paths_identical(built, monkeypatch):
    """The candidate count stays on the device between collect and insertion;
    the synchronous path (GDP2D_SYNC_COLLECT=1) and the region-overflow redo
    (GDP2D_REGIONS_TIGHT=1 makes every no-round-trip batch overflow and redo)
    must give bit-identical meshes.  So must the small-list collect (append +
    one-CTA sort) switched off (GDP2D_SMALL_COLLECT=0) or forced onto every
    no-round-trip batch, big ones overflowing into the full-collect redo, and
    the device-resident tail loop switched off (GDP2D_TAIL_LOOP=0)."""
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    pts, segs = host.generate_pslg(40_000, 4_000, "gaussian", 13)
    m, closed = host.build_cdt(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    outs = []
    for env in ({}, {"GDP2D_SYNC_COLLECT": "1"}, {"GDP2D_REGIONS_TIGHT": "1"},
                {"GDP2D_SMALL_COLLECT": "0"}, {"GDP2D_SMALL_COLLECT": "1000000000"},
                {"GDP2D_TAIL_LOOP": "0"}):
        for k in ("GDP2D_SYNC_COLLECT", "GDP2D_REGIONS_TIGHT", "GDP2D_SMALL_COLLECT",
                  "GDP2D_TAIL_LOOP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with Engine(0) as eng:
            eng.upload(m)
            rep = eng.refine(q)
            outs.append((rep, eng.download()))
    base = outs[0][1]
    for rep, out in outs[1:]:
        assert rep.bad_triangles == 0 and len(rep.batches) == len(outs[0][0].batches)
        for name in ("xy", "tri_v", "tri_n", "tri_seg", "tri_alive", "seg_v", "seg_alive"):
            assert np.array_equal(getattr(base, name), getattr(out, name)), name


def test_pinned_round_trip(built):
    """Engine.upload from / download_to page-locked pools (the bench e2e path)."""
    from paper_2007_00324_b200 import Engine, PinnedPool, QualityCriteria, host
    pts, segs = host.generate_pslg(20_000, 2_000, "uniform", 12)
    m, closed = host.build_cdt(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    pin_in = PinnedPool(m.n_vertices, m.n_triangles, m.n_subsegments)
    pin_out = PinnedPool(3 * m.n_vertices, 3 * m.n_triangles, 3 * m.n_subsegments)
    src = pin_in.load(m)
    with Engine(0) as eng:
        eng.upload(src)
        rep = eng.refine(q)
        out = eng.download_to(pin_out)
        ref = eng.download()
    for name in ("xy", "tri_v", "tri_n", "seg_v", "vert_kind"):
        assert np.array_equal(getattr(out, name), getattr(ref, name)), name
    assert rep.bad_triangles == 0
    check_invariants(out, pts, closed, q, cdt_check=False)


@pytest.mark.parametrize("small_c", ["0", "100000000"])
def test_block_and_grid_modes_agree(built, monkeypatch, small_c):
    """Block mode (whole batch in one CTA) and grid mode give the same mesh."""
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    pts, segs = host.generate_pslg(10_000, 1_000, "gaussian", 13)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    with Engine(0) as eng:
        eng.upload(m)
        eng.refine(q)
        base = eng.download()
    monkeypatch.setenv("GDP2D_SMALL_C", small_c)
    with Engine(0) as eng:
        eng.upload(m)
        eng.refine(q)
        other = eng.download()
    assert np.array_equal(base.tri_v, other.tri_v)
    assert np.array_equal(base.xy, other.xy)


@pytest.mark.parametrize("cfgkw", [dict(batch_size_cap=500), dict(little_batch_sizing=True)])
def test_batch_sizing(built, cfgkw):
    """Capped batches (refine.hpp:252-261) and the Little's-law cap refine to
    quality with every batch at most the cap."""
    from paper_2007_00324_b200 import EngineConfig, QualityCriteria, host
    q = QualityCriteria(B_SQRT2_THETA)
    pts, segs = host.generate_pslg(20_000, 2_000, "uniform", 21)
    out, closed, rep, rref = _run(pts, segs, q, EngineConfig(**cfgkw))
    check_invariants(out, pts, closed, q, cdt_check=True)
    if "batch_size_cap" in cfgkw:
        assert max(b.attempted for b in rep.batches) <= cfgkw["batch_size_cap"]
    assert abs(rep.steiner_points - rref.steiner_points) <= 0.10 * rref.steiner_points


def test_edge_length_bound(built):
    """test_refine.cpp:392-401: quality + ell bound on every triangle."""
    from paper_2007_00324_b200 import QualityCriteria
    pts, segs = unit_square()
    q = QualityCriteria(20.0, 0.2)
    out, closed, rep, _ = _run(pts, segs, q)
    assert rep.bad_triangles == 0 and rep.max_edge <= 0.2
    check_invariants(out, pts, closed, q)


def test_small_input_angle_stays_local(built):
    """test_refine.cpp:403-425: a 10-degree wedge; any triangle left bad hugs the
    small-angle apex, and the mesh is a conforming CDT."""
    from paper_2007_00324_b200 import QualityCriteria
    from oracle.ref import RefMesh
    r = math.radians(10.0)
    pts = np.array([[0, 0], [4, 0], [4 * math.cos(r), 4 * math.sin(r)], [4, 4], [0, 4]], float)
    segs = np.array([[0, 1], [0, 2], [1, 3], [3, 4], [4, 0]], np.uint32)
    q = QualityCriteria(20.0, 1e9)
    out, closed, rep, _ = _run(pts, segs, q)
    rm = RefMesh.from_mesh(out)
    rm.check_structure()
    assert rm.conformity_ok(pts, closed)
    assert rm.cdt_violations() == 0
    # bad triangles (if any) near the apex only
    alive = out.tri_alive.astype(bool)
    t = out.tri_v[alive]
    xy = out.xy
    a, b, c = xy[t[:, 0]], xy[t[:, 1]], xy[t[:, 2]]

    def ang(p, u, v):
        e1, e2 = u - p, v - p
        return np.degrees(np.arctan2(np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]),
                                     (e1 * e2).sum(1)))
    mins = np.minimum(np.minimum(ang(a, b, c), ang(b, c, a)), ang(c, a, b))
    bad = mins < 20.0 - 1e-9
    if bad.any():
        far = np.linalg.norm(np.concatenate([a[bad], b[bad], c[bad]]), axis=1)
        assert far.max() < 0.1


def test_iteration_cap_and_batch_prefixes(built):
    """refine.hpp:659-662 (iteration_cap_hit) and acceptance C3: after every
    batch prefix the mesh is a valid conforming CDT."""
    from paper_2007_00324_b200 import EngineConfig, QualityCriteria, host
    from oracle.ref import RefMesh
    pts, segs = host.generate_pslg(5_000, 500, "uniform", 31)
    q = QualityCriteria(B_SQRT2_THETA)
    for k in (0, 1, 2, 5):
        out, closed, rep, _ = _run(pts, segs, q, EngineConfig(iteration_cap=k))
        assert rep.iteration_cap_hit and len(rep.batches) == k
        rm = RefMesh.from_mesh(out)
        rm.check_structure()
        assert rm.euler_holds() and rm.conformity_ok(pts, closed)
        assert rm.cdt_violations() == 0


def test_quality_report_fractions(built):
    """test_refine.cpp:454-489 analogues through the GPU quality summary
    (refine.hpp:614-645), reached with iteration_cap = 0."""
    from paper_2007_00324_b200 import EngineConfig, QualityCriteria, host, refine
    s = math.sqrt(3.0) / 2.0
    m, _ = host.build_cdt(np.array([[0, 0], [1, 0], [0.5, s]], float),
                          np.array([[0, 1], [1, 2], [2, 0]], np.uint32))
    rep = refine(m.copy(), QualityCriteria(20.0, 1e9), EngineConfig(iteration_cap=0))
    assert rep.bad_triangles == 0 and rep.bad_area_percent == 0.0
    rep = refine(m.copy(), QualityCriteria(20.0, 0.9), EngineConfig(iteration_cap=0))
    assert rep.bad_triangles == 1 and rep.bad_area_percent == 100.0
    m, _ = host.build_cdt(np.array([[0, 0], [10, 0], [5, 0.01]], float),
                          np.array([[0, 1], [1, 2], [2, 0]], np.uint32))
    rep = refine(m.copy(), QualityCriteria(0.0, math.inf), EngineConfig(iteration_cap=0))
    assert rep.bad_triangles == 0 and rep.bad_area_percent == 0.0


@pytest.mark.parametrize("mode,ell", [(1, math.inf), (0, 0.01), (1, 0.01)])
def test_chew_and_edge_bound_at_scale(built, mode, ell):
    """Chew's lens rule (predicates.hpp:126-162) and the
    edge-length bound (refine.hpp:192-206) on a 50K-point PSLG: quality,
    conforming CDT (device validators + reference validators) and Steiner
    count within 10% of the reference."""
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    from oracle.ref import RefMesh
    q = QualityCriteria(B_SQRT2_THETA, ell, mode)
    pts, segs = host.generate_pslg(50_000, 5_000, "uniform", 51)
    m, closed = host.build_cdt(pts, segs)
    with Engine(0) as eng:
        eng.upload(m)
        rep = eng.refine(q)
        val = eng.validate(q)
        out = eng.download()
    rref = RefMesh.from_mesh(m).refine(q)
    assert val["structure_failure"] == 0 and val["cdt_violations"] == 0
    assert val["conformity_failures"] == 0 and val["bad_triangles"] == 0
    rm = RefMesh.from_mesh(out)
    assert rm.conformity_ok(pts, closed) and len(rm.collect(q)) == 0
    if math.isfinite(ell):
        assert rep.max_edge <= ell
    assert abs(rep.steiner_points - rref.steiner_points) <= 0.10 * rref.steiner_points, \
        (rep.steiner_points, rref.steiner_points)


@pytest.mark.parametrize("mode,ell", [(1, math.inf), (1, 0.002)])
def test_chew_and_edge_bound_at_million_points(built, mode, ell):
    """SURVEY 8(f) row 3 at BASELINE size: Lines 1-9 on the device (device CDT,
    Chew lens rule, edge-length bound) on config 2's 1M-point PSLG, checked by
    the device validators (structure, exact local CDT, quality, conformity)."""
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    q = QualityCriteria(B_SQRT2_THETA, ell, mode)
    pts, segs = host.generate_pslg(1_000_000, 100_000, "uniform", 20261017)
    closed = host.close_hull(pts, segs, check=False)
    with Engine(0) as eng:
        eng.build_cdt(pts, closed)
        rep = eng.refine(q)
        val = eng.validate(q)
    assert val["structure_failure"] == 0 and val["cdt_violations"] == 0
    assert val["conformity_failures"] == 0 and val["bad_triangles"] == 0
    assert rep.bad_triangles == 0 and rep.steiner_points > 500_000
    assert val["min_angle_deg"] >= B_SQRT2_THETA - 1e-9 or mode == 1
    if math.isfinite(ell):
        assert rep.max_edge <= ell


def test_warmup_then_one_shot_refine(built):
    """gdp2d_warmup prepares the cached context (tiny build + refinement); a
    one-shot refine afterwards gives the same result as without it."""
    from paper_2007_00324_b200 import QualityCriteria, host
    from paper_2007_00324_b200.gdp2d import refine, warmup
    pts, segs = host.generate_pslg(20_000, 2_000, "uniform", 5)
    m0, _ = host.build_cdt(pts, segs)
    a = m0.copy()
    ra = refine(a, QualityCriteria(30.0))
    warmup(0)
    b = m0.copy()
    rb = refine(b, QualityCriteria(30.0))
    assert ra.steiner_points == rb.steiner_points and rb.bad_triangles == 0
    np.testing.assert_array_equal(a.tri_v, b.tri_v)
    with pytest.raises(Exception):
        warmup(999)


@pytest.mark.parametrize("n_sides", [97, 128, 400])
def test_high_degree_ngon(built, n_sides):
    """A disc bounded by a regular N-gon with no interior points: after batch 1
    the inserted centre has degree N, and every fan triangle has a subsegment
    opposite it, so redundancy detection walks a star of N triangles
    (walk_star capped stars at MAX_STAR = 96 and failed the
    refine).  The reference finishes this input; so must the device."""
    from gdp2d_testlib import regular_polygon
    from paper_2007_00324_b200 import QualityCriteria
    b = np.array(regular_polygon(n_sides, 1.0), np.float64)
    segs = np.array([(i, (i + 1) % n_sides) for i in range(n_sides)], np.uint32)
    q = QualityCriteria(B_SQRT2_THETA)
    out, closed, rep, rref = _run(b, segs, q)
    assert not rep.iteration_cap_hit
    check_invariants(out, b, closed, q)
    assert rep.bad_triangles == 0
    assert abs(rep.steiner_points - rref.steiner_points) <= 0.10 * rref.steiner_points + 8, \
        (rep.steiner_points, rref.steiner_points)


@pytest.mark.parametrize("insert_mode", [0, 1, 2])
@pytest.mark.parametrize("theta", [B_SQRT2_THETA, 30.0])
def test_tail_loop_identical(built, monkeypatch, insert_mode, theta):
    """The device-resident tail loop (k_tail_loop: incremental collect from the
    last list + the dirty elements, the block-mode batch, no host round trip)
    gives the very mesh the per-batch host loop gives (GDP2D_TAIL_LOOP=0), in
    every insertion policy."""
    from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host
    pts, segs = host.generate_pslg(100_000, 10_000, "gaussian", 31)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(theta)
    outs = []
    for env in ({}, {"GDP2D_TAIL_LOOP": "0"}):
        monkeypatch.delenv("GDP2D_TAIL_LOOP", raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with Engine(0) as eng:
            eng.upload(m)
            rep = eng.refine(q, EngineConfig(insert_mode=insert_mode))
            v = eng.validate(q)
            assert v["bad_triangles"] == 0 and v["cdt_violations"] == 0, v
            outs.append((rep, eng.download()))
    (r0, a), (r1, b) = outs
    assert len(r0.batches) == len(r1.batches) and r0.steiner_points == r1.steiner_points
    for name in ("xy", "tri_v", "tri_n", "tri_seg", "tri_alive", "seg_v", "seg_alive",
                 "vert_tri", "seg_tri"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("insert_mode", [1, 2])
def test_warp_removal_identical(built, monkeypatch, insert_mode):
    """Removal rounds with one warp per removal (lanes test the ears from head
    in parallel, GDP2D_RM_WARP) clip the same ears in the same order as one
    thread per removal: the refined mesh is identical whether no round
    (GDP2D_RM_WARP=0), the default few-removal rounds, or every round runs in
    warp mode."""
    from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host
    pts, segs = host.generate_pslg(100_000, 10_000, "gaussian", 37)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(B_SQRT2_THETA)
    outs = []
    for val in ("0", None, "1000000"):
        monkeypatch.delenv("GDP2D_RM_WARP", raising=False)
        if val is not None:
            monkeypatch.setenv("GDP2D_RM_WARP", val)
        with Engine(0) as eng:
            eng.upload(m)
            rep = eng.refine(q, EngineConfig(insert_mode=insert_mode))
            v = eng.validate(q)
            assert v["bad_triangles"] == 0 and v["cdt_violations"] == 0, v
            assert rep.totals["total_removed"] > 0
            outs.append((rep, eng.download()))
    (r0, a) = outs[0]
    for r1, b in outs[1:]:
        assert len(r0.batches) == len(r1.batches) and r0.steiner_points == r1.steiner_points
        for name in ("xy", "tri_v", "tri_n", "tri_seg", "tri_alive", "seg_v", "seg_alive",
                     "vert_tri", "seg_tri"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("insert_mode", [0, 1])
@pytest.mark.parametrize("theta", [B_SQRT2_THETA, 30.0])
def test_cluster_mode_identical(built, monkeypatch, insert_mode, theta):
    """Batches run as ONE thread-block cluster (barrier.cluster instead of grid
    barriers, GDP2D_CLUSTER_C) give the very mesh the cooperative grid gives:
    cluster mode off, the default mid-size band, and every batch that does not
    run in block mode forced into a cluster (16 or 8 CTAs)."""
    from paper_2007_00324_b200 import Engine, EngineConfig, QualityCriteria, host
    pts, segs = host.generate_pslg(100_000, 10_000, "gaussian", 41)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(theta)
    outs = []
    for env in ({"GDP2D_CLUSTER_C": "0"}, {}, {"GDP2D_CLUSTER_C": "1000000000"},
                {"GDP2D_CLUSTER_C": "1000000000", "GDP2D_CLUSTER": "8"}):
        for k in ("GDP2D_CLUSTER_C", "GDP2D_CLUSTER"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        with Engine(0) as eng:
            eng.upload(m)
            rep = eng.refine(q, EngineConfig(insert_mode=insert_mode))
            v = eng.validate(q)
            assert v["bad_triangles"] == 0 and v["cdt_violations"] == 0, v
            outs.append((rep, eng.download()))
    (r0, a) = outs[0]
    for r1, b in outs[1:]:
        assert len(r0.batches) == len(r1.batches) and r0.steiner_points == r1.steiner_points
        for name in ("xy", "tri_v", "tri_n", "tri_seg", "tri_alive", "seg_v", "seg_alive",
                     "vert_tri", "seg_tri"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("theta", [B_SQRT2_THETA, 23.5])
def test_dropin_shim_matches_context_path(built, theta):
    """gdp2d::refine on the reference's own AoS Mesh (include/gdp2d_cdtref.hpp:
    the element vectors go to gdp2d_refine_aos as they are, the records are
    converted on the device and the result is written back into the vectors)
    gives the mesh the SoA context path gives, array for array.  At 23.5 deg
    the output outgrows the shim's size hint (2.2x), so the resize callback's
    reallocating branch runs too."""
    from paper_2007_00324_b200 import Engine, QualityCriteria, host
    from paper_2007_00324_b200.gdp2d import _FIELDS
    pts, segs = host.generate_pslg(60_000, 6_000, "gaussian", 41)
    m, _ = host.build_cdt(pts, segs)
    q = QualityCriteria(theta)
    with Engine(0) as eng:
        eng.upload(m)
        rep = eng.refine(q)
        ref = eng.download()
    got, steiner = host.dropin_refine(m, theta)
    assert steiner == rep.steiner_points
    if theta > 23.0:
        assert got.n_triangles > 2.2 * m.n_triangles
    assert got.batch_epoch == ref.batch_epoch
    for name, _, _ in _FIELDS:
        assert np.array_equal(getattr(got, name), getattr(ref, name)), name
