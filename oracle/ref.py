"""TEST INFRASTRUCTURE ONLY -- Python handle on the checkers.

  RefMesh / ref_*  : the UNMODIFIED reference (cdtref headers from
                     /root/reference/proj/include) compiled into
                     oracle/_ref/libcdtref_ref.so by oracle/Makefile
  orc_*            : the plain-C restatement oracle/cdt_oracle.c
                     (oracle/_ref/libgdp2d_oracle.so)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.  Neither library ever runs on
the product path.
"""
from __future__ import annotations

import ctypes as C
import math
from pathlib import Path

import numpy as np

from paper_2007_00324_b200 import _abi as A
from paper_2007_00324_b200.gdp2d import Mesh, QualityCriteria, EngineConfig, RunReport, \
    BatchMetrics

REF_DIR = Path(__file__).resolve().parent / "_ref"
_ref = None
_orc = None

mp = C.c_void_p


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        path = REF_DIR / "libcdtref_ref.so"
        if not path.exists():
            raise RuntimeError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        lib = C.CDLL(str(path))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_mesh_free": (None, [mp]),
            "ref_mesh_clone": (mp, [mp]),
            "ref_mesh_from_view": (mp, [C.POINTER(A.MeshView)]),
            "ref_mesh_to_buf": (None, [mp, C.POINTER(A.MeshBuf)]),
            "ref_buf_free": (None, [C.POINTER(A.MeshBuf)]),
            "ref_close_hull": (C.c_uint32, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                            C.c_void_p]),
            "ref_build_cdt": (mp, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]),
            "ref_build_delaunay": (mp, [C.c_void_p, C.c_uint32]),
            "ref_mesh_sizes": (None, [mp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                      C.POINTER(C.c_uint32)]),
            "ref_refine": (C.c_int, [mp, C.POINTER(A.Params), C.POINTER(A.Report), C.c_uint]),
            "ref_refine_sequential": (C.c_int, [mp, C.POINTER(A.Params), C.POINTER(A.Report)]),
            "ref_quality": (None, [mp, C.POINTER(A.Params), C.POINTER(A.Report)]),
            "ref_collect": (C.c_int, [mp, C.POINTER(A.Params), C.c_void_p, C.c_uint32,
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
            "ref_split_points": (C.c_int, [mp, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32)]),
            "ref_locate": (C.c_int, [mp, C.c_void_p, C.c_uint32]),
            "ref_claim": (C.c_int, [mp, C.c_void_p, C.c_uint32]),
            "ref_cavity": (C.c_int, [mp, C.c_void_p, C.c_uint32, C.c_uint32]),
            "ref_insert_batch": (C.c_int, [mp, C.c_void_p, C.c_uint32, C.POINTER(A.Params),
                                           C.POINTER(C.c_uint64)]),
            "ref_split_only": (C.c_int, [mp, C.c_void_p, C.c_uint32, C.c_void_p,
                                         C.POINTER(C.c_uint32)]),
            "ref_incident": (C.c_uint32, [mp, C.c_uint32, C.c_void_p, C.c_uint32]),
            "ref_lawson": (C.c_int, [mp, C.c_void_p, C.c_void_p, C.c_uint32]),
            "ref_check_structure": (C.c_int, [mp]),
            "ref_euler_holds": (C.c_int, [mp]),
            "ref_conformity_ok": (C.c_int, [mp, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]),
            "ref_cdt_violations": (C.c_uint64, [mp, C.c_uint64]),
            "ref_delaunay_violations": (C.c_uint64, [mp, C.c_uint64]),
            "ref_count_bad": (C.c_uint64, [mp, C.POINTER(A.Params)]),
            "ref_canonical_triangles": (C.c_uint32, [mp, C.c_void_p]),
            "ref_predicates_batch": (None, [C.c_int, C.c_void_p, C.c_uint32, C.POINTER(A.Params),
                                            C.c_void_p]),
            "ref_circumcenter_batch": (None, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
            "ref_min_angle_hist": (C.c_uint64, [mp, C.c_double, C.c_uint32, C.c_void_p,
                                                C.POINTER(C.c_double)]),
            "gdp2d_host_generate": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int, C.c_uint64,
                                               C.POINTER(C.POINTER(C.c_double)),
                                               C.POINTER(C.POINTER(C.c_uint32)),
                                               C.POINTER(C.c_uint32)]),
            "gdp2d_host_free": (None, [C.c_void_p]),
        }
        for k, (res, args) in sig.items():
            f = getattr(lib, k)
            f.restype = res
            f.argtypes = args
        _ref = lib
    return _ref


def orc_lib() -> C.CDLL:
    global _orc
    if _orc is None:
        path = REF_DIR / "libgdp2d_oracle.so"
        if not path.exists():
            raise RuntimeError(f"{path} missing: run `make -C oracle oracle-only`")
        lib = C.CDLL(str(path))
        vp = C.c_void_p
        sig = {
            "orc_predicates_batch": (None, [C.c_int, vp, C.c_uint32, C.POINTER(A.Params), vp]),
            "orc_circumcenter": (C.c_int, [vp, vp, vp, vp]),
            "orc_collect": (C.c_uint32, [C.POINTER(A.MeshView), C.POINTER(A.Params), vp,
                                         C.c_uint32]),
            "orc_locate": (None, [C.POINTER(A.MeshView), vp, C.c_uint32]),
            "orc_claim": (None, [C.POINTER(A.MeshView), vp, C.c_uint32]),
            "orc_cavity": (None, [C.POINTER(A.MeshView), vp, C.c_uint32, C.c_uint32, vp, vp]),
        }
        for k, (res, args) in sig.items():
            f = getattr(lib, k)
            f.restype = res
            f.argtypes = args
        _orc = lib
    return _orc


def params(q: QualityCriteria, cfg: EngineConfig | None = None) -> A.Params:
    """gdp2d_params equivalent built WITHOUT the CUDA engine (CPU-only tests)."""
    cfg = cfg or EngineConfig()
    p = A.Params()
    p.theta_deg = q.theta
    c = math.cos(q.theta * 3.14159265358979323846 / 180.0)
    p.cos2_theta = c * c
    p.ell = q.ell
    p.mode = q.mode
    p.cavity_n = cfg.cavity_n
    p.rule1_compaction_threshold = cfg.rules.rule1_compaction_threshold
    p.rule2_filtering_enabled = int(cfg.rules.rule2_filtering_enabled)
    p.rule4_unified_collection = int(cfg.rules.rule4_unified_collection)
    p.little_batch_sizing = 0
    p.iteration_cap = cfg.iteration_cap
    p.split_depth_cap = cfg.split_depth_cap
    p.batch_size_cap = cfg.batch_size_cap
    return p


HIST_BIN_DEG = 0.5   # min-angle histogram: 120 bins of 0.5 degrees over [0, 60]
HIST_BINS = 120


def ref_generate_pslg(n: int, m: int, dist: str = "uniform", seed: int = 20261017):
    """The SURVEY 8(d) generator (pslg_gen.cpp) as compiled into the oracle
    library: (points (n,2) f64, segments (m',2) u32), hull not yet closed.
    Bit-identical to paper_2007_00324_b200.host.generate_pslg (same source)."""
    lib = ref_lib()
    xy = C.POINTER(C.c_double)()
    segs = C.POINTER(C.c_uint32)()
    mout = C.c_uint32(0)
    if lib.gdp2d_host_generate(n, m, 1 if dist == "gaussian" else 0, seed, C.byref(xy),
                               C.byref(segs), C.byref(mout)):
        raise RuntimeError("generator failed")
    pts = np.ctypeslib.as_array(xy, shape=(2 * n,)).reshape(n, 2).copy()
    s = (np.ctypeslib.as_array(segs, shape=(2 * mout.value,)).reshape(-1, 2).copy()
         if mout.value else np.zeros((0, 2), np.uint32))
    lib.gdp2d_host_free(C.cast(xy, C.c_void_p))
    lib.gdp2d_host_free(C.cast(segs, C.c_void_p))
    return pts, s


def ref_close_hull(pts, segs) -> np.ndarray:
    """close_hull (cdt.hpp:447) through the reference library."""
    pts = np.ascontiguousarray(pts, np.float64)
    segs = np.ascontiguousarray(segs, np.uint32).reshape(-1, 2)
    out = np.zeros((len(segs) + len(pts), 2), np.uint32)
    k = ref_lib().ref_close_hull(pts.ctypes.data, len(pts), segs.ctypes.data, len(segs),
                                 out.ctypes.data)
    return out[:k].copy()


def ref_workload(n: int, m: int, dist: str, seed: int):
    """Generator + close_hull + build_cdt entirely inside oracle/_ref:
    (points, closed segments, RefMesh of the initial CDT)."""
    pts, segs = ref_generate_pslg(n, m, dist, seed)
    closed = ref_close_hull(pts, segs)
    return pts, closed, RefMesh.build_cdt(pts, closed)


def _err() -> str:
    return ref_lib().ref_last_error().decode(errors="replace")


class RefMesh:
    """A cdtref::Mesh owned by the reference library."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference: " + _err())
        self.h = C.c_void_p(handle)

    def __del__(self):
        try:
            if self.h:
                ref_lib().ref_mesh_free(self.h)
        except Exception:
            pass

    @classmethod
    def from_mesh(cls, m: Mesh) -> "RefMesh":
        v = m.view()
        return cls(ref_lib().ref_mesh_from_view(C.byref(v)))

    @classmethod
    def build_cdt(cls, pts, segs) -> "RefMesh":
        pts = np.ascontiguousarray(pts, np.float64)
        segs = np.ascontiguousarray(segs, np.uint32).reshape(-1, 2)
        return cls(ref_lib().ref_build_cdt(pts.ctypes.data, len(pts), segs.ctypes.data, len(segs)))

    @classmethod
    def build_delaunay(cls, pts) -> "RefMesh":
        pts = np.ascontiguousarray(pts, np.float64)
        return cls(ref_lib().ref_build_delaunay(pts.ctypes.data, len(pts)))

    def clone(self) -> "RefMesh":
        return RefMesh(ref_lib().ref_mesh_clone(self.h))

    def to_mesh(self) -> Mesh:
        b = A.MeshBuf()
        ref_lib().ref_mesh_to_buf(self.h, C.byref(b))
        return Mesh.from_buf(b, ref_lib().ref_buf_free)

    def sizes(self):
        v, t, s = C.c_uint32(), C.c_uint32(), C.c_uint32()
        ref_lib().ref_mesh_sizes(self.h, C.byref(v), C.byref(t), C.byref(s))
        return v.value, t.value, s.value

    # -- refinement --
    def refine(self, q: QualityCriteria, cfg: EngineConfig | None = None,
               executors: int = 1) -> RunReport:
        p = params(q, cfg)
        arr = (A.BatchMetrics * 20000)()
        r = A.Report()
        r.batches = C.cast(arr, C.POINTER(A.BatchMetrics))
        r.batches_capacity = 20000
        rc = ref_lib().ref_refine(self.h, C.byref(p), C.byref(r), executors)
        if rc:
            raise RuntimeError("reference refine: " + _err())
        return _report(r, arr)

    def refine_sequential(self, q: QualityCriteria) -> RunReport:
        p = params(q)
        r = A.Report()
        if ref_lib().ref_refine_sequential(self.h, C.byref(p), C.byref(r)):
            raise RuntimeError(_err())
        return _report(r, None)

    def quality(self, q: QualityCriteria) -> RunReport:
        p = params(q)
        r = A.Report()
        ref_lib().ref_quality(self.h, C.byref(p), C.byref(r))
        return _report(r, None)

    # -- phases --
    def collect(self, q: QualityCriteria, cfg: EngineConfig | None = None) -> np.ndarray:
        p = params(q, cfg)
        n, fb = C.c_uint32(), C.c_uint32()
        cap = 1 << 16
        while True:
            out = np.zeros(cap, dtype=A.candidate_dtype())
            rc = ref_lib().ref_collect(self.h, C.byref(p), out.ctypes.data, cap, C.byref(n),
                                       C.byref(fb))
            if rc == 2:
                cap = n.value
                continue
            if rc:
                raise RuntimeError(_err())
            return out[: n.value].copy()

    def _inplace(self, fn, cands, *extra):
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        if fn(self.h, c.ctypes.data, len(c), *extra):
            raise RuntimeError(_err())
        return c

    def locate(self, cands):
        return self._inplace(ref_lib().ref_locate, cands)

    def split_points(self, cands):
        """compute_splitting_points (refine.hpp:267) on a candidate list."""
        fb = C.c_uint32()
        return self._inplace(ref_lib().ref_split_points, cands, C.byref(fb))

    def claim_filter(self, cands):
        return self._inplace(ref_lib().ref_claim, cands)

    def cavity_filter(self, cands, n: int = 32):
        return self._inplace(ref_lib().ref_cavity, cands, n)

    def insert_batch(self, cands, q: QualityCriteria, cfg: EngineConfig | None = None) -> dict:
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        p = params(q, cfg)
        out = (C.c_uint64 * 7)()
        if ref_lib().ref_insert_batch(self.h, c.ctypes.data, len(c), C.byref(p), out):
            raise RuntimeError(_err())
        keys = ("inserted_midpoints", "inserted_circumcenters", "removed_redundant",
                "removed_dependent", "dropped", "marked_encroached", "retained")
        return dict(zip(keys, list(out)))

    def split_only(self, cands) -> np.ndarray:
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        fresh = np.zeros(len(c) + 1, np.uint32)
        n = C.c_uint32()
        if ref_lib().ref_split_only(self.h, c.ctypes.data, len(c), fresh.ctypes.data, C.byref(n)):
            raise RuntimeError(_err())
        return fresh[: n.value]

    def incident(self, v: int) -> np.ndarray:
        out = np.zeros(256, np.uint32)
        k = ref_lib().ref_incident(self.h, v, out.ctypes.data, 256)
        return out[:k]

    def lawson(self, tris, edges) -> None:
        t = np.ascontiguousarray(tris, np.uint32)
        e = np.ascontiguousarray(edges, np.uint8)
        if ref_lib().ref_lawson(self.h, t.ctypes.data, e.ctypes.data, len(t)):
            raise RuntimeError(_err())

    # -- validators --
    def check_structure(self) -> None:
        if ref_lib().ref_check_structure(self.h):
            raise AssertionError("check_structure: " + _err())

    def euler_holds(self) -> bool:
        return bool(ref_lib().ref_euler_holds(self.h))

    def conformity_ok(self, pts, segs) -> bool:
        pts = np.ascontiguousarray(pts, np.float64)
        segs = np.ascontiguousarray(segs, np.uint32).reshape(-1, 2)
        return ref_lib().ref_conformity_ok(self.h, pts.ctypes.data, len(pts), segs.ctypes.data,
                                           len(segs)) == 1

    def cdt_violations(self, cap: int = 32) -> int:
        return int(ref_lib().ref_cdt_violations(self.h, cap))

    def delaunay_violations(self, cap: int = 32) -> int:
        return int(ref_lib().ref_delaunay_violations(self.h, cap))

    def count_bad(self, q: QualityCriteria) -> int:
        p = params(q)
        return int(ref_lib().ref_count_bad(self.h, C.byref(p)))

    def min_angle_hist(self, bin_deg: float = HIST_BIN_DEG, nbins: int = HIST_BINS):
        """(histogram of per-triangle min angles, mean min angle) with the
        corner-angle formula of min_angle_degrees (verify.hpp:186-200)."""
        h = np.zeros(nbins, np.uint64)
        s = C.c_double()
        n = ref_lib().ref_min_angle_hist(self.h, bin_deg, nbins, h.ctypes.data, C.byref(s))
        return h, (s.value / n if n else 0.0)

    def canonical_triangles(self) -> np.ndarray:
        _, t, _ = self.sizes()
        out = np.zeros((max(t, 1), 3), np.uint32)
        k = ref_lib().ref_canonical_triangles(self.h, out.ctypes.data)
        return out[:k]


def _report(r: A.Report, arr) -> RunReport:
    batches = []
    if arr is not None:
        for i in range(min(r.n_batches, r.batches_capacity)):
            b = arr[i]
            batches.append(BatchMetrics(
                batch_index=b.batch_index, attempted=b.attempted, concurrency=b.concurrency,
                latency=b.latency, throughput=b.throughput, waste_fraction=b.waste_fraction,
                phase_breakdown={A.PHASES[k]: b.phase_seconds[k] for k in range(6)},
                counters={}))
    return RunReport(batches=batches, output_points=r.output_points,
                     steiner_points=r.steiner_points, bad_triangles=r.bad_triangles,
                     bad_area_percent=r.bad_area_percent, min_angle_deg=r.min_angle_deg,
                     max_edge=r.max_edge, wall_seconds=r.wall_seconds,
                     iteration_cap_hit=bool(r.iteration_cap_hit),
                     totals={"total_candidates": r.total_candidates, "n_batches": r.n_batches})


def ref_predicates(kind: int, pts: np.ndarray, q: QualityCriteria | None = None) -> np.ndarray:
    pts = np.ascontiguousarray(pts, np.float64)
    out = np.zeros(len(pts), np.int8)
    p = params(q or QualityCriteria())
    ref_lib().ref_predicates_batch(kind, pts.ctypes.data, len(pts), C.byref(p), out.ctypes.data)
    return out


def ref_circumcenters(pts: np.ndarray):
    pts = np.ascontiguousarray(pts, np.float64)
    out = np.zeros((len(pts), 2), np.float64)
    ok = np.zeros(len(pts), np.uint8)
    ref_lib().ref_circumcenter_batch(pts.ctypes.data, len(pts), out.ctypes.data, ok.ctypes.data)
    return out, ok


def orc_predicates(kind: int, pts: np.ndarray, q: QualityCriteria | None = None) -> np.ndarray:
    pts = np.ascontiguousarray(pts, np.float64)
    out = np.zeros(len(pts), np.int8)
    p = params(q or QualityCriteria())
    orc_lib().orc_predicates_batch(kind, pts.ctypes.data, len(pts), C.byref(p), out.ctypes.data)
    return out


def orc_collect(m: Mesh, q: QualityCriteria, cfg: EngineConfig | None = None) -> np.ndarray:
    v = m.view()
    p = params(q, cfg)
    cap = m.n_triangles + m.n_subsegments + 1
    out = np.zeros(cap, dtype=A.candidate_dtype())
    n = orc_lib().orc_collect(C.byref(v), C.byref(p), out.ctypes.data, cap)
    return out[:n].copy()


def orc_locate(m: Mesh, cands) -> np.ndarray:
    v = m.view()
    c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
    orc_lib().orc_locate(C.byref(v), c.ctypes.data, len(c))
    return c


def orc_claim(m: Mesh, cands) -> np.ndarray:
    v = m.view()
    c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
    orc_lib().orc_claim(C.byref(v), c.ctypes.data, len(c))
    return c


def orc_cavity(m: Mesh, cands, n: int = 32, with_regions: bool = False):
    v = m.view()
    c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
    reg = np.zeros((len(c), n + 1), np.uint32)
    ln = np.zeros(len(c), np.uint32)
    orc_lib().orc_cavity(C.byref(v), c.ctypes.data, len(c), n, reg.ctypes.data, ln.ctypes.data)
    if with_regions:
        return c, [reg[i, : ln[i]].copy() for i in range(len(c))]
    return c
