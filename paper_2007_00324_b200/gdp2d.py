"""Host-side mirror of the reference's refinement interface, backed by libgdp2d.so.

Names, argument meaning and error behaviour follow cdtref (refine.hpp):

  QualityCriteria   refine.hpp:31     EngineConfig   refine.hpp:37
  RuleFlags         ruleskit.hpp:24   RunReport      ruleskit.hpp:42
  Mesh              mesh.hpp:64 (SoA numpy arrays, identical ids)
  refine(m, q, cfg) refine.hpp:651    -- runs entirely on the GPU
  Engine.collect / locate / claim_filter / cavity_filter / lawson_fixpoint:
                    refine.hpp:226,301,367,382, cdt.hpp:111 -- per-phase parity hooks

There is no CPU fallback: every call goes through the CUDA engine and raises
``MeshError`` / ``RuntimeError`` when the engine reports a failure.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi as A

RUPPERT = A.RUPPERT
CHEW = A.CHEW


class MeshError(RuntimeError):
    """Structural failure reported by the engine (cdtref::MeshError, mesh.hpp:38)."""


class CapacityExceeded(RuntimeError):
    """Device work-list capacity exceeded (cdtref::CapacityExceeded, expandlist.hpp:21)."""


class CdtError(RuntimeError):
    """The PSLG cannot be triangulated (cdtref::CdtError, cdt.hpp:20): duplicate
    points, all points collinear, crossing segments, non-finite coordinates."""


def _raise(rc: int, what: str = "") -> None:
    if rc == A.OK:
        return
    msg = A.engine().gdp2d_last_error().decode(errors="replace")
    text = f"{what}: {A.STATUS_NAMES.get(rc, rc)}: {msg}"
    if rc == A.EMESH:
        raise MeshError(text)
    if rc == A.ECAPACITY:
        raise CapacityExceeded(text)
    if rc == A.ECDT:
        raise CdtError(text)
    raise RuntimeError(text)


# ---- configuration --------------------------------------------------------------


@dataclass
class QualityCriteria:
    theta: float = 20.0
    ell: float = math.inf
    mode: int = RUPPERT


@dataclass
class RuleFlags:
    rule1_compaction_threshold: int = 1024
    rule2_filtering_enabled: bool = True
    rule3_gamma: float = 0.2
    rule4_unified_collection: bool = True
    rule5_split_lengthy_work: bool = True


@dataclass
class EngineConfig:
    cavity_n: int = 32
    rules: RuleFlags = field(default_factory=RuleFlags)
    iteration_cap: int = 10000
    split_depth_cap: int = 64
    batch_size_cap: int = 0
    seed: int = 0
    little_batch_sizing: bool = True   # Little's-law sizing from measured C / L (engine.cu)
    insert_mode: int = 1          # 1 = rollback (reference, default), 0 = isolated, 2 = precedence
    device: int = 0


def radius_edge_to_theta(b: float) -> float:
    """Radius-edge bound B -> min-angle theta = asin(1/(2B)) in degrees."""
    return math.degrees(math.asin(1.0 / (2.0 * b)))


def make_params(q: QualityCriteria, cfg: Optional[EngineConfig] = None) -> A.Params:
    cfg = cfg or EngineConfig()
    p = A.Params()
    A.engine().gdp2d_params_init(C.byref(p), float(q.theta), float(q.ell), int(q.mode))
    p.cavity_n = cfg.cavity_n
    p.rule1_compaction_threshold = cfg.rules.rule1_compaction_threshold
    p.rule2_filtering_enabled = int(bool(cfg.rules.rule2_filtering_enabled))
    p.rule4_unified_collection = int(bool(cfg.rules.rule4_unified_collection))
    p.little_batch_sizing = int(bool(cfg.little_batch_sizing))
    p.insert_mode = int(cfg.insert_mode)
    p.iteration_cap = cfg.iteration_cap
    p.split_depth_cap = cfg.split_depth_cap
    p.batch_size_cap = cfg.batch_size_cap
    return p


# ---- reports ------------------------------------------------------------------------


@dataclass
class BatchMetrics:
    batch_index: int
    attempted: int
    concurrency: int
    latency: float
    throughput: float
    waste_fraction: float
    phase_breakdown: dict
    counters: dict


@dataclass
class RunReport:
    batches: list
    output_points: int = 0
    steiner_points: int = 0
    bad_triangles: int = 0
    bad_area_percent: float = 0.0
    min_angle_deg: float = 0.0
    max_edge: float = 0.0
    wall_seconds: float = 0.0
    iteration_cap_hit: bool = False
    device_seconds: float = 0.0
    totals: dict = field(default_factory=dict)
    scan_seconds: float = 0.0
    scan_bytes: int = 0
    scan_launches: int = 0
    split_seconds: float = 0.0
    split_bytes: int = 0
    split_launches: int = 0
    rollback_seconds: float = 0.0
    rollback_bytes: int = 0
    rollback_launches: int = 0
    kernel_launches: int = 0
    e2e_seconds: float = 0.0

    def algorithmic_bytes(self) -> int:
        """SURVEY §8(d) bytes_alg from the per-batch counters."""
        t = self.totals
        return int(16 * t["sum_tris_alive"] + 16 * t["sum_verts_alive"] + 48 * t["sum_subsegs_alive"]
                   + 160 * t["total_candidates"] + 64 * t["total_walk_steps"]
                   + 64 * t["total_cavity_visits"] + 128 * t["total_inserted"]
                   + 128 * t["total_flips"])


_TOTALS = ("total_candidates", "total_walk_steps", "total_cavity_visits", "total_inserted",
           "total_flips", "total_removed", "sum_tris_alive", "sum_verts_alive",
           "sum_subsegs_alive")
_COUNTERS = ("tris_alive", "verts_alive", "subsegs_alive", "walk_steps", "cavity_visits",
             "survivors_claim", "survivors_cavity", "inserted_midpoints",
             "inserted_circumcenters", "removed_redundant", "removed_dependent", "dropped",
             "marked_encroached", "flips", "flip_rounds", "removal_rounds", "removals_kept")


def _report(r: A.Report, arr) -> RunReport:
    batches = []
    for i in range(min(r.n_batches, r.batches_capacity)):
        b = arr[i]
        batches.append(BatchMetrics(
            batch_index=b.batch_index, attempted=b.attempted, concurrency=b.concurrency,
            latency=b.latency, throughput=b.throughput, waste_fraction=b.waste_fraction,
            phase_breakdown={A.PHASES[k]: b.phase_seconds[k] for k in range(6)},
            counters={k: getattr(b, k) for k in _COUNTERS}))
    return RunReport(batches=batches, output_points=r.output_points,
                     steiner_points=r.steiner_points, bad_triangles=r.bad_triangles,
                     bad_area_percent=r.bad_area_percent, min_angle_deg=r.min_angle_deg,
                     max_edge=r.max_edge, wall_seconds=r.wall_seconds,
                     iteration_cap_hit=bool(r.iteration_cap_hit), device_seconds=r.device_seconds,
                     totals={k: getattr(r, k) for k in _TOTALS}, scan_seconds=r.scan_seconds,
                     scan_bytes=r.scan_bytes, scan_launches=r.scan_launches,
                     split_seconds=r.split_seconds, split_bytes=r.split_bytes,
                     split_launches=r.split_launches, rollback_seconds=r.rollback_seconds,
                     rollback_bytes=r.rollback_bytes, rollback_launches=r.rollback_launches,
                     e2e_seconds=r.e2e_seconds,
                     kernel_launches=r.kernel_launches)


def _new_report(cap: int = 20000):
    arr = (A.BatchMetrics * cap)()
    r = A.Report()
    r.batches = C.cast(arr, C.POINTER(A.BatchMetrics))
    r.batches_capacity = cap
    return r, arr


# ---- mesh ------------------------------------------------------------------------------

_FIELDS = (("xy", np.float64, 2), ("vert_kind", np.uint8, 1), ("vert_birth", np.uint32, 1),
           ("vert_alive", np.uint8, 1), ("vert_tri", np.uint32, 1), ("tri_v", np.uint32, 3),
           ("tri_n", np.uint32, 3), ("tri_seg", np.uint32, 3), ("tri_alive", np.uint8, 1),
           ("seg_v", np.uint32, 2), ("seg_parent", np.uint32, 1),
           ("seg_encroached", np.uint8, 1), ("seg_alive", np.uint8, 1), ("seg_tri", np.uint32, 1))
_VERT = {"xy", "vert_kind", "vert_birth", "vert_alive", "vert_tri"}
_TRI = {"tri_v", "tri_n", "tri_seg", "tri_alive"}


class Mesh:
    """cdtref::Mesh (mesh.hpp:64) as structure-of-arrays, ids identical."""

    def __init__(self, **arrays):
        self.batch_epoch = int(arrays.pop("batch_epoch", 0))
        for name, dt, w in _FIELDS:
            a = np.ascontiguousarray(arrays[name], dtype=dt)
            if w > 1:
                a = a.reshape(-1, w)
            setattr(self, name, a)

    @property
    def n_vertices(self) -> int:
        return int(self.xy.shape[0])

    @property
    def n_triangles(self) -> int:
        return int(self.tri_v.shape[0])

    @property
    def n_subsegments(self) -> int:
        return int(self.seg_v.shape[0])

    def alive_vertex_count(self) -> int:
        return int(self.vert_alive.sum())

    def alive_triangle_count(self) -> int:
        return int(self.tri_alive.sum())

    def alive_subsegment_count(self) -> int:
        return int(self.seg_alive.sum())

    def copy(self) -> "Mesh":
        return Mesh(batch_epoch=self.batch_epoch,
                    **{n: getattr(self, n).copy() for n, _, _ in _FIELDS})

    def view(self) -> A.MeshView:
        v = A.MeshView()
        v.n_vertices = self.n_vertices
        v.n_triangles = self.n_triangles
        v.n_subsegments = self.n_subsegments
        v.batch_epoch = self.batch_epoch
        for name, dt, _ in _FIELDS:
            arr = getattr(self, name)
            ct = {np.float64: C.c_double, np.uint8: C.c_uint8, np.uint32: C.c_uint32}[dt]
            setattr(v, name, arr.ctypes.data_as(C.POINTER(ct)))
        v._keep = self  # keep arrays alive
        return v

    @classmethod
    def from_buf(cls, b: A.MeshBuf, free) -> "Mesh":
        counts = {"v": b.n_vertices, "t": b.n_triangles, "s": b.n_subsegments}
        arrays = {}
        for name, dt, w in _FIELDS:
            n = counts["v"] if name in _VERT else counts["t"] if name in _TRI else counts["s"]
            ptr = getattr(b, name)
            if n == 0:
                arrays[name] = np.zeros((0, w) if w > 1 else 0, dtype=dt)
                continue
            a = np.ctypeslib.as_array(ptr, shape=(n * w,)).copy()
            arrays[name] = a.reshape(-1, w) if w > 1 else a
        mesh = cls(batch_epoch=b.batch_epoch, **arrays)
        free(C.byref(b))
        return mesh

    def assign(self, other: "Mesh") -> None:
        for name, _, _ in _FIELDS:
            setattr(self, name, getattr(other, name))
        self.batch_epoch = other.batch_epoch

    def canonical_triangles(self) -> np.ndarray:
        """Alive triangles as vertex triples rotated to start at the min id (orientation kept)."""
        t = self.tri_v[self.tri_alive.astype(bool)]
        r = np.argmin(t, axis=1)
        idx = (r[:, None] + np.arange(3)[None, :]) % 3
        return np.take_along_axis(t, idx, axis=1)


class _PinnedBlock:
    """One gdp2d_pinned_alloc allocation, freed when the last numpy view of it
    is gone (the views reference it through their ctypes base buffer)."""

    def __init__(self, lib, nbytes: int):
        self.lib = lib
        self.ptr = lib.gdp2d_pinned_alloc(nbytes)
        if not self.ptr:
            raise MemoryError(f"gdp2d_pinned_alloc({nbytes}) failed")

    def __del__(self):
        try:
            if self.ptr:
                self.lib.gdp2d_pinned_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


class PinnedPool:
    """Page-locked host buffers (gdp2d_pinned_alloc) for meshes of up to
    (nv, nt, ns) elements: uploads / downloads from here run at full link rate.
    ``mesh(...)`` returns a Mesh whose arrays are views into the pool (no copy).
    Each allocation lives as long as any view of it, so growing or closing the
    pool never frees memory a returned mesh still uses."""

    def __init__(self, nv: int, nt: int, ns: int):
        self.lib = A.engine()
        self._bufs = {}
        self._alloc(nv, nt, ns)

    def reserve(self, nv: int, nt: int, ns: int) -> None:
        """Grow (reallocate) so a mesh of (nv, nt, ns) fits; contents are not kept."""
        if nv > self.caps["v"] or nt > self.caps["t"] or ns > self.caps["s"]:
            self.close()
            self._alloc(max(nv, self.caps["v"]) * 5 // 4, max(nt, self.caps["t"]) * 5 // 4,
                        max(ns, self.caps["s"]) * 5 // 4)

    def _alloc(self, nv: int, nt: int, ns: int) -> None:
        self.caps = {"v": max(1, nv), "t": max(1, nt), "s": max(1, ns)}
        for name, dt, w in _FIELDS:
            n = self.caps["v" if name in _VERT else "t" if name in _TRI else "s"] * w
            nbytes = n * np.dtype(dt).itemsize
            block = _PinnedBlock(self.lib, nbytes)
            buf = (C.c_uint8 * nbytes).from_address(block.ptr)
            buf._owner = block          # views -> buf -> block: freed with the last view
            self._bufs[name] = np.frombuffer(buf, dtype=dt, count=n)

    def close(self) -> None:
        """Drop the pool's references (memory still viewed elsewhere stays valid)."""
        self._bufs = {}

    def mesh(self, nv: int, nt: int, ns: int, batch_epoch: int = 0) -> "Mesh":
        counts = {"v": nv, "t": nt, "s": ns}
        if any(counts[k] > self.caps[k] for k in counts):
            raise ValueError(f"mesh {counts} exceeds pinned capacity {self.caps}")
        arrays = {}
        for name, dt, w in _FIELDS:
            n = counts["v" if name in _VERT else "t" if name in _TRI else "s"]
            a = self._bufs[name][: n * w]
            arrays[name] = a.reshape(-1, w) if w > 1 else a
        return Mesh(batch_epoch=batch_epoch, **arrays)

    def load(self, src: "Mesh") -> "Mesh":
        """Copy a mesh into the pool (outside any timed region)."""
        m = self.mesh(src.n_vertices, src.n_triangles, src.n_subsegments, src.batch_epoch)
        for name, _, _ in _FIELDS:
            getattr(m, name)[...] = getattr(src, name)
        return m


# ---- whole-run entry point ---------------------------------------------------------


_ENGINES: dict = {}


def _engine_for(device: int) -> "Engine":
    eng = _ENGINES.get(device)
    if eng is None:
        eng = _ENGINES[device] = Engine(device)
    return eng


def warmup(device: int = 0) -> None:
    """gdp2d_warmup: create the cached device context and load the kernels
    (one tiny build + refinement), e.g. on a thread while inputs are read."""
    _raise(A.engine().gdp2d_warmup(int(device)), "gdp2d_warmup")


def refine(m: Mesh, q: QualityCriteria, cfg: Optional[EngineConfig] = None) -> RunReport:
    """cdtref::refine (refine.hpp:651) on the GPU; `m` is replaced by the refined mesh.

    Host buffers in, host buffers out, through the C ABI: upload (H2D of the
    input mesh), device-resident refinement, download straight into freshly
    allocated numpy arrays (D2H).  The device context is cached per device.
    report.wall_seconds covers the three steps.
    """
    import time
    cfg = cfg or EngineConfig()
    eng = _engine_for(cfg.device)
    t0 = time.perf_counter()
    eng.upload(m)
    rep = eng.refine(q, cfg)
    m.assign(eng.download())
    rep.wall_seconds = time.perf_counter() - t0
    return rep


def refine_c(m: Mesh, q: QualityCriteria, cfg: Optional[EngineConfig] = None) -> RunReport:
    """The single-call C entry point gdp2d_refine (library-owned output buffers)."""
    cfg = cfg or EngineConfig()
    lib = A.engine()
    p = make_params(q, cfg)
    r, arr = _new_report()
    out = A.MeshBuf()
    v = m.view()
    rc = lib.gdp2d_refine(C.byref(v), C.byref(out), C.byref(p), C.byref(r), cfg.device)
    _raise(rc, "gdp2d_refine")
    m.assign(Mesh.from_buf(out, lib.gdp2d_free))
    return _report(r, arr)


# ---- device-resident engine ---------------------------------------------------------


def build_cdt(points: np.ndarray, segments: np.ndarray, device: int = 0):
    """build_cdt (cdt.hpp:483) on the GPU: (Mesh, report).  ``segments`` must
    already include the hull edges (host.close_hull / read_poly).  Raises
    CdtError where the reference throws CdtError."""
    lib = A.engine()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    seg = np.ascontiguousarray(segments, dtype=np.uint32).reshape(-1, 2)
    out = A.MeshBuf()
    r = A.CdtReport()
    _raise(lib.gdp2d_build_cdt(pts.ctypes.data, len(pts), seg.ctypes.data, len(seg),
                               C.byref(out), C.byref(r), device), "gdp2d_build_cdt")
    return (Mesh.from_buf(out, lib.gdp2d_free),
            {name: getattr(r, name) for name, _ in A.CdtReport._fields_})


class Engine:
    """One device context: a pristine copy of the input mesh and a working mesh in HBM."""

    def __init__(self, device: int = 0):
        self.lib = A.engine()
        self.ctx = C.c_void_p()
        _raise(self.lib.gdp2d_ctx_create(C.byref(self.ctx), device), "gdp2d_ctx_create")
        self.device = device

    def close(self) -> None:
        if self.ctx:
            self.lib.gdp2d_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, m: Mesh) -> None:
        v = m.view()
        _raise(self.lib.gdp2d_ctx_upload(self.ctx, C.byref(v)), "gdp2d_ctx_upload")

    def reset(self) -> None:
        _raise(self.lib.gdp2d_ctx_reset(self.ctx), "gdp2d_ctx_reset")

    def build_cdt(self, points: np.ndarray, segments: np.ndarray) -> dict:
        """Line 1 on the device (build_cdt, cdt.hpp:483): the CDT of the PSLG
        (segments already hull-closed, host.close_hull) becomes this context's
        input mesh, as upload() would make it.  Returns the build report."""
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        seg = np.ascontiguousarray(segments, dtype=np.uint32).reshape(-1, 2)
        r = A.CdtReport()
        _raise(self.lib.gdp2d_ctx_build_cdt(self.ctx, pts.ctypes.data, len(pts), seg.ctypes.data,
                                            len(seg), C.byref(r)), "gdp2d_ctx_build_cdt")
        return {name: getattr(r, name) for name, _ in A.CdtReport._fields_}

    def refine(self, q: QualityCriteria, cfg: Optional[EngineConfig] = None) -> RunReport:
        p = make_params(q, cfg)
        r, arr = _new_report()
        _raise(self.lib.gdp2d_ctx_refine(self.ctx, C.byref(p), C.byref(r)), "gdp2d_ctx_refine")
        return _report(r, arr)

    def sizes(self):
        v, t, s = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _raise(self.lib.gdp2d_ctx_sizes(self.ctx, C.byref(v), C.byref(t), C.byref(s)),
               "gdp2d_ctx_sizes")
        return v.value, t.value, s.value

    def download(self) -> Mesh:
        """D2H of the working mesh straight into new numpy arrays."""
        nv, nt, ns = self.sizes()
        arrays = {}
        for name, dt, w in _FIELDS:
            n = nv if name in _VERT else nt if name in _TRI else ns
            arrays[name] = np.empty((n, w) if w > 1 else n, dtype=dt)
        mesh = Mesh(**arrays)
        b = A.MeshBuf()
        v = mesh.view()
        for fname, _ in A.MeshView._fields_[4:]:
            setattr(b, fname, getattr(v, fname))
        _raise(self.lib.gdp2d_ctx_download_to(self.ctx, C.byref(b)), "gdp2d_ctx_download_to")
        mesh.batch_epoch = b.batch_epoch
        return mesh

    def download_to(self, pool: "PinnedPool") -> Mesh:
        """D2H of the working mesh into page-locked pool buffers (allocation only
        when the pool is too small)."""
        nv, nt, ns = self.sizes()
        pool.reserve(nv, nt, ns)
        mesh = pool.mesh(nv, nt, ns)
        b = A.MeshBuf()
        b.n_vertices, b.n_triangles, b.n_subsegments = nv, nt, ns
        for name, dt, _ in _FIELDS:
            ct = {np.float64: C.c_double, np.uint8: C.c_uint8, np.uint32: C.c_uint32}[dt]
            setattr(b, name, getattr(mesh, name).ctypes.data_as(C.POINTER(ct)))
        _raise(self.lib.gdp2d_ctx_download_to(self.ctx, C.byref(b)), "gdp2d_ctx_download_to")
        mesh.batch_epoch = b.batch_epoch
        return mesh

    def export_node_ele(self):
        """Compacted write_node_ele data (gdp2d_ctx_export): (xy[n,2], marker[n],
        tri[m,3]) with dense vertex numbering, alive elements in id order."""
        nv, nt, _ = self.sizes()
        xy = np.empty((max(nv, 1), 2), np.float64)
        marker = np.empty(max(nv, 1), np.uint8)
        tri = np.empty((max(nt, 1), 3), np.uint32)
        o = A.NodeEle()
        o.xy = xy.ctypes.data_as(C.POINTER(C.c_double))
        o.marker = marker.ctypes.data_as(C.POINTER(C.c_uint8))
        o.tri = tri.ctypes.data_as(C.POINTER(C.c_uint32))
        _raise(self.lib.gdp2d_ctx_export(self.ctx, C.byref(o)), "gdp2d_ctx_export")
        return xy[: o.n_nodes], marker[: o.n_nodes], tri[: o.n_tris]

    def validate(self, q: QualityCriteria) -> dict:
        """Device validators (k_verify.cu) on the working mesh: structure, local
        CDT, quality, conformity to the uploaded input segments, and the
        histogram of per-triangle min angles (GDP2D_HIST_BINS bins of
        GDP2D_HIST_BIN_DEG degrees) with their mean."""
        p = make_params(q)
        v = A.Validation()
        _raise(self.lib.gdp2d_ctx_validate(self.ctx, C.byref(p), C.byref(v)), "gdp2d_ctx_validate")
        out = {f: getattr(v, f) for f, _ in A.Validation._fields_}
        out["min_angle_hist"] = [int(x) for x in v.min_angle_hist]
        return out

    def device_bytes(self) -> int:
        return int(self.lib.gdp2d_ctx_device_bytes(self.ctx))

    # -- per-phase parity hooks (operate on the working mesh) --

    def collect(self, q: QualityCriteria, cfg: Optional[EngineConfig] = None) -> np.ndarray:
        """collect + compute_splitting_points (refine.hpp:226-296)."""
        p = make_params(q, cfg)
        n = C.c_uint32(0)
        cap = 1 << 16
        while True:
            out = np.zeros(cap, dtype=A.candidate_dtype())
            rc = self.lib.gdp2d_collect(self.ctx, C.byref(p), out.ctypes.data, cap, C.byref(n))
            if rc == A.ECAPACITY and n.value > cap:
                cap = n.value
                continue
            _raise(rc, "gdp2d_collect")
            return out[: n.value].copy()

    def split_points(self, cands: np.ndarray) -> np.ndarray:
        """compute_splitting_points (refine.hpp:267-296) on a caller list."""
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        _raise(self.lib.gdp2d_split_points(self.ctx, c.ctypes.data, len(c)), "gdp2d_split_points")
        return c

    def locate(self, cands: np.ndarray) -> np.ndarray:
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        _raise(self.lib.gdp2d_locate(self.ctx, c.ctypes.data, len(c)), "gdp2d_locate")
        return c

    def claim_filter(self, cands: np.ndarray) -> np.ndarray:
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        _raise(self.lib.gdp2d_claim(self.ctx, c.ctypes.data, len(c)), "gdp2d_claim")
        return c

    def cavity_filter(self, cands: np.ndarray, n: int = 32, with_regions: bool = False):
        c = np.ascontiguousarray(cands, dtype=A.candidate_dtype()).copy()
        regions = np.zeros((len(c), n + 1), dtype=np.uint32)
        lens = np.zeros(len(c), dtype=np.uint32)
        _raise(self.lib.gdp2d_cavity(self.ctx, c.ctypes.data, len(c), n, regions.ctypes.data,
                                     lens.ctypes.data), "gdp2d_cavity")
        if with_regions:
            return c, [regions[i, : lens[i]].copy() for i in range(len(c))]
        return c

    def lawson_fixpoint(self, seeds_tri, seeds_edge) -> int:
        t = np.ascontiguousarray(seeds_tri, dtype=np.uint32)
        e = np.ascontiguousarray(seeds_edge, dtype=np.uint8)
        flips = C.c_uint64(0)
        _raise(self.lib.gdp2d_flip_fixpoint(self.ctx, t.ctypes.data, e.ctypes.data, len(t),
                                            C.byref(flips)), "gdp2d_flip_fixpoint")
        return int(flips.value)


# ---- predicates ------------------------------------------------------------------------------


def predicates(kind: int, pts: np.ndarray, q: Optional[QualityCriteria] = None,
               device: int = 0) -> np.ndarray:
    """Batch of one predicate on the GPU; pts shape (n, arity, 2)."""
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n = pts.shape[0]
    out = np.zeros(n, dtype=np.int8)
    p = make_params(q or QualityCriteria())
    _raise(A.engine().gdp2d_predicates_batch(device, kind, pts.ctypes.data, n, C.byref(p),
                                              out.ctypes.data), "gdp2d_predicates_batch")
    return out


def circumcenters(pts: np.ndarray, device: int = 0):
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n = pts.shape[0]
    out = np.zeros((n, 2), dtype=np.float64)
    ok = np.zeros(n, dtype=np.uint8)
    _raise(A.engine().gdp2d_circumcenter_batch(device, pts.ctypes.data, n, out.ctypes.data,
                                                ok.ctypes.data), "gdp2d_circumcenter_batch")
    return out, ok
