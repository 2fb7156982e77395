"""ctypes mirror of include/gdp2d.h (layouts checked against gdp2d_struct_size)."""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"

NONE = 0xFFFFFFFF
PENDING = 0xFFFFFFFE

# status codes
OK, EINVAL, ECUDA, ENODEVICE, ECAPACITY, EMESH, EINTERNAL, ECDT = range(8)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ECUDA", 3: "ENODEVICE", 4: "ECAPACITY", 5: "EMESH",
                6: "EINTERNAL", 7: "ECDT"}
RUPPERT, CHEW = 0, 1
CAND_SUBSEG, CAND_TRI = 0, 1
BAND_CIRCUMCENTER, BAND_MIDPOINT = 0, 1
PRED_ORIENT2D, PRED_INCIRCLE, PRED_DIAMETRIC, PRED_LENS, PRED_BAD_TRIANGLE = range(5)
PHASES = ("collect", "split_points", "locate", "claim", "cavity", "insert")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)


class MeshView(C.Structure):
    _fields_ = [("n_vertices", C.c_uint32), ("n_triangles", C.c_uint32),
                ("n_subsegments", C.c_uint32), ("batch_epoch", C.c_uint32),
                ("xy", f64p), ("vert_kind", u8p), ("vert_birth", u32p), ("vert_alive", u8p),
                ("vert_tri", u32p), ("tri_v", u32p), ("tri_n", u32p), ("tri_seg", u32p),
                ("tri_alive", u8p), ("seg_v", u32p), ("seg_parent", u32p),
                ("seg_encroached", u8p), ("seg_alive", u8p), ("seg_tri", u32p)]


MeshBuf = type("MeshBuf", (C.Structure,), {"_fields_": MeshView._fields_})


class Params(C.Structure):
    _fields_ = [("theta_deg", C.c_double), ("cos2_theta", C.c_double), ("ell", C.c_double),
                ("mode", C.c_uint32), ("cavity_n", C.c_uint32),
                ("rule1_compaction_threshold", C.c_uint32),
                ("rule2_filtering_enabled", C.c_uint32),
                ("rule4_unified_collection", C.c_uint32), ("little_batch_sizing", C.c_uint32),
                ("insert_mode", C.c_uint32), ("reserved0", C.c_uint32),
                ("iteration_cap", C.c_uint64), ("split_depth_cap", C.c_uint64),
                ("batch_size_cap", C.c_uint64)]


class BatchMetrics(C.Structure):
    _fields_ = [("batch_index", C.c_uint32), ("attempted", C.c_uint32),
                ("concurrency", C.c_uint32), ("removals_kept", C.c_uint32), ("latency", C.c_double),
                ("throughput", C.c_double), ("waste_fraction", C.c_double),
                ("phase_seconds", C.c_double * 6), ("tris_alive", C.c_uint64),
                ("verts_alive", C.c_uint64), ("subsegs_alive", C.c_uint64),
                ("walk_steps", C.c_uint64), ("cavity_visits", C.c_uint64),
                ("survivors_claim", C.c_uint32), ("survivors_cavity", C.c_uint32),
                ("inserted_midpoints", C.c_uint32), ("inserted_circumcenters", C.c_uint32),
                ("removed_redundant", C.c_uint32), ("removed_dependent", C.c_uint32),
                ("dropped", C.c_uint32), ("marked_encroached", C.c_uint32),
                ("flips", C.c_uint64), ("flip_rounds", C.c_uint32),
                ("removal_rounds", C.c_uint32)]


class Report(C.Structure):
    _fields_ = [("batches", C.POINTER(BatchMetrics)), ("batches_capacity", C.c_uint32),
                ("n_batches", C.c_uint32), ("output_points", C.c_uint64),
                ("steiner_points", C.c_uint64), ("bad_triangles", C.c_uint64),
                ("bad_area_percent", C.c_double), ("min_angle_deg", C.c_double),
                ("max_edge", C.c_double), ("wall_seconds", C.c_double),
                ("iteration_cap_hit", C.c_int32), ("pad0", C.c_int32),
                ("total_candidates", C.c_uint64), ("total_walk_steps", C.c_uint64),
                ("total_cavity_visits", C.c_uint64), ("total_inserted", C.c_uint64),
                ("total_flips", C.c_uint64), ("total_removed", C.c_uint64),
                ("sum_tris_alive", C.c_uint64), ("sum_verts_alive", C.c_uint64),
                ("sum_subsegs_alive", C.c_uint64), ("device_seconds", C.c_double),
                ("scan_seconds", C.c_double), ("scan_bytes", C.c_uint64),
                ("scan_launches", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("split_seconds", C.c_double), ("split_bytes", C.c_uint64),
                ("split_launches", C.c_uint64), ("rollback_seconds", C.c_double),
                ("rollback_bytes", C.c_uint64), ("rollback_launches", C.c_uint64),
                ("e2e_seconds", C.c_double)]


class Validation(C.Structure):
    _fields_ = [("structure_failure", C.c_uint32), ("structure_tri", C.c_uint32),
                ("cdt_violations", C.c_uint64), ("bad_triangles", C.c_uint64),
                ("conformity_failures", C.c_uint64), ("min_angle_deg", C.c_double),
                ("mean_min_angle_deg", C.c_double), ("min_angle_hist", C.c_uint64 * 120)]


class NodeEle(C.Structure):
    _fields_ = [("n_nodes", C.c_uint32), ("n_tris", C.c_uint32),
                ("xy", C.POINTER(C.c_double)), ("marker", C.POINTER(C.c_uint8)),
                ("tri", C.POINTER(C.c_uint32))]


class CdtReport(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("n_triangles", C.c_uint32),
                ("n_subsegments", C.c_uint32), ("insert_rounds", C.c_uint32),
                ("flip_rounds", C.c_uint32), ("recover_rounds", C.c_uint32),
                ("segments_present", C.c_uint32), ("pipes_recovered", C.c_uint32),
                ("collinear_splits", C.c_uint32), ("max_pipe", C.c_uint32),
                ("final_flip_rounds", C.c_uint32), ("reserved", C.c_uint32),
                ("flips", C.c_uint64), ("seconds", C.c_double),
                ("delaunay_seconds", C.c_double), ("recover_seconds", C.c_double),
                ("finish_seconds", C.c_double)]


class Candidate(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("measure", C.c_double),
                ("id", C.c_uint32), ("tiebreak", C.c_uint32), ("located", C.c_uint32),
                ("kind", C.c_uint8), ("band", C.c_uint8), ("alive", C.c_uint8),
                ("fallback", C.c_uint8)]


# numpy dtype with the same layout as gdp2d_candidate
def candidate_dtype():
    import numpy as np
    return np.dtype([("x", "<f8"), ("y", "<f8"), ("measure", "<f8"), ("id", "<u4"),
                     ("tiebreak", "<u4"), ("located", "<u4"), ("kind", "u1"), ("band", "u1"),
                     ("alive", "u1"), ("fallback", "u1")])


class AosLayout(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "vert_size", "vert_pos", "vert_kind", "vert_birth", "vert_alive",
        "tri_size", "tri_v", "tri_nbr", "tri_seg", "tri_alive",
        "seg_size", "seg_v", "seg_parent", "seg_encroached", "seg_alive")]


AOS_RESIZE = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_int, C.c_uint64)


class AosMesh(C.Structure):
    _fields_ = [("n_vertices", C.c_uint32), ("n_triangles", C.c_uint32),
                ("n_subsegments", C.c_uint32), ("batch_epoch", C.c_uint32),
                ("verts", C.c_void_p), ("tris", C.c_void_p), ("segs", C.c_void_p),
                ("vert_tri", C.c_void_p), ("seg_tri", C.c_void_p),
                ("resize", AOS_RESIZE), ("user", C.c_void_p)]


STRUCTS = [MeshView, MeshBuf, Params, BatchMetrics, Report, Candidate, Validation, NodeEle,
           CdtReport, AosLayout, AosMesh]

# Every entry point of include/gdp2d.h: name -> (restype, argtypes)
ctx_p = C.c_void_p
SIGNATURES = {
    "gdp2d_params_init": (None, [C.POINTER(Params), C.c_double, C.c_double, C.c_uint32]),
    "gdp2d_refine_aos": (C.c_int, [C.POINTER(AosLayout), C.POINTER(AosMesh), C.POINTER(Params),
                                   C.POINTER(Report), C.c_int]),
    "gdp2d_refine": (C.c_int, [C.POINTER(MeshView), C.POINTER(MeshBuf), C.POINTER(Params),
                               C.POINTER(Report), C.c_int]),
    "gdp2d_free": (None, [C.POINTER(MeshBuf)]),
    "gdp2d_pinned_alloc": (C.c_void_p, [C.c_size_t]),
    "gdp2d_pinned_free": (None, [C.c_void_p]),
    "gdp2d_ctx_validate": (C.c_int, [ctx_p, C.POINTER(Params), C.POINTER(Validation)]),
    "gdp2d_ctx_export": (C.c_int, [ctx_p, C.POINTER(NodeEle)]),
    "gdp2d_ctx_build_cdt": (C.c_int, [ctx_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                      C.POINTER(CdtReport)]),
    "gdp2d_build_cdt": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                  C.POINTER(MeshBuf), C.POINTER(CdtReport), C.c_int]),
    "gdp2d_last_error": (C.c_char_p, []),
    "gdp2d_version": (C.c_char_p, []),
    "gdp2d_struct_size": (C.c_size_t, [C.c_int]),
    "gdp2d_kernel_launches": (C.c_uint64, []),
    "gdp2d_ctx_create": (C.c_int, [C.POINTER(ctx_p), C.c_int]),
    "gdp2d_ctx_destroy": (None, [ctx_p]),
    "gdp2d_ctx_upload": (C.c_int, [ctx_p, C.POINTER(MeshView)]),
    "gdp2d_ctx_reset": (C.c_int, [ctx_p]),
    "gdp2d_ctx_refine": (C.c_int, [ctx_p, C.POINTER(Params), C.POINTER(Report)]),
    "gdp2d_ctx_download": (C.c_int, [ctx_p, C.POINTER(MeshBuf)]),
    "gdp2d_ctx_device_bytes": (C.c_uint64, [ctx_p]),
    "gdp2d_ctx_sizes": (C.c_int, [ctx_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                  C.POINTER(C.c_uint32)]),
    "gdp2d_ctx_download_to": (C.c_int, [ctx_p, C.POINTER(MeshBuf)]),
    "gdp2d_release_cached": (None, []),
    "gdp2d_warmup": (C.c_int, [C.c_int]),
    "gdp2d_collect": (C.c_int, [ctx_p, C.POINTER(Params), C.c_void_p, C.c_uint32,
                                C.POINTER(C.c_uint32)]),
    "gdp2d_split_points": (C.c_int, [ctx_p, C.c_void_p, C.c_uint32]),
    "gdp2d_locate": (C.c_int, [ctx_p, C.c_void_p, C.c_uint32]),
    "gdp2d_claim": (C.c_int, [ctx_p, C.c_void_p, C.c_uint32]),
    "gdp2d_cavity": (C.c_int, [ctx_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p,
                               C.c_void_p]),
    "gdp2d_flip_fixpoint": (C.c_int, [ctx_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                      C.POINTER(C.c_uint64)]),
    "gdp2d_predicates_batch": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_uint32,
                                         C.POINTER(Params), C.c_void_p]),
    "gdp2d_circumcenter_batch": (C.c_int, [C.c_int, C.c_void_p, C.c_uint32, C.c_void_p,
                                           C.c_void_p]),
}

HOST_SIGNATURES = {
    "gdp2d_host_generate": (C.c_int, [C.c_uint64, C.c_uint32, C.c_int, C.c_uint64,
                                      C.POINTER(f64p), C.POINTER(u32p), C.POINTER(C.c_uint32)]),
    "gdp2d_host_free": (None, [C.c_void_p]),
    "gdp2d_host_build_cdt": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int,
                                       C.POINTER(MeshBuf), C.POINTER(u32p),
                                       C.POINTER(C.c_uint32)]),
    "gdp2d_host_close_hull": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int,
                                        C.POINTER(u32p), C.POINTER(C.c_uint32)]),
    "gdp2d_host_read_poly": (C.c_int, [C.c_char_p, C.POINTER(f64p), C.POINTER(C.c_uint32),
                                       C.POINTER(u32p), C.POINTER(C.c_uint32)]),
    "gdp2d_host_write_node_ele": (C.c_int, [C.POINTER(MeshView), C.POINTER(C.c_char_p),
                                            C.POINTER(C.c_char_p)]),
    "gdp2d_host_format_node_ele": (C.c_int, [C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint32,
                                             C.c_void_p, C.POINTER(C.c_char_p),
                                             C.POINTER(C.c_char_p)]),
    "gdp2d_host_free_buf": (None, [C.POINTER(MeshBuf)]),
    "gdp2d_host_last_error": (C.c_char_p, []),
    "gdp2d_host_dropin_refine": (C.c_int, [C.POINTER(MeshView), C.c_double, C.c_int,
                                           C.POINTER(MeshBuf), C.POINTER(C.c_uint64)]),
    "gdp2d_host_time_dropin": (C.c_int, [C.POINTER(MeshView), C.c_double, C.c_int, C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                         C.c_void_p]),
}

_LIBS: dict[str, C.CDLL] = {}


def _load(name: str, sigs: dict) -> C.CDLL:
    if name in _LIBS:
        return _LIBS[name]
    path = LIB_DIR / name
    if name == "libgdp2d.so" and os.environ.get("GDP2D_ENGINE_LIB"):
        path = Path(os.environ["GDP2D_ENGINE_LIB"])   # A/B builds (tools/ab_bench.sh)
    if not path.exists():
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2007_00324_b200.build` "
            "(there is no CPU fallback for the refinement engine)")
    lib = C.CDLL(str(path))
    for sym, (res, args) in sigs.items():
        fn = getattr(lib, sym)
        fn.restype = res
        fn.argtypes = args
    _LIBS[name] = lib
    return lib


def engine() -> C.CDLL:
    """libgdp2d.so (the CUDA engine)."""
    return _load("libgdp2d.so", SIGNATURES)


def host() -> C.CDLL:
    """libgdp2d_host.so (reference-side PSLG/mesh I/O + generator)."""
    return _load("libgdp2d_host.so", HOST_SIGNATURES)


def check_layouts() -> None:
    lib = engine()
    for i, st in enumerate(STRUCTS):
        want = lib.gdp2d_struct_size(i)
        if C.sizeof(st) != want:
            raise RuntimeError(f"ABI mismatch for {st.__name__}: python {C.sizeof(st)} vs C {want}")
