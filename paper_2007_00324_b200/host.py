"""Host side kept from the reference (north_star): PSLG/mesh I/O and the untimed
Line-1 CDT construction (cdtref build_cdt, cdt.hpp:483), plus the SURVEY §8(d)
synthetic PSLG generator.  Backed by lib/libgdp2d_host.so."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .gdp2d import Mesh

SEED = 20261017


def generate_pslg(n: int, m: int, dist: str = "uniform", seed: int = SEED):
    """(points (n,2) f64, segments (m',2) u32) -- hull not yet closed."""
    lib = A.host()
    xy = C.POINTER(C.c_double)()
    segs = C.POINTER(C.c_uint32)()
    mout = C.c_uint32(0)
    rc = lib.gdp2d_host_generate(n, m, 1 if dist == "gaussian" else 0, seed, C.byref(xy),
                                 C.byref(segs), C.byref(mout))
    if rc:
        raise RuntimeError("generator failed")
    pts = np.ctypeslib.as_array(xy, shape=(2 * n,)).reshape(n, 2).copy()
    s = (np.ctypeslib.as_array(segs, shape=(2 * mout.value,)).reshape(-1, 2).copy()
         if mout.value else np.zeros((0, 2), np.uint32))
    lib.gdp2d_host_free(C.cast(xy, C.c_void_p))
    lib.gdp2d_host_free(C.cast(segs, C.c_void_p))
    return pts, s


def build_cdt(points: np.ndarray, segments: np.ndarray, close_hull: bool = True):
    """close_hull (cdt.hpp:447) + check_crossings + build_cdt (cdt.hpp:483).

    Returns (Mesh, closed segment list)."""
    lib = A.host()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    seg = np.ascontiguousarray(segments, dtype=np.uint32).reshape(-1, 2)
    out = A.MeshBuf()
    so = C.POINTER(C.c_uint32)()
    mo = C.c_uint32(0)
    rc = lib.gdp2d_host_build_cdt(pts.ctypes.data, len(pts), seg.ctypes.data, len(seg),
                                  1 if close_hull else 0, C.byref(out), C.byref(so), C.byref(mo))
    if rc:
        raise RuntimeError("build_cdt: " + lib.gdp2d_host_last_error().decode())
    closed = np.ctypeslib.as_array(so, shape=(2 * mo.value,)).reshape(-1, 2).copy()
    lib.gdp2d_host_free(C.cast(so, C.c_void_p))
    return Mesh.from_buf(out, lib.gdp2d_host_free_buf), closed


def dropin_refine(mesh: Mesh, theta: float, device: int = 0):
    """One gdp2d::refine(cdtref::Mesh&, q, EngineConfig{}) call (the drop-in
    shim, include/gdp2d_cdtref.hpp) on the mesh as a reference AoS Mesh.
    Returns (refined Mesh, Steiner count)."""
    lib = A.host()
    v = mesh.view()
    out = A.MeshBuf()
    st = C.c_uint64()
    if lib.gdp2d_host_dropin_refine(C.byref(v), theta, device, C.byref(out), C.byref(st)):
        raise RuntimeError("gdp2d::refine: " + lib.gdp2d_host_last_error().decode())
    return Mesh.from_buf(out, lib.gdp2d_host_free_buf), int(st.value)


def time_dropin(mesh: Mesh, theta: float, steps: int, device: int = 0, parts: bool = False):
    """The drop-in caller's path (include/gdp2d_cdtref.hpp): `steps` calls of
    gdp2d::refine(cdtref::Mesh&, q, EngineConfig{}) on copies of the mesh as
    a reference AoS Mesh in pageable memory.  Returns (seconds summed over
    the calls, Steiner count of the last call[, per-step breakdown dict when
    parts: transfers (H2D, device record conversion, D2H), the refinement
    loop, and the shim around the library call])."""
    lib = A.host()
    v = mesh.view()
    secs = C.c_double()
    st = C.c_uint64()
    pv = (C.c_double * 4)()
    if lib.gdp2d_host_time_dropin(C.byref(v), theta, steps, device, C.byref(secs), C.byref(st),
                                  pv if parts else None):
        raise RuntimeError("gdp2d::refine: " + lib.gdp2d_host_last_error().decode())
    if not parts:
        return secs.value, int(st.value)
    names = ("transfers_s", "refine_loop_s", "shim_s")
    return secs.value, int(st.value), {k: pv[i] / steps for i, k in enumerate(names)}


def close_hull(points: np.ndarray, segments: np.ndarray, check: bool = True) -> np.ndarray:
    """close_hull (cdt.hpp:447) [+ check_crossings]: the closed segment list."""
    lib = A.host()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    seg = np.ascontiguousarray(segments, dtype=np.uint32).reshape(-1, 2)
    so = C.POINTER(C.c_uint32)()
    mo = C.c_uint32(0)
    rc = lib.gdp2d_host_close_hull(pts.ctypes.data, len(pts), seg.ctypes.data, len(seg),
                                   1 if check else 0, C.byref(so), C.byref(mo))
    if rc:
        raise RuntimeError("close_hull: " + lib.gdp2d_host_last_error().decode())
    closed = np.ctypeslib.as_array(so, shape=(2 * mo.value,)).reshape(-1, 2).copy() \
        if mo.value else np.zeros((0, 2), np.uint32)
    lib.gdp2d_host_free(C.cast(so, C.c_void_p))
    return closed


def read_poly(text: str):
    """read_poly (pslg_io.hpp:272): parsed, de-duplicated, crossing-checked, hull closed."""
    lib = A.host()
    xy = C.POINTER(C.c_double)()
    segs = C.POINTER(C.c_uint32)()
    n = C.c_uint32(0)
    m = C.c_uint32(0)
    rc = lib.gdp2d_host_read_poly(text.encode(), C.byref(xy), C.byref(n), C.byref(segs),
                                  C.byref(m))
    if rc:
        raise ValueError(lib.gdp2d_host_last_error().decode())
    pts = np.ctypeslib.as_array(xy, shape=(2 * n.value,)).reshape(-1, 2).copy()
    s = np.ctypeslib.as_array(segs, shape=(2 * m.value,)).reshape(-1, 2).copy() if m.value else \
        np.zeros((0, 2), np.uint32)
    lib.gdp2d_host_free(C.cast(xy, C.c_void_p))
    lib.gdp2d_host_free(C.cast(segs, C.c_void_p))
    return pts, s


def write_node_ele(mesh: Mesh):
    """write_node_ele (pslg_io.hpp:294) -> (node text, ele text)."""
    lib = A.host()
    node = C.c_char_p()
    ele = C.c_char_p()
    v = mesh.view()
    rc = lib.gdp2d_host_write_node_ele(C.byref(v), C.byref(node), C.byref(ele))
    if rc:
        raise RuntimeError(lib.gdp2d_host_last_error().decode())
    return _take_texts(lib, node, ele)


def _take_texts(lib, node, ele):
    """Decode two malloc'ed C strings from the host library and free them."""
    try:
        return node.value.decode(), ele.value.decode()
    finally:
        lib.gdp2d_host_free(C.cast(node, C.c_void_p))
        lib.gdp2d_host_free(C.cast(ele, C.c_void_p))


def format_node_ele(xy: np.ndarray, marker: np.ndarray, tri: np.ndarray):
    """.node/.ele text of a compacted export (Engine.export_node_ele), byte-
    identical to write_node_ele (pslg_io.hpp:294) of the same mesh."""
    lib = A.host()
    node = C.c_char_p()
    ele = C.c_char_p()
    xy = np.ascontiguousarray(xy, np.float64)
    marker = np.ascontiguousarray(marker, np.uint8)
    tri = np.ascontiguousarray(tri, np.uint32)
    rc = lib.gdp2d_host_format_node_ele(len(xy), xy.ctypes.data, marker.ctypes.data, len(tri),
                                        tri.ctypes.data, C.byref(node), C.byref(ele))
    if rc:
        raise RuntimeError(lib.gdp2d_host_last_error().decode())
    return _take_texts(lib, node, ele)


def workload(config: int, seed: int = SEED):
    """BASELINE.json configs -> (points, segments, theta).  Theta in degrees."""
    import math
    b_theta = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))  # radius-edge sqrt(2)
    table = {
        1: (100_000, 1_000, "uniform", b_theta),
        2: (1_000_000, 100_000, "uniform", b_theta),
        3: (5_000_000, 500_000, "gaussian", b_theta),
        4: (1_000_000, 100_000, "uniform", 30.0),
        5: (2_000_000, 200_000, "uniform", b_theta),
    }
    n, m, dist, theta = table[config]
    pts, segs = generate_pslg(n, m, dist, seed)
    return pts, segs, theta
