"""Seeded predicate inputs mirroring the reference's predicate tests
(test_predicates.cpp:65-124): random, near-collinear (+-2 ulp at 2^-50) and
near-cocircular quadruples.  Shared by the CPU oracle tests and the GPU tests."""
from __future__ import annotations

import math

import numpy as np


def near_collinear(n: int, seed: int = 42) -> np.ndarray:
    """test_predicates.cpp:90-107: points on y = 0.5x + 0.25 jittered by k*2^-50."""
    rng = np.random.default_rng(seed)
    ulp = math.ldexp(1.0, -50)
    x = rng.uniform(-1.0, 1.0, size=(n, 3))
    jx = rng.integers(-2, 3, size=(n, 3)) * ulp
    jy = rng.integers(-2, 3, size=(n, 3)) * ulp
    pts = np.empty((n, 3, 2))
    pts[..., 0] = x + jx
    pts[..., 1] = 0.5 * x + 0.25 + jy
    return pts


def near_cocircular(n: int, seed: int = 43) -> np.ndarray:
    """test_predicates.cpp:109-124: 4 points on the unit circle jittered by k*2^-50,
    first three in CCW order."""
    rng = np.random.default_rng(seed)
    ulp = math.ldexp(1.0, -50)
    t = rng.uniform(0.0, 6.28318, size=(n, 4))
    pts = np.empty((n, 4, 2))
    pts[..., 0] = np.cos(t) + rng.integers(-2, 3, size=(n, 4)) * ulp
    pts[..., 1] = np.sin(t) + rng.integers(-2, 3, size=(n, 4)) * ulp
    a, b, c = pts[:, 0], pts[:, 1], pts[:, 2]
    o = (a[:, 0] - c[:, 0]) * (b[:, 1] - c[:, 1]) - (a[:, 1] - c[:, 1]) * (b[:, 0] - c[:, 0])
    swap = o < 0
    tmp = pts[swap, 1].copy()
    pts[swap, 1] = pts[swap, 2]
    pts[swap, 2] = tmp
    return pts


def random_points(n: int, arity: int, lo=-10.0, hi=10.0, seed: int = 7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(n, arity, 2))


def grid_degenerate(n: int, arity: int, seed: int = 5) -> np.ndarray:
    """Exactly degenerate inputs on a small integer grid (many zero signs)."""
    rng = np.random.default_rng(seed)
    return rng.integers(-3, 4, size=(n, arity, 2)).astype(np.float64) * 0.25


def diametric_cases(n: int, seed: int = 13) -> np.ndarray:
    """Segment + point with the point near the diametral circle / lens boundary."""
    rng = np.random.default_rng(seed)
    sa = rng.uniform(-3, 3, size=(n, 2))
    sb = rng.uniform(-3, 3, size=(n, 2))
    mid = 0.5 * (sa + sb)
    r = 0.5 * np.linalg.norm(sb - sa, axis=1)
    ang = rng.uniform(0, 2 * math.pi, size=n)
    scale = rng.choice([1.0, 1.0 - 1e-15, 1.0 + 1e-15, 0.9, 0.577, 0.5773502691896258], size=n)
    p = mid + (r * scale)[:, None] * np.stack([np.cos(ang), np.sin(ang)], axis=1)
    return np.stack([sa, sb, p], axis=1)


def triangles_near_bound(theta_deg: float, n: int, seed: int = 3) -> np.ndarray:
    """Isoceles triangles with apex angle around theta (test_refine.cpp:57-67) + random."""
    rng = np.random.default_rng(seed)
    ang = np.radians(theta_deg + rng.uniform(-5, 5, size=n))
    a = np.zeros((n, 2))
    b = np.stack([np.full(n, 2.0), np.zeros(n)], axis=1)
    c = np.stack([2 * np.cos(ang), 2 * np.sin(ang)], axis=1)
    tri = np.stack([a, b, c], axis=1)
    rnd = rng.uniform(0, 1, size=(n, 3, 2))
    return np.concatenate([tri, rnd])


def mesh_scale_cocircular(n: int, seed: int = 17) -> np.ndarray:
    """Near-cocircular quadruples at mesh scale: centre in the unit square,
    radius 1e-2..1e-7, jitter of a few ulps of the coordinates (first three CCW)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.0, 1.0, size=(n, 1, 2))
    r = 10.0 ** rng.uniform(-7, -2, size=(n, 1, 1))
    t = np.sort(rng.uniform(0.0, 2 * math.pi, size=(n, 4)), axis=1)
    pts = c + r * np.stack([np.cos(t), np.sin(t)], axis=2)
    ulp = np.spacing(np.abs(pts) + 1e-300)
    pts = pts + rng.integers(-2, 3, size=pts.shape) * ulp
    return pts


def mesh_scale_collinear(n: int, seed: int = 19) -> np.ndarray:
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 1.0, size=(n, 1, 2))
    d = rng.normal(size=(n, 1, 2)) * 10.0 ** rng.uniform(-7, -2, size=(n, 1, 1))
    s = rng.uniform(-1, 2, size=(n, 3, 1))
    pts = a + s * d
    ulp = np.spacing(np.abs(pts) + 1e-300)
    return pts + rng.integers(-1, 2, size=pts.shape) * ulp
