"""Shared test helpers (imported as a top-level module; tests/ has no __init__)."""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

B_SQRT2_THETA = math.degrees(math.asin(1.0 / (2.0 * math.sqrt(2.0))))  # 20.7048...


def unit_square():
    pts = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)
    segs = np.array([[0, 1], [1, 2], [2, 3], [3, 0]], dtype=np.uint32)
    return pts, segs


def regular_polygon(n, r, c=(0.0, 0.0)):
    return [(c[0] + r * math.cos(2 * math.pi * i / n), c[1] + r * math.sin(2 * math.pi * i / n))
            for i in range(n)]


def polygon_input(boundary, interior, seed):
    """acceptance.cpp:60-90 analogue: boundary polygon + interior points with a margin."""
    rng = np.random.default_rng(seed)
    b = np.array(boundary, dtype=np.float64)
    segs = [(i, (i + 1) % len(b)) for i in range(len(b))]
    lo, hi = b.min(0), b.max(0)
    margin = 0.01 * float((hi - lo).max())
    pts = [tuple(p) for p in b]

    def inside(p):
        x, y = p
        ins = False
        j = len(b) - 1
        for i in range(len(b)):
            if (b[i, 1] > y) != (b[j, 1] > y) and \
                    x < (b[j, 0] - b[i, 0]) * (y - b[i, 1]) / (b[j, 1] - b[i, 1]) + b[i, 0]:
                ins = not ins
            j = i
        return ins

    def dseg(p, a, c):
        ab = c - a
        t = np.clip(np.dot(p - a, ab) / max(np.dot(ab, ab), 1e-300), 0, 1)
        return np.linalg.norm(p - (a + t * ab))

    seen = set(pts)
    while interior > 0:
        p = (float(rng.uniform(lo[0], hi[0])), float(rng.uniform(lo[1], hi[1])))
        if p in seen or not inside(p):
            continue
        pa = np.array(p)
        if any(dseg(pa, b[i], b[j]) <= margin for i, j in segs):
            continue
        seen.add(p)
        pts.append(p)
        interior -= 1
    return np.array(pts, dtype=np.float64), np.array(segs, dtype=np.uint32)


def small_corpus():
    """A subset of acceptance.cpp:119-154's corpus (sizes trimmed for test time)."""
    h = 0.8660254037844386
    return {
        "square-100": polygon_input([(0, 0), (1, 0), (1, 1), (0, 1)], 96, 1),
        "triangle-400": polygon_input(regular_polygon(3, 2.0), 397, 4),
        "hexagon-200": polygon_input(regular_polygon(6, 1.0), 194, 5),
        "12gon-500": polygon_input(regular_polygon(12, 3.0), 488, 6),
        "notch-300": polygon_input([(0, 0), (4, 0), (4, 4), (2.5, 4), (2, 4 - h), (1.5, 4), (0, 4)],
                                   293, 9),
    }
