"""Shared, seeded test workloads (used by the parity tests and by
oracle/pin_against_reference.py so that golden digests are reproducible)."""

from __future__ import annotations

import math

import numpy as np

from paper_2407_02215_b200 import halfedge


def pentagon_cluster() -> halfedge.HalfedgeMesh:
    """Triangle + quad + pentagon sharing edges (H = 12): the mesh of the
    paper's Fig. 2/3, numbered as in the reference's tests/conftest.py:40-67."""
    ring = [[math.cos(a), math.sin(a), 0.0]
            for a in (math.pi / 2 + 2 * math.pi * k / 5 for k in range(5))]
    p0, p1, p2, p3, p4 = (np.array(p) for p in ring)
    x = p0 + p1 - (p2 + p4) / 2
    y = p1 + (p1 - p0)
    z = p2 + (p2 - p3)
    pts = [list(p) for p in (p0, p1, p2, p3, p4, x, y, z)]
    return halfedge.from_polygons(pts, [[5, 1, 0], [2, 1, 6, 7], [0, 1, 2, 3, 4]])


MESHES = {
    "triangle": halfedge.single_triangle,
    "quad": halfedge.single_quad,
    "grid2x2": lambda: halfedge.quad_grid(2, 2),
    "grid3x2": lambda: halfedge.quad_grid(3, 2),
    "dodeca": halfedge.dodecahedron,
    "pentagon_cluster": pentagon_cluster,
    "cube_sphere": lambda: halfedge.cube_sphere(1.0),
    "icosphere": lambda: halfedge.icosphere(1.0, 1),
}


def random_verdicts(n: int, seed: int, frame: int, split_p: float,
                    merge_p: float) -> np.ndarray:
    """int8[n] verdicts in cache_live order: 1 with prob split_p, 2 with prob
    merge_p, else 0.  Deliberately NOT budgeted against the free count, so
    reservation-pressure (OOM) rejections occur and are part of the parity."""
    rng = np.random.default_rng((seed * 7919 + frame * 104729 + n) & 0xFFFFFFFF)
    u = rng.random(n)
    v = np.zeros(n, dtype=np.int8)
    v[u < split_p] = 1
    v[u > 1.0 - merge_p] = 2
    return v


def soup_schedule(frame: int) -> tuple[float, float]:
    """Split/merge probabilities per frame: grow, churn, shrink, churn."""
    phase = frame % 8
    if phase < 3:
        return 0.45, 0.10
    if phase < 5:
        return 0.25, 0.35
    if phase < 7:
        return 0.05, 0.80
    return 0.35, 0.35


# (mesh name, pool depth, seed, frames): small pools so that OOM pressure and
# the admission tail path are exercised constantly
SOUP_CASES = [
    ("triangle", 4, 1, 24),
    ("triangle", 7, 2, 24),
    ("quad", 6, 3, 24),
    ("grid2x2", 8, 4, 24),
    ("grid3x2", 9, 5, 24),
    ("pentagon_cluster", 7, 6, 24),
    ("pentagon_cluster", 10, 7, 32),
    ("dodeca", 9, 8, 24),
    ("dodeca", 12, 9, 32),
    ("cube_sphere", 11, 10, 32),
    ("icosphere", 11, 11, 24),
    ("icosphere", 14, 12, 40),
]
