"""Bisector heap ids and host-side fp64 vertex decoding.

A bisector id packs its whole split path: the root bisector of halfedge
``h`` is ``2**R + h`` (``R = max(1, ceil(log2 H))``) and the two halves of
``j`` are ``2j`` / ``2j+1``.  Depth and root halfedge fall out of the id, so
the pool stores one u64 per record (reference: pkg/src/cbtmesh/bisector.py:23-60
for the id helpers, :100-183 for the subdivision-matrix decode).

The device classifier (csrc/cbtm_classify.cuh) and the C oracle
(oracle/cbtm_oracle.c) implement the same decode; this module is the host
mirror used by validators, tests and the python-callable verdict path.
"""

from __future__ import annotations

import numpy as np

# Rows of M @ [v0; v1; v2] are the child's vertices: child 0 keeps v0, child 1
# keeps v1, both get v2 := midpoint(v0, v1) and the old apex moves to row 1 / 0.
M0 = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0], [0.5, 0.5, 0.0]])
M1 = np.array([[0.0, 0.0, 1.0], [0.0, 1.0, 0.0], [0.5, 0.5, 0.0]])


def root_rank(n_halfedges: int) -> int:
    if n_halfedges < 1:
        raise ValueError("halfedge count must be >= 1")
    return max(1, (n_halfedges - 1).bit_length())


def max_depth(n_halfedges: int) -> int:
    """Deepest level whose ids still fit 64 bits."""
    return 63 - root_rank(n_halfedges)


def make_root_id(n_halfedges: int, h: int) -> int:
    if not 0 <= h < n_halfedges:
        raise ValueError(f"halfedge {h} out of range [0, {n_halfedges})")
    return (1 << root_rank(n_halfedges)) + h


def depth_of(bid: int, rank: int) -> int:
    d = int(bid).bit_length() - 1 - rank
    assert d >= 0, f"id {bid} below root rank {rank}"
    return d


def root_halfedge(bid: int, rank: int) -> int:
    return (int(bid) >> depth_of(bid, rank)) - (1 << rank)


def children(bid: int) -> tuple[int, int]:
    if int(bid) >> 63:
        raise OverflowError(
            f"children of {bid} exceed the 64-bit index range")
    return 2 * int(bid), 2 * int(bid) + 1


def parent(bid: int) -> int:
    return int(bid) >> 1


def path_matrix(bid: int, rank: int) -> np.ndarray:
    """Product of split matrices along the id's path, deepest bit first."""
    bid = int(bid)
    root = bid >> depth_of(bid, rank)
    m = np.eye(3)
    while bid != root:
        m = m @ (M1 if bid & 1 else M0)
        bid >>= 1
    return m


def bisector_vertices(mesh, bid: int) -> np.ndarray:
    """(3, 3) fp64 vertex rows of bisector ``bid`` on ``mesh``."""
    rank = root_rank(mesh.n_halfedges)
    h = root_halfedge(bid, rank)
    assert 0 <= h < mesh.n_halfedges, f"id {bid} maps outside the mesh"
    return path_matrix(bid, rank) @ mesh.root_bisector_vertices(h)


def decode_tri(bid: int, rank: int, he_next, he_vert, positions) -> np.ndarray:
    """Scalar restatement of the device decode (same operation order).

    Mirrors bisector.py:100-183 of the reference: the 3x3 matrix is updated
    per path bit as ``M <- M @ M1`` / ``M @ M0`` written out per entry, the
    apex is the face mean accumulated along ``next``, and each output
    coordinate is ``(m0*r0 + m1*r1) + m2*r2`` with no fused multiply-add.
    Python floats are IEEE doubles, so this is bit-identical to the kernels.
    """
    bid = int(bid)
    d = bid.bit_length() - 1 - rank
    root = bid >> d
    m = [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    h = bid
    while h != root:
        for r in range(3):
            a, b, c = m[r]
            if h & 1:
                m[r] = [0.5 * c, b + 0.5 * c, a]
            else:
                m[r] = [a + 0.5 * c, 0.5 * c, b]
        h >>= 1
    he = root - (1 << rank)
    nxt = int(he_next[he])
    r0 = [float(positions[he_vert[he], k]) for k in range(3)]
    r1 = [float(positions[he_vert[nxt], k]) for k in range(3)]
    acc = list(r0)
    n = 1
    w = nxt
    while w != he:
        for k in range(3):
            acc[k] += float(positions[he_vert[w], k])
        n += 1
        w = int(he_next[w])
    r2 = [acc[k] / n for k in range(3)]
    out = np.empty((3, 3), dtype=np.float64)
    for r in range(3):
        for k in range(3):
            out[r, k] = m[r][0] * r0[k] + m[r][1] * r1[k] + m[r][2] * r2[k]
    return out
