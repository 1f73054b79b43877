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


# -- the reference's array-level entry points (bisector.py:92-189) ------------------

def nb_depth_of(bid, rank) -> int:
    """Depth of ``bid`` below its root (bisector.py:92-97)."""
    return int(bid).bit_length() - 1 - int(rank)


def nb_decode_tri(bid, rank, he_next, he_vert, positions, out) -> None:
    """Same call shape as the reference's jitted scalar decode (bisector.py:100-183):
    writes the (3, 3) fp64 vertices of ``bid`` into ``out``.  Host mirror
    (:func:`decode_tri`, bit-identical to the device decode)."""
    out[...] = decode_tri(int(bid), int(rank), he_next, he_vert, positions)


def nb_decode_tris(ids, rank, he_next, he_vert, positions, out, start, end) -> None:
    """Batch decode ``out[start:end]`` (bisector.py:186-189) -- on the GPU
    (cbtm_decode_triangles) when a device is present, as every bulk decode of
    this package."""
    from . import _lib
    t = _lib.torch()
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64)[start:end])
    if ids.size == 0:
        return
    dev = _lib.require_cuda()
    L = _lib.load()
    H = len(he_next)
    d_next = _lib.to_device(np.asarray(he_next, np.int32), dev)
    d_vert = _lib.to_device(np.asarray(he_vert, np.int32), dev)
    d_pos = _lib.to_device(np.asarray(positions, np.float64), dev)
    d_roots = t.empty(H * 9, dtype=t.float64, device=dev)
    stream = _lib.stream_handle(dev)
    _lib.check(L.cbtm_root_triangles(_lib.ptr(d_next), _lib.ptr(d_vert), _lib.ptr(d_pos), H,
                                     _lib.ptr(d_roots), stream), "cbtm_root_triangles")
    d_ids = _lib.to_device(ids, dev)
    d_out = t.empty((ids.size, 3, 3), dtype=t.float64, device=dev)
    _lib.check(L.cbtm_decode_triangles(_lib.ptr(d_ids), ids.size, int(rank), _lib.ptr(d_roots),
                                       _lib.ptr(d_out), stream), "cbtm_decode_triangles")
    out[start:end] = _lib.to_host(d_out)


def decode_tris_host(ids, rank, he_next, he_vert, positions, dtype=np.float64) -> np.ndarray:
    """Vectorised host decode of many ids in ``dtype`` arithmetic ((n, 3, 3)).
    With float64 it performs the operations of :func:`decode_tri` per id; with
    float32 every matrix entry, product and sum is rounded to single precision
    (the 32-bit pipeline of the reference's precision study, bisector.py:192-260)."""
    ids = np.asarray(ids, dtype=np.uint64)
    n = ids.size
    rank = int(rank)
    f = np.dtype(dtype).type
    half = f(0.5)
    depth = np.array([int(b).bit_length() - 1 - rank for b in ids], dtype=np.int64)
    m = np.zeros((n, 3, 3), dtype=dtype)
    m[:, 0, 0] = m[:, 1, 1] = m[:, 2, 2] = f(1.0)
    h = ids.copy()
    for level in range(int(depth.max()) if n else 0):
        active = depth > level
        odd = (h & np.uint64(1)).astype(bool)
        a, b, c = m[:, :, 0].copy(), m[:, :, 1].copy(), m[:, :, 2].copy()
        hc = half * c
        new0 = np.where(odd[:, None], hc, a + hc)
        new1 = np.where(odd[:, None], b + hc, hc)
        new2 = np.where(odd[:, None], a, b)
        for col, new in enumerate((new0, new1, new2)):
            m[:, :, col] = np.where(active[:, None], new, m[:, :, col])
        h = np.where(active, h >> np.uint64(1), h)
    he = (h - np.uint64(1 << rank)).astype(np.int64)
    he_next = np.asarray(he_next, dtype=np.int64)
    he_vert = np.asarray(he_vert, dtype=np.int64)
    pos = np.asarray(positions, dtype=dtype)
    out = np.empty((n, 3, 3), dtype=dtype)
    apex_cache: dict[int, np.ndarray] = {}
    for i in range(n):
        e = int(he[i])
        if e not in apex_cache:
            acc = pos[he_vert[e]].copy()
            cnt = 1
            w = int(he_next[e])
            while w != e:
                acc = acc + pos[he_vert[w]]
                cnt += 1
                w = int(he_next[w])
            apex_cache[e] = acc / f(cnt)
        r0, r1, r2 = pos[he_vert[e]], pos[he_vert[he_next[e]]], apex_cache[e]
        mi = m[i]
        out[i] = (mi[:, 0:1] * r0[None, :] + mi[:, 1:2] * r1[None, :]) + mi[:, 2:3] * r2[None, :]
    return out
