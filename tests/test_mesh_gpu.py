"""GPU parity of the device mesh ingest (cbtm_mesh_from_polygons) against the host
restatement of the reference's ``halfedge.from_polygons`` (halfedge.py:158-212), which
tests/test_host_logic.py pins against the reference's own golden meshes."""

import numpy as np
import pytest

from paper_2407_02215_b200 import halfedge
from paper_2407_02215_b200.halfedge import MeshError, from_polygons, from_polygons_device

pytestmark = pytest.mark.gpu

FIELDS = ("twin", "next", "prev", "vert", "edge", "face")


def polygons_of(mesh):
    faces = [[] for _ in range(mesh.n_faces)]
    for h in range(mesh.n_halfedges):
        faces[int(mesh.face[h])].append(int(mesh.vert[h]))
    return mesh.positions, faces


def same(a, b):
    for k in FIELDS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert np.array_equal(a.positions, b.positions)


@pytest.mark.parametrize("name", ["triangle", "quad", "grid", "dodeca", "cube_sphere", "icosphere2", "open_strip"])
def test_builtin_meshes(name):
    mesh = {"triangle": halfedge.single_triangle, "quad": halfedge.single_quad,
            "grid": lambda: halfedge.quad_grid(7, 5), "dodeca": halfedge.dodecahedron,
            "cube_sphere": lambda: halfedge.cube_sphere(1.0),
            "icosphere2": lambda: halfedge.icosphere(1.0, 2),
            "open_strip": lambda: halfedge.quad_grid(40, 1)}[name]()
    pos, faces = polygons_of(mesh)
    same(from_polygons(pos, faces), from_polygons_device(pos, faces))
    assert not halfedge.validate(from_polygons_device(pos, faces))


def test_large_mixed_polygon_mesh_and_csr_input():
    """A 300 x 200 grid whose cells are split at random into two triangles or
    kept as quads (mixed loop lengths, boundary, ~200 k halfedges), vertices
    randomly renumbered so that the edge numbering is not the face order."""
    rng = np.random.default_rng(7)
    nx, ny = 300, 200
    perm = rng.permutation((nx + 1) * (ny + 1))
    vid = lambda i, j: int(perm[j * (nx + 1) + i])  # noqa: E731
    faces = []
    for j in range(ny):
        for i in range(nx):
            a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            r = rng.integers(3)
            if r == 0:
                faces.append([a, b, c, d])
            elif r == 1:
                faces += [[a, b, c], [a, c, d]]
            else:
                faces += [[a, b, d], [b, c, d]]
    pos = rng.random(((nx + 1) * (ny + 1), 3))
    host = from_polygons(pos, faces)
    same(host, from_polygons_device(pos, faces))
    offsets = np.concatenate([[0], np.cumsum([len(f) for f in faces])]).astype(np.int32)
    verts = np.concatenate([np.asarray(f, np.int32) for f in faces])
    same(host, from_polygons_device(pos, (offsets, verts)))


@pytest.mark.parametrize("faces,what", [
    ([[0, 1, 2], [0, 1, 3], [0, 1, 4]], "non-manifold"),   # three faces on edge (0, 1)
    ([[0, 1, 2], [0, 1, 3]], "winding"),                    # both traverse 0 -> 1
    ([[0, 1, 1]], "degenerate"),
    ([[0, 1, 0, 1]], "degenerate"),
    ([[0, 1, 9]], "vertex"),
])
def test_rejections_match_the_host_builder(faces, what):
    pos = np.zeros((5, 3))
    with pytest.raises(MeshError):
        from_polygons(pos, faces)
    with pytest.raises(MeshError, match=what):
        from_polygons_device(pos, faces)


def test_device_built_mesh_drives_an_update():
    """End to end: ingest on the device, initialize, subdivide; same pool as with the host builder."""
    from paper_2407_02215_b200.pipeline import ParallelEngine, UniformSplit
    from paper_2407_02215_b200.state import initialize
    pos, faces = polygons_of(halfedge.icosphere(1.0, 1))
    a = initialize(from_polygons(pos, faces), 14)
    b = initialize(from_polygons_device(pos, faces), 14)
    with ParallelEngine() as eng:
        for e in range(4):
            sa, sb = eng.update(a, UniformSplit(3), epoch=e), eng.update(b, UniformSplit(3), epoch=e)
            assert sa.live_after == sb.live_after
    ha, hb = a.to_host(), b.to_host()
    for k in ha:
        assert np.array_equal(ha[k], hb[k]), k


def test_device_ingest_rejects_malformed_csr_before_any_launch():
    """Caller-supplied CSR offsets index device arrays directly: non-monotonic or mis-sized
    offsets are rejected on the host with MeshError."""
    import pytest
    from paper_2407_02215_b200.halfedge import MeshError, from_polygons_device
    pts = np.array([[0.0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]])
    verts = np.array([0, 1, 2, 0, 2, 3], dtype=np.int32)
    good = from_polygons_device(pts, (np.array([0, 3, 6], dtype=np.int32), verts))
    assert good.n_halfedges == 6
    for offsets in ([0, 4, 3, 6], [1, 3, 6], [0, 3, 7], [0, 3, 5], [0]):
        with pytest.raises(MeshError):
            from_polygons_device(pts, (np.array(offsets, dtype=np.int32), verts))
