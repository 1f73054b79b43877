"""CPU: the C oracle reproduces the digests that oracle/pin_against_reference.py
recorded from the REAL reference (every array, every frame).  This keeps the
oracle pinned on machines where /root/reference does not exist."""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import OraclePool, OracleVerdict
from paper_2407_02215_b200 import halfedge, workloads
from tests import workloads as tw
from tests.parity import GOLDEN, STAT_NAMES, digest, load_golden

ARRAYS = ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter",
          "cache_live", "cache_free", "nodes")


def check(name, mesh, depth, frames, verdict_of, max_depth=None, every=1, threads=1):
    rec = load_golden(name)
    assert rec["depth"] == depth and rec["H"] == mesh.n_halfedges
    assert len(rec["frames"]) == frames
    op = OraclePool(mesh, depth)
    if max_depth is not None:
        op.max_depth = max_depth
    for k in ARRAYS:
        assert digest(getattr(op, k)) == rec["init"][k], (name, "init", k)
    for f in range(frames):
        stats, _ = op.update(verdict_of(f, op), threads=threads)
        want = rec["frames"][f]
        assert dict(zip(STAT_NAMES, (int(x) for x in stats))) == want["stats"], (name, f)
        if f % every == 0 or f == frames - 1:
            for k in ARRAYS:
                assert digest(getattr(op, k)) == want[k], (name, f, k)


def test_pinned_marker_present():
    with open(os.path.join(GOLDEN, "PINNED.txt")) as fh:
        assert "pinned against reference cbtmesh" in fh.read()


def test_const_and_uniform_cases():
    check("quad_d16_uniform12", halfedge.single_quad(), 16, 18, lambda f, op: OracleVerdict.uniform(12))
    check("grid_d9_uniform2", halfedge.quad_grid(2, 2), 9, 3, lambda f, op: OracleVerdict.uniform(2))
    check("triangle_d4_splitall", halfedge.single_triangle(), 4, 6, lambda f, op: OracleVerdict.const(1))
    check("grid_d12_alternate", halfedge.quad_grid(2, 2), 12, 8, lambda f, op: OracleVerdict.const(1 + f % 2))
    check("dodeca_d9_keep", halfedge.dodecahedron(), 9, 2, lambda f, op: OracleVerdict.const(0))
    check("triangle_d4_depthlimit1", halfedge.single_triangle(), 4, 3,
          lambda f, op: OracleVerdict.const(1), max_depth=1)


@pytest.mark.parametrize("case", tw.SOUP_CASES, ids=lambda c: f"{c[0]}_d{c[1]}")
def test_soups(case):
    mesh_name, depth, seed, frames = case

    def verdict_of(f, op):
        sp, mp = tw.soup_schedule(f)
        return OracleVerdict.explicit_array(tw.random_verdicts(op.count(), seed, f, sp, mp))

    check(f"soup_{mesh_name}_d{depth}_s{seed}", tw.MESHES[mesh_name](), depth, frames, verdict_of)


def _lod(seq):
    prms = seq.params()
    return lambda f, op: OracleVerdict.lod(seq.mesh, prms[f])


def test_config2_cube_sphere_flyin():
    seq = workloads.cube_sphere_flyin(depth=20, frames=64)
    check("cube_sphere_flyin_d20", seq.mesh, 20, 64, _lod(seq), every=8, threads=oracle.max_threads())


def test_config3_stress_d20():
    seq = workloads.earth_sweep(depth=20, frames=64)
    check("earth_sweep_d20", seq.mesh, 20, 128, _lod(seq), every=16, threads=oracle.max_threads())


def test_threads_do_not_change_results():
    """The OpenMP stages (2, classifier, 9) are order independent: 1 thread and
    all threads give identical arrays."""
    seq = workloads.cube_sphere_flyin(depth=14, frames=12)
    a, b = OraclePool(seq.mesh, 14), OraclePool(seq.mesh, 14)
    v = _lod(seq)
    for f in range(12):
        sa, _ = a.update(v(f, a), threads=1)
        sb, _ = b.update(v(f, b), threads=max(2, oracle.max_threads()))
        assert (sa == sb).all()
    for k in ARRAYS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_cbt_vectors():
    with open(os.path.join(GOLDEN, "cbt_vectors.json")) as fh:
        vectors = json.load(fh)
    assert len(vectors) >= 40
    for v in vectors:
        n = 1 << v["depth"]
        packed = np.frombuffer(bytes.fromhex(v["leaves"]), dtype=np.uint8)
        nodes = np.zeros(2 * n, np.uint32)
        nodes[n:] = np.unpackbits(packed, bitorder="little")[:n]
        oracle.sum_reduce_nodes(nodes, v["depth"])
        assert digest(nodes) == v["nodes_digest"]
        assert oracle.decode_ones(nodes, n, v["ranks1"]).tolist() == v["slots1"]
        assert oracle.decode_zeros(nodes, n, v["ranks0"]).tolist() == v["slots0"]
        # linear-scan definition (reference tests/test_cbt.py:116-132)
        ones = np.flatnonzero(nodes[n:])
        zeros = np.flatnonzero(nodes[n:] == 0)
        assert [int(ones[r]) for r in v["ranks1"]] == v["slots1"]
        assert [int(zeros[r]) for r in v["ranks0"]] == v["slots0"]


def test_classifier_vectors():
    with open(os.path.join(GOLDEN, "classifier_vectors.json")) as fh:
        rec = json.load(fh)
    seq = workloads.cube_sphere_flyin(depth=16, frames=24)
    prms = seq.params()
    gold = np.load(os.path.join(GOLDEN, "prm_cube_sphere_d16.npz"))["prm"]
    assert np.array_equal(prms.view(np.uint64), gold.view(np.uint64))
    mesh = seq.mesh
    L = oracle.lib()
    for vec in rec["vectors"]:
        ids = np.array(vec["ids"], dtype=np.uint64)
        tri = oracle.decode_tris(ids, rec["rank"], mesh.next, mesh.vert, mesh.positions)
        assert digest(tri) == vec["tri_digest"]
        n = len(ids)
        order = np.arange(n, dtype=np.int32)
        out = np.zeros(n, np.int8)
        L.orc_verdict_lod(out.ctypes.data, order.ctypes.data, ids.ctypes.data, rec["rank"],
                          rec["max_depth"], np.ascontiguousarray(mesh.next).ctypes.data,
                          np.ascontiguousarray(mesh.vert).ctypes.data, mesh.positions.ctypes.data,
                          prms[vec["frame"]].ctypes.data, 0, n, 1)
        assert out.tolist() == vec["verdicts"]
