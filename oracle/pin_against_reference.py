#!/usr/bin/env python
"""Pin the C oracle against the real reference and write tests/golden/.

Runs ONLY in the build container (it imports the reference package from
/root/reference/pkg/src, which does not exist on the GPU box).  For every
workload it steps the reference's ``ParallelEngine(threads=1)`` and the C
oracle side by side, requires ALL state arrays to be identical after every
frame, and records per-frame digests (+ stats) as JSON fixtures that
tests/test_oracle_golden.py re-checks without the reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/pin_against_reference.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import cbtmesh  # noqa: E402  (the reference)
import cbtmesh.cbt as ref_cbt  # noqa: E402
from cbtmesh import bisector as ref_bisector  # noqa: E402
from cbtmesh import halfedge as ref_halfedge  # noqa: E402
from cbtmesh import lod as ref_lod  # noqa: E402
from cbtmesh import sequential as ref_sequential  # noqa: E402
from cbtmesh.pipeline import (KeepAll, MergeAll, ParallelEngine,  # noqa: E402
                              SplitAll, UniformSplit)

import oracle  # noqa: E402
from oracle import OraclePool, OracleVerdict  # noqa: E402
from paper_2407_02215_b200 import halfedge, lod, workloads  # noqa: E402
from tests import workloads as tw  # noqa: E402

GOLDEN = os.path.join(REPO, "tests", "golden")
STATE_ARRAYS = ("ids", "nexts", "prevs", "twins", "commands", "reserved",
                "counter", "cache_live", "cache_free")
STAT_NAMES = ("oom_splits", "oom_merges", "split_freed", "merge_freed",
              "split_alloc", "merge_alloc", "live_before", "live_after")


def digest(a: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(a).tobytes(),
                           digest_size=8).hexdigest()


def ref_mesh_of(mesh) -> ref_halfedge.HalfedgeMesh:
    """The same mesh as a reference object (arrays are identical by test)."""
    return ref_halfedge.HalfedgeMesh(mesh.twin, mesh.next, mesh.prev,
                                     mesh.vert, mesh.edge, mesh.face,
                                     mesh.positions)


def compare_states(st, op, tag) -> dict:
    out = {}
    for k in STATE_ARRAYS:
        a, b = getattr(st, k), getattr(op, k)
        if not np.array_equal(a, b):
            bad = np.flatnonzero((a != b).reshape(a.shape[0], -1).any(axis=1))
            raise SystemExit(f"MISMATCH {tag}: {k} differs at {bad[:8]} "
                             f"({bad.size} rows)")
        out[k] = digest(b)
    if not np.array_equal(st.cbt.nodes, op.nodes):
        raise SystemExit(f"MISMATCH {tag}: cbt.nodes")
    out["nodes"] = digest(op.nodes)
    return out


def stats_tuple(s) -> tuple:
    return (s.splits_rejected_oom, s.merges_rejected_oom, s.splits_applied,
            s.merges_applied, s.split_allocs, s.merge_allocs, s.live_before,
            s.live_after)


def run_case(name, mesh, depth, frames, ref_decide_of, orc_verdict_of,
             max_depth=None) -> dict:
    """Step both engines; returns the golden record."""
    if depth > ref_cbt.MAX_DEPTH:
        ref_cbt.MAX_DEPTH = 30
    st = ref_sequential.initialize(ref_mesh_of(mesh), depth)
    op = OraclePool(mesh, depth)
    if max_depth is not None:
        st.max_depth = max_depth
        op.max_depth = max_depth
    record = {"name": name, "depth": depth, "H": mesh.n_halfedges,
              "frames": [], "init": compare_states(st, op, f"{name}/init")}
    t0 = time.time()
    with ParallelEngine(threads=1) as eng:
        for f in range(frames):
            s = eng.update(st, ref_decide_of(f, st), epoch=f)
            o, _ = op.update(orc_verdict_of(f, op))
            if stats_tuple(s) != tuple(int(x) for x in o):
                raise SystemExit(f"MISMATCH {name}/{f}: stats {s} vs {o}")
            rec = compare_states(st, op, f"{name}/{f}")
            rec["stats"] = dict(zip(STAT_NAMES, (int(x) for x in o)))
            record["frames"].append(rec)
    ooms = sum(r["stats"]["oom_splits"] + r["stats"]["oom_merges"]
               for r in record["frames"])
    peak = max(r["stats"]["live_after"] for r in record["frames"])
    print(f"  {name}: {frames} frames identical, peak live {peak}, "
          f"oom rejections {ooms}, {time.time() - t0:.1f}s")
    return record


def save(record: dict) -> None:
    path = os.path.join(GOLDEN, record["name"] + ".json")
    with open(path, "w") as fh:
        json.dump(record, fh, indent=0, separators=(",", ":"))


# -- individual pins ---------------------------------------------------------

def pin_meshes():
    pairs = [
        (halfedge.single_triangle(), ref_halfedge.single_triangle()),
        (halfedge.single_quad(), ref_halfedge.single_quad()),
        (halfedge.quad_grid(2, 2), ref_halfedge.quad_grid(2, 2)),
        (halfedge.quad_grid(3, 5), ref_halfedge.quad_grid(3, 5)),
        (halfedge.dodecahedron(), ref_halfedge.dodecahedron()),
        (halfedge.dodecahedron(2.5), ref_halfedge.dodecahedron(2.5)),
    ]
    for mine, ref in pairs:
        for k in ("twin", "next", "prev", "vert", "edge", "face", "positions"):
            assert np.array_equal(getattr(mine, k), getattr(ref, k)), k
    for mesh in (halfedge.cube_sphere(), halfedge.icosphere()):
        assert ref_halfedge.validate(ref_mesh_of(mesh)) == []
        assert halfedge.validate(mesh) == []
    obj = halfedge.write_obj_text(halfedge.dodecahedron())
    assert obj == ref_halfedge.write_obj_text(ref_halfedge.dodecahedron())
    a, b = halfedge.load_obj(obj), ref_halfedge.load_obj(obj)
    assert np.array_equal(a.twin, b.twin) and np.array_equal(a.next, b.next)
    print("  meshes: builders identical to the reference; planets validate")


def pin_cbt():
    vectors = []
    rng = np.random.default_rng(20240702)
    for depth in list(range(1, 13)) + [16, 20]:
        n = 1 << depth
        for occ in (0.0, 0.03, 0.5, 0.97, 1.0):
            leaves = (rng.random(n) < occ).astype(np.uint32)
            ref_nodes = np.zeros(2 * n, np.uint32)
            ref_nodes[n:] = leaves
            mine = ref_nodes.copy()
            ref_cbt.sum_reduce_array(ref_nodes, depth)
            oracle.sum_reduce_nodes(mine, depth)
            assert np.array_equal(ref_nodes, mine), (depth, occ)
            ones = int(ref_nodes[1])
            k = min(ones, 4096)
            ranks1 = np.sort(rng.choice(ones, k, replace=False)) if ones else np.zeros(0, np.int64)
            k0 = min(n - ones, 4096)
            ranks0 = np.sort(rng.choice(n - ones, k0, replace=False)) if n - ones else np.zeros(0, np.int64)
            out_ref = np.zeros(k, np.int64)
            ref_cbt.nb_one_to_bit_ids(ref_nodes, n, ranks1.astype(np.int64), out_ref, 0, k)
            assert np.array_equal(out_ref, oracle.decode_ones(mine, n, ranks1))
            out_ref0 = np.zeros(k0, np.int64)
            ref_cbt.nb_zero_to_bit_ids(ref_nodes, n, ranks0.astype(np.int64), out_ref0, 0, k0)
            assert np.array_equal(out_ref0, oracle.decode_zeros(mine, n, ranks0))
            if depth <= 10:
                vectors.append({
                    "depth": depth, "occ": occ,
                    "leaves": np.packbits(leaves.astype(np.uint8), bitorder="little").tobytes().hex(),
                    "nodes_digest": digest(mine),
                    "ranks1": ranks1[:64].tolist(), "slots1": out_ref[:64].tolist(),
                    "ranks0": ranks0[:64].tolist(), "slots0": out_ref0[:64].tolist(),
                })
    # the reference's own worked example, tests/test_cbt.py:56-69
    c = cbtmesh.Cbt(4)
    for s in (0, 3, 10):
        c.set_bit(s, 1)
    c.sum_reduce()
    assert [c.one_to_bit_id(r) for r in range(3)] == [0, 3, 10]
    assert c.zero_to_bit_id(0) == 1
    assert oracle.decode_ones(c.nodes, 16, [0, 1, 2]).tolist() == [0, 3, 10]
    assert oracle.decode_zeros(c.nodes, 16, [0]).tolist() == [1]
    with open(os.path.join(GOLDEN, "cbt_vectors.json"), "w") as fh:
        json.dump(vectors, fh, separators=(",", ":"))
    print(f"  cbt: reduce + ranked decode identical (14 depths x 5 occupancies);"
          f" {len(vectors)} vectors saved")


def pin_classifier():
    """decode_tri and the LOD verdicts on ids harvested from real runs."""
    seq = workloads.cube_sphere_flyin(depth=16, frames=24)
    mesh = seq.mesh
    rmesh = ref_mesh_of(mesh)
    prms = seq.params()
    st = ref_sequential.initialize(rmesh, 16)
    harvested = []
    with ParallelEngine(threads=1) as eng:
        for f, cam in enumerate(seq.cameras):
            rcam = ref_lod.Camera(cam.position, cam.forward, cam.up, cam.fov_y,
                                  cam.width, cam.height, cam.near)
            rcfg = ref_lod.LodConfig(planet_mode=True, planet_radius=workloads.EARTH_RADIUS)
            dec = ref_lod.LodDecide(rcfg, rcam, rmesh)
            assert np.array_equal(dec._prm, prms[f]), f"prm differs at frame {f}"
            eng.update(st, dec, epoch=f)
            live = st.ids[st.live_slots()]
            harvested.append((f, live.copy()))
    rank = st.rank
    total = 0
    vec = []
    for f, ids in harvested[::3]:
        ref_tri = np.empty((len(ids), 3, 3))
        ref_bisector.nb_decode_tris(ids, rank, rmesh.next, rmesh.vert, rmesh.positions, ref_tri, 0, len(ids))
        mine = oracle.decode_tris(ids, rank, mesh.next, mesh.vert, mesh.positions)
        assert np.array_equal(ref_tri.view(np.uint64), mine.view(np.uint64)), "decode_tri bits"
        # verdicts through the reference kernel vs the oracle kernel
        n = len(ids)
        order = np.arange(n, dtype=np.int32)
        v_ref = np.zeros(n, np.int8)
        ref_lod._k_verdict_lod(v_ref, order, ids, rank, np.int64(st.max_depth), rmesh.next,
                               rmesh.vert, rmesh.positions, prms[f], 0, n)
        v_orc = np.zeros(n, np.int8)
        L = oracle.lib()
        ids_c = np.ascontiguousarray(ids)
        L.orc_verdict_lod(v_orc.ctypes.data, order.ctypes.data, ids_c.ctypes.data, rank, st.max_depth,
                          np.ascontiguousarray(mesh.next).ctypes.data,
                          np.ascontiguousarray(mesh.vert).ctypes.data,
                          mesh.positions.ctypes.data, prms[f].ctypes.data, 0, n, 1)
        assert np.array_equal(v_ref, v_orc), f"lod verdicts differ at frame {f}"
        total += n
        pick = np.linspace(0, n - 1, min(n, 96)).astype(np.int64)
        vec.append({"frame": f, "ids": [int(x) for x in ids[pick]],
                    "verdicts": v_ref[pick].tolist(),
                    "tri_digest": digest(ref_tri[pick])})
    np.savez_compressed(os.path.join(GOLDEN, "prm_cube_sphere_d16.npz"), prm=prms)
    with open(os.path.join(GOLDEN, "classifier_vectors.json"), "w") as fh:
        json.dump({"rank": rank, "max_depth": int(st.max_depth), "vectors": vec}, fh,
                  separators=(",", ":"))
    print(f"  classifier: decode_tri bit-identical and verdicts identical on {total} ids")


def pin_camera_params():
    for seq in (workloads.cube_sphere_flyin(), workloads.earth_sweep(depth=20)):
        rmesh = ref_mesh_of(seq.mesh)
        if seq.name == "cube_sphere_flyin":
            keys = ref_lod.make_zoom_path(workloads.EARTH_RADIUS, 3 * workloads.EARTH_RADIUS, 1000.0)
        else:
            keys = ref_lod.make_zoom_path(workloads.EARTH_RADIUS, 3 * workloads.EARTH_RADIUS, 10.0)
        n = 64
        cams = []
        t0, t1 = keys[0].t, keys[-1].t
        for i in range(n):  # cli.py:227-231
            t = t0 + (t1 - t0) * i / (n - 1)
            cams.append(ref_lod.camera_path_at(keys, t, 1920, 1080))
        if seq.name == "earth_sweep":
            cams = cams + cams[::-1]
        rcfg = ref_lod.LodConfig(planet_mode=True, planet_radius=workloads.EARTH_RADIUS)
        ref_prm = np.stack([ref_lod.LodDecide(rcfg, c, rmesh)._prm for c in cams])
        assert np.array_equal(ref_prm.view(np.uint64), seq.params().view(np.uint64)), seq.name
        np.savez_compressed(os.path.join(GOLDEN, f"prm_{seq.name}.npz"), prm=ref_prm)
    print("  camera paths: per-frame parameter vectors bit-identical")


def explicit_pair(frame_verdicts):
    """(ref decide factory, oracle verdict factory) for explicit verdicts in
    cache_live order; the reference receives them as an id -> verdict map."""
    def ref_decide_of(f, st):
        ids = st.ids[np.flatnonzero(st.cbt.leaves)]
        v = frame_verdicts(f, len(ids))
        table = {int(i): int(x) for i, x in zip(ids, v)}
        return lambda bid: table[bid]

    def orc_verdict_of(f, op):
        return OracleVerdict.explicit_array(frame_verdicts(f, op.count()))
    return ref_decide_of, orc_verdict_of


def pin_frames():
    # config 1: quad, D=16, UniformSplit(12) until 16384 live (18 frames)
    rec = run_case("quad_d16_uniform12", halfedge.single_quad(), 16, 18,
                   lambda f, st: UniformSplit(12),
                   lambda f, op: OracleVerdict.uniform(12))
    assert rec["frames"][-1]["stats"]["live_after"] == 16384
    save(rec)

    # the reference's CSV known answer: grid 2x2, UniformSplit(2), first row
    rec = run_case("grid_d9_uniform2", halfedge.quad_grid(2, 2), 9, 3,
                   lambda f, st: UniformSplit(2),
                   lambda f, op: OracleVerdict.uniform(2))
    s0 = rec["frames"][0]["stats"]
    assert (s0["live_before"], s0["live_after"], s0["split_freed"]) == (16, 32, 16)
    save(rec)

    # const verdict sources incl. OOM at capacity 16 and split/merge alternation
    consts = [SplitAll, MergeAll]
    rec = run_case("triangle_d4_splitall", halfedge.single_triangle(), 4, 6,
                   lambda f, st: SplitAll(), lambda f, op: OracleVerdict.const(1))
    save(rec)
    rec = run_case("grid_d12_alternate", halfedge.quad_grid(2, 2), 12, 8,
                   lambda f, st: consts[f % 2](),
                   lambda f, op: OracleVerdict.const(1 + f % 2))
    save(rec)
    rec = run_case("dodeca_d9_keep", halfedge.dodecahedron(), 9, 2,
                   lambda f, st: KeepAll(), lambda f, op: OracleVerdict.const(0))
    save(rec)
    rec = run_case("triangle_d4_depthlimit1", halfedge.single_triangle(), 4, 3,
                   lambda f, st: SplitAll(), lambda f, op: OracleVerdict.const(1),
                   max_depth=1)
    save(rec)

    # random split/merge soups under reservation pressure (explicit verdicts)
    for mesh_name, depth, seed, frames in tw.SOUP_CASES:
        def fv(f, n, seed=seed):
            sp, mp = tw.soup_schedule(f)
            return tw.random_verdicts(n, seed, f, sp, mp)
        r, o = explicit_pair(fv)
        save(run_case(f"soup_{mesh_name}_d{depth}_s{seed}", tw.MESHES[mesh_name](),
                      depth, frames, r, o))

    # config 2: cube-sphere fly-in, D=20, 64 frames (LOD classifier)
    def lod_pair(seq):
        rmesh = ref_mesh_of(seq.mesh)
        rcfg = ref_lod.LodConfig(planet_mode=True, planet_radius=workloads.EARTH_RADIUS)
        prms = seq.params()

        def ref_decide_of(f, st):
            c = seq.cameras[f]
            rc = ref_lod.Camera(c.position, c.forward, c.up, c.fov_y, c.width, c.height, c.near)
            return ref_lod.LodDecide(rcfg, rc, rmesh)

        def orc_verdict_of(f, op):
            return OracleVerdict.lod(seq.mesh, prms[f])
        return ref_decide_of, orc_verdict_of

    seq = workloads.cube_sphere_flyin(depth=20, frames=64)
    r, o = lod_pair(seq)
    save(run_case("cube_sphere_flyin_d20", seq.mesh, 20, seq.n_frames, r, o))

    # config 3 at D=20: descent + ascent, heavy reservation pressure (stress)
    seq = workloads.earth_sweep(depth=20, frames=64)
    r, o = lod_pair(seq)
    save(run_case("earth_sweep_d20", seq.mesh, 20, seq.n_frames, r, o))

    # config 3, D=22, shortened (16 + 16 frames): a no-pressure large-pool run
    seq = workloads.earth_sweep(depth=22, frames=16)
    r, o = lod_pair(seq)
    save(run_case("earth_sweep_d22_short", seq.mesh, 22, seq.n_frames, r, o))


def main():
    os.makedirs(GOLDEN, exist_ok=True)
    print("pinning oracle against reference", cbtmesh.__version__)
    # warm the reference's JIT like its conftest does (tests/conftest.py:10-17)
    st = ref_sequential.initialize(ref_halfedge.single_triangle(), 5)
    with ParallelEngine(threads=1) as eng:
        eng.update(st, KeepAll())
    pin_meshes()
    pin_cbt()
    pin_classifier()
    pin_camera_params()
    pin_frames()
    with open(os.path.join(GOLDEN, "PINNED.txt"), "w") as fh:
        fh.write("oracle pinned against reference cbtmesh "
                 f"{cbtmesh.__version__} (numpy {np.__version__}); "
                 "regenerate with oracle/pin_against_reference.py\n")
    print("all pins passed; fixtures written to tests/golden/")


if __name__ == "__main__":
    main()
