"""CPU: host-side mirrors of the reference interface (meshes, ids, camera/LOD
parameters).  Known answers follow the reference's own tests
(pkg/tests/test_halfedge.py, test_bisector.py, test_lod.py)."""

import math
import os

import numpy as np
import pytest

from paper_2407_02215_b200 import bisector, halfedge, lod, workloads
from paper_2407_02215_b200.pipeline import (CSV_HEADER, EpochFactory, ParallelEngine,
                                            UpdateStats, converged_epoch, write_stats_csv)
from tests.parity import GOLDEN


# -- halfedge ------------------------------------------------------------------

def test_builtin_meshes_are_sound():
    for mesh, H, V, border in ((halfedge.single_triangle(), 3, 3, 3),
                               (halfedge.single_quad(), 4, 4, 4),
                               (halfedge.quad_grid(2, 2), 16, 9, 8),
                               (halfedge.dodecahedron(), 60, 20, 0),
                               (halfedge.cube_sphere(), 24, 8, 0),
                               (halfedge.icosphere(), 240, 42, 0)):
        assert halfedge.validate(mesh) == []
        st = mesh.stats()
        assert (st["H"], st["V"], st["boundary_halfedges"]) == (H, V, border)
    assert halfedge.dodecahedron().stats()["max_degree"] == 5
    ico = halfedge.icosphere()
    assert np.allclose(np.linalg.norm(ico.positions, axis=1), workloads.EARTH_RADIUS)


def test_planets_face_outward():
    for mesh in (halfedge.cube_sphere(1.0), halfedge.icosphere(1.0)):
        vol = 0.0
        for h in range(mesh.n_halfedges):
            if mesh.face[h] != mesh.face[mesh.prev[h]] or h == 0 or mesh.face[h] != mesh.face[h - 1]:
                loop = mesh._face_loop(h)
                p = mesh.positions[mesh.vert[loop]]
                for i in range(1, len(loop) - 1):
                    vol += np.linalg.det(np.stack([p[0], p[i], p[i + 1]]))
        assert vol > 0


def test_from_polygons_rejections():
    pts = [[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [2, 0, 0]]
    with pytest.raises(halfedge.MeshError):
        halfedge.from_polygons(pts, [[0, 1, 1]])                     # degenerate
    with pytest.raises(halfedge.MeshError):
        halfedge.from_polygons(pts, [[0, 1, 9]])                     # bad vertex index
    with pytest.raises(halfedge.MeshError):
        halfedge.from_polygons(pts, [[0, 1, 2], [0, 1, 3]])          # same direction twice
    with pytest.raises(halfedge.MeshError):
        halfedge.from_polygons(pts, [[0, 1, 2], [1, 0, 3], [0, 1, 4]])  # non-manifold
    with pytest.raises(halfedge.MeshError):
        halfedge.from_polygons(pts[:2], [[0, 1]])


def test_validate_reports_broken_operators():
    mesh = halfedge.quad_grid(2, 1)
    mesh.twin[int(np.flatnonzero(mesh.twin >= 0)[0])] = 0
    assert halfedge.validate(mesh)
    mesh = halfedge.single_quad()
    mesh.prev[2] = 0
    kinds = {v.operator for v in halfedge.validate(mesh)}
    assert "prev(next(h)) = h" in kinds or "next(prev(h)) = h" in kinds


def test_obj_roundtrip_and_errors():
    mesh = halfedge.dodecahedron()
    again = halfedge.load_obj(halfedge.write_obj_text(mesh))
    for k in ("twin", "next", "prev", "vert", "edge", "face"):
        assert np.array_equal(getattr(mesh, k), getattr(again, k))
    assert np.array_equal(mesh.positions, again.positions)
    rel = halfedge.parse_obj("v 0 0 0\nv 1 0 0\nv 0 1 0\nf -3 -2 -1\n")
    assert rel.n_halfedges == 3
    for bad in ("v 0 0\nf 1 2 3\n", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n", "v 0 0 0\n",
                "v 0 0 0\nv 1 0 0\nf 1 2\n"):
        with pytest.raises(halfedge.MeshError):
            halfedge.parse_obj(bad)


def test_root_bisector_vertices():
    quad = halfedge.single_quad()
    tri = quad.root_bisector_vertices(1)
    assert np.allclose(tri, [[1, 0, 0], [1, 1, 0], [0.5, 0.5, 0]])
    with pytest.raises(IndexError):
        quad.root_bisector_vertices(4)


# -- bisector ids -----------------------------------------------------------------

def test_id_helpers():
    assert bisector.root_rank(12) == 4 and bisector.make_root_id(12, 7) == 23
    assert bisector.root_rank(1) == 1 and bisector.root_rank(2) == 1 and bisector.root_rank(3) == 2
    assert bisector.max_depth(60) == 57
    assert bisector.depth_of(23, 4) == 0 and bisector.depth_of(23 * 8 + 5, 4) == 3
    assert bisector.root_halfedge(23 * 8 + 5, 4) == 7
    assert bisector.children(23) == (46, 47) and bisector.parent(47) == 23
    with pytest.raises(OverflowError):
        bisector.children(1 << 63)
    with pytest.raises(ValueError):
        bisector.make_root_id(12, 12)


def test_decode_matches_matrix_product_and_halves_area():
    mesh = halfedge.dodecahedron()
    rank = bisector.root_rank(60)
    rng = np.random.default_rng(0)
    for _ in range(50):
        bid = bisector.make_root_id(60, int(rng.integers(60)))
        for _ in range(int(rng.integers(0, 30))):
            bid = 2 * bid + int(rng.integers(2))
        a = bisector.bisector_vertices(mesh, bid)
        b = bisector.decode_tri(bid, rank, mesh.next, mesh.vert, mesh.positions)
        assert np.allclose(a, b, rtol=0, atol=1e-12)
    assert abs(np.linalg.det(bisector.M0) + 0.5) < 1e-15 and abs(np.linalg.det(bisector.M1) + 0.5) < 1e-15


# -- camera / LOD -----------------------------------------------------------------

def test_camera_validation_and_basis():
    cam = lod.Camera([0, 0, 5], [0, 0, -2], [0.1, 1, 0.3])
    assert abs(np.linalg.norm(cam.forward) - 1) < 1e-15 and abs(cam.forward @ cam.up) < 1e-12
    assert np.allclose(cam.right, np.cross(cam.forward, cam.up))
    with pytest.raises(ValueError):
        lod.Camera([0, 0, 0], [0, 0, 1], [0, 0, 2])
    with pytest.raises(ValueError):
        lod.Camera([0, 0, 0], [0, 0, 1], [0, 1, 0], fov_y=4.0)
    with pytest.raises(ValueError):
        lod.Camera([0, 0, 0], [0, 0, 1], [0, 1, 0], width=0)


def test_lod_config_validation():
    for kw in ({"split_factor": 1.0}, {"merge_factor": 1.0}, {"merge_factor": 0.0},
               {"split_factor": 1.5, "merge_factor": 0.8}):
        with pytest.raises(ValueError):
            lod.LodConfig(**kw)
    cfg = lod.LodConfig.from_json('{"target_area_px": 25.0, "planet_mode": true}')
    assert cfg.target_area_px == 25.0 and cfg.planet_mode


def test_known_screen_area_and_frustum():
    # a 10 x 10 px right triangle straight ahead: area 50 px (reference test_lod.py:72-77)
    cam = lod.Camera([0, 0, 0], [0, 0, 1], [0, 1, 0], fov_y=math.radians(90), width=200, height=200)
    z = 10.0
    s = z / cam.focal_px
    tri = np.array([[0, 0, z], [10 * s, 0, z], [0, 10 * s, z]])
    assert abs(lod.screen_space_area(cam, tri) - 50.0) < 1e-9
    assert not lod.outside_frustum(cam, tri)
    assert lod.outside_frustum(cam, tri - np.array([0, 0, 2 * z]))       # behind
    assert lod.outside_frustum(cam, tri + np.array([5 * z, 0, 0]))       # off to one side


def test_decide_thresholds_on_flat_mesh():
    mesh = halfedge.single_quad()
    cfg = lod.LodConfig(target_area_px=100.0)
    near = lod.Camera([0.5, 0.5, 1.0], [0, 0, -1], [0, 1, 0])
    far = lod.Camera([0.5, 0.5, 5000.0], [0, 0, -1], [0, 1, 0])
    away = lod.Camera([0.5, 0.5, 1.0], [0, 0, 1], [0, 1, 0])
    root = bisector.make_root_id(4, 0)
    assert lod.decide(cfg, near, mesh, root) == lod.SPLIT
    assert lod.decide(cfg, far, mesh, root) == lod.MERGE
    assert lod.decide(cfg, away, mesh, root) == lod.MERGE      # culled


def test_camera_paths():
    keys = lod.make_zoom_path(100.0, 300.0, 1.0)
    assert len(keys) == 25 and keys[0].t == 0.0 and keys[-1].t == 1.0
    assert np.allclose(keys[0].position, [400.0, 0, 0]) and np.allclose(keys[-1].position, [101.0, 0, 0])
    mid = lod.camera_path_at(keys, 0.5)
    assert abs(mid.position[0] - (100 + 300 * (1 / 300) ** 0.5)) < 1e-9
    assert np.allclose(lod.camera_path_at(keys, -1).position, keys[0].position)
    assert np.allclose(lod.camera_path_at(keys, 9).position, keys[-1].position)
    again = lod.load_camera_path(lod.dump_camera_path(keys))
    assert all(np.allclose(a.position, b.position) for a, b in zip(keys, again))
    with pytest.raises(ValueError):
        lod.load_camera_path("[]")
    with pytest.raises(ValueError):
        lod.camera_path_at([], 0.0)
    assert len(lod.sample_path(keys, 64)) == 64


def test_golden_camera_parameters():
    """prm vectors of configs 2 and 3 are bit-identical to the reference's."""
    for seq in (workloads.cube_sphere_flyin(), workloads.earth_sweep(depth=20)):
        gold = np.load(os.path.join(GOLDEN, f"prm_{seq.name}.npz"))["prm"]
        assert np.array_equal(seq.params().view(np.uint64), gold.view(np.uint64)), seq.name


def test_predicted_live_count_is_positive_and_capped():
    cfg = workloads.planet_config()
    cams = lod.sample_path(lod.make_zoom_path(cfg.planet_radius, 3 * cfg.planet_radius, 1000.0), 8)
    vals = [lod.predicted_live_count(cfg, c) for c in cams]
    assert all(v > 0 for v in vals) and max(vals) <= 2 * 1920 * 1080 / 49.0 + 1e-6


# -- stats plumbing ------------------------------------------------------------------

def test_stats_csv_and_convergence():
    a = UpdateStats(0, 16, 32, 16, 0, 0, 0, 32, 0, stage_times_us=[1] * 9)
    b = UpdateStats(1, 32, 32, 0, 0, 0, 0, 0, 0)
    text = write_stats_csv([a, b], no_timing=True)
    assert text.splitlines()[0] == CSV_HEADER
    assert text.splitlines()[1] == "0,16,32,16,0,0,0" + ",0" * 9
    assert write_stats_csv([a]).splitlines()[1].endswith(",1" * 9)
    assert converged_epoch([a, b]) == 1 and converged_epoch([a]) is None
    assert a.structural_ops == 16
    assert EpochFactory(lambda e: e * 2)(3) == 6 and EpochFactory.per_epoch
    with pytest.raises(ValueError):
        ParallelEngine(threads=0)
    words = [1, 2, 3, 4, 5, 6, 7, 8, 9, 10] + [0] * 22
    s = UpdateStats.from_device_words(words, 5)
    assert (s.epoch, s.live_before, s.live_after, s.splits_applied, s.merges_applied,
            s.splits_rejected_oom, s.merges_rejected_oom, s.split_allocs, s.merge_allocs) == \
        (5, 7, 8, 3, 4, 1, 2, 5, 6)


def test_bench_reference_arm_runs_on_cpu_and_prints_the_contract_line():
    """`bench.py --impl reference` (here: the C port only, a small pool) needs no GPU, runs on rank 0
    only, and prints ONE JSON line with the keys the driver reads."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = [sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--port-only", "--depth", "14",
            "--steps", "3", "--warmup", "3", "--gpus", "2"]
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run(base, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["unit"] == "bisectors/s" and line["higher_is_better"] is True
    assert line["steps"] == 3 and line["warmup"] == 3 and line["n_gpus"] == 2 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "bisectors/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["config"]["planets"] == 8 and line["scaling"] == "strong"          # N > 1: BASELINE config 5
    # every other rank of a torchrun launch exits 0 without work
    other = subprocess.run(base, cwd=root, env=dict(env, RANK="1", WORLD_SIZE="2"), capture_output=True, text=True, timeout=60)
    assert other.returncode == 0 and other.stdout.strip() == ""
