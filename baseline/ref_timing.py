"""Timing of the REAL reference (`cbtmesh` from baseline/_ref, unmodified) on this box's host
cores, beside the GPU path.  Method of the reference's own `cmd_bench`
(pkg/src/cbtmesh/cli.py:263-308): kernels JIT-warmed first, `time.perf_counter_ns` around
`ParallelEngine.update`, per-frame list -> median and total.

Used only by bench.py (cpu_baseline kind "reference" / `--impl reference`).  The product
package never imports this; nothing here touches the GPU.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_ROOT = os.path.join(HERE, "_ref")
RECORD_ARRAYS = ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter",
                 "cache_live", "cache_free")


def available() -> bool:
    return os.path.exists(os.path.join(REF_ROOT, "cbtmesh", "__init__.py"))


def load():
    """Import the reference package (numba JIT cache in a writable directory next to it)."""
    if not available():
        raise RuntimeError("baseline/_ref/cbtmesh is missing: run `python baseline/install_ref.py` "
                           "where /root/reference exists")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(REF_ROOT, ".numba_cache"))
    if REF_ROOT not in sys.path:
        sys.path.insert(0, REF_ROOT)
    import cbtmesh  # noqa: F401
    import cbtmesh.cbt as ref_cbt
    ref_cbt.MAX_DEPTH = 30      # the reference caps D at 25 (cbt.py:16-28); uint32 counters are safe to 31
    return cbtmesh


def ref_mesh_of(mesh):
    from cbtmesh import halfedge as ref_halfedge
    return ref_halfedge.HalfedgeMesh(mesh.twin, mesh.next, mesh.prev, mesh.vert, mesh.edge, mesh.face,
                                     mesh.positions)


def ref_camera_of(cam):
    from cbtmesh import lod as ref_lod
    return ref_lod.Camera(cam.position, cam.forward, cam.up, cam.fov_y, cam.width, cam.height, cam.near)


def ref_config_of(cfg):
    from cbtmesh import lod as ref_lod
    return ref_lod.LodConfig(target_area_px=cfg.target_area_px, split_factor=cfg.split_factor,
                             merge_factor=cfg.merge_factor, frustum_cull=cfg.frustum_cull,
                             planet_mode=cfg.planet_mode, planet_radius=cfg.planet_radius)


def warm_jit(threads: int) -> float:
    """Compile / load every jitted kernel once (conftest.warm_kernels + the LOD classifier)."""
    t0 = time.perf_counter()
    from cbtmesh import halfedge as ref_halfedge, lod as ref_lod, sequential as ref_seq
    from cbtmesh.pipeline import KeepAll, ParallelEngine
    mesh = ref_halfedge.dodecahedron()
    st = ref_seq.initialize(mesh, 10)
    cfg = ref_lod.LodConfig(planet_mode=True, planet_radius=0.9)
    cam = ref_lod.Camera([3.0, 0.4, 0.2], [-1, 0, 0], [0, 0, 1], width=256, height=256)
    for t in sorted({1, threads}):
        with ParallelEngine(threads=t) as eng:
            eng.update(st, KeepAll())
            eng.update(st, lambda bid: 0)
            for _ in range(3):
                eng.update(st, ref_lod.LodDecide(cfg, cam, mesh))
    return time.perf_counter() - t0


def state_from_arrays(mesh, depth: int, arrays: dict):
    """A reference TriangulationState holding the given pool (reference layout: the record
    arrays + `nodes`, the uint32[2N] heap)."""
    from cbtmesh import state as ref_state
    st = ref_state.TriangulationState(ref_mesh_of(mesh), depth)
    for k in RECORD_ARRAYS:
        getattr(st, k)[...] = arrays[k]
    st.cbt.nodes[...] = arrays["nodes"]
    return st


def time_frames(st, mesh, config, cameras, threads: int):
    """Run one update per camera on `st`; returns (seconds per frame list, stats rows)."""
    from cbtmesh import lod as ref_lod
    from cbtmesh.pipeline import ParallelEngine
    rmesh = st.mesh
    rcfg = ref_config_of(config)
    per_frame, rows = [], []
    with ParallelEngine(threads=threads) as eng:
        for f, cam in enumerate(cameras):
            decide = ref_lod.LodDecide(rcfg, ref_camera_of(cam), rmesh)
            t0 = time.perf_counter_ns()
            s = eng.update(st, decide, epoch=f)
            per_frame.append((time.perf_counter_ns() - t0) * 1e-9)
            rows.append([s.splits_rejected_oom, s.merges_rejected_oom, s.splits_applied, s.merges_applied,
                         s.split_allocs, s.merge_allocs, s.live_before, s.live_after])
    return per_frame, rows


def clone_state(st):
    return st.clone()
