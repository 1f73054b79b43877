"""Named workloads of BASELINE.json: meshes + camera sequences.

Pure host-side description shared by bench.py, the parity tests and the
oracle pinning script, so that every arm runs exactly the same input.  Nothing
here touches the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import halfedge, lod

EARTH_RADIUS = 6.371e6


@dataclass
class LodSequence:
    """A mesh, a pool depth and one 23-double parameter vector per frame."""

    name: str
    mesh: halfedge.HalfedgeMesh
    depth: int
    config: lod.LodConfig
    cameras: list = field(default_factory=list)

    @property
    def n_frames(self) -> int:
        return len(self.cameras)

    def params(self) -> np.ndarray:
        """float64[n_frames, 23] classifier parameters, frame by frame."""
        return np.stack([lod.pack_lod_params(self.config, c)
                         for c in self.cameras])


def planet_config() -> lod.LodConfig:
    return lod.LodConfig(planet_mode=True, planet_radius=EARTH_RADIUS)


def cube_sphere_flyin(depth: int = 20, frames: int = 64) -> LodSequence:
    """Config 2: cube-sphere planet, 3R -> 1000 m zoom, 1920x1080."""
    keys = lod.make_zoom_path(EARTH_RADIUS, 3.0 * EARTH_RADIUS, 1000.0)
    return LodSequence("cube_sphere_flyin", halfedge.cube_sphere(EARTH_RADIUS),
                       depth, planet_config(), lod.sample_path(keys, frames))


def earth_sweep(depth: int = 26, frames: int = 64, rotate_deg: float = 0.0,
                mesh=None) -> LodSequence:
    """Config 3: coarse icosphere (H=240); `frames` samples descending from
    3R to 10 m altitude (warm-up), then the same samples in reverse (the
    ground-to-space sweep): 2*frames frames in total."""
    keys = lod.make_zoom_path(EARTH_RADIUS, 3.0 * EARTH_RADIUS, 10.0)
    down = lod.sample_path(keys, frames)
    cams = down + down[::-1]
    if rotate_deg:
        cams = [lod.rotate_z(c, rotate_deg) for c in cams]
    return LodSequence("earth_sweep", mesh or halfedge.icosphere(EARTH_RADIUS, 1),
                       depth, planet_config(), cams)


def planet_batch(n_planets: int = 8, depth: int = 24,
                 frames: int = 64) -> list[LodSequence]:
    """Config 5: independent planets, planet p's path rotated by p*45 deg."""
    mesh = halfedge.icosphere(EARTH_RADIUS, 1)
    return [earth_sweep(depth, frames, rotate_deg=45.0 * p, mesh=mesh)
            for p in range(n_planets)]


def microbench_leaves(depth: int, occupancy: float,
                      pool_like: bool = False) -> np.ndarray:
    """Config 4 bitfields: bool[2**depth] with the documented seeds."""
    n = 1 << depth
    rng = np.random.default_rng(1000 * depth + round(100 * occupancy))
    if not pool_like:
        return rng.random(n) < occupancy
    leaves = np.zeros(n, dtype=bool)
    head = int(occupancy * n / 2)
    leaves[:head] = True
    rest = rng.random(n - head) < (occupancy / 2) / max(1e-12, 1 - occupancy / 2)
    leaves[head:] = rest
    return leaves
