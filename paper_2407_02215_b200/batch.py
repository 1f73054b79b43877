"""Batches of independent planets across the GPUs of one box.

One tessellation does not shard (global ranks: admission order, scan
placement), so a single mesh is "replicas only".  Batches shard trivially:
planet ``p`` belongs to rank ``p mod world`` and lives entirely on that rank's
GPU; there is no peer traffic per frame.  The only collective is the final
gather of the per-frame stats tensor (NCCL on GPUs; gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def planets_of_rank(n_planets: int, world: int, rank: int) -> list[int]:
    """Round-robin ownership: planet p -> rank p mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return [p for p in range(n_planets) if p % world == rank]


def gather_stats(local: np.ndarray, owned: list[int], n_planets: int, world: int,
                 device=None) -> np.ndarray | None:
    """Assemble int64[n_planets, frames, words] on every rank from each rank's
    int64[len(owned), frames, words].  Uses torch.distributed when initialised
    (all_gather of equally padded blocks -- also at world size 1, so that a
    one-GPU run goes through the same NCCL path), otherwise returns the local
    block re-indexed (single process)."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, dtype=np.int64)
    frames, words = local.shape[1], local.shape[2]
    out = np.zeros((n_planets, frames, words), dtype=np.int64)
    if not (dist.is_available() and dist.is_initialized()):
        for k, p in enumerate(owned):
            out[p] = local[k]
        return out
    per_rank = (n_planets + world - 1) // world
    block = torch.zeros((per_rank, frames, words), dtype=torch.int64)
    block[:len(owned)] = torch.from_numpy(local)
    if device is not None:
        block = block.to(device)
    blocks = [torch.zeros_like(block) for _ in range(world)]
    dist.all_gather(blocks, block)
    for r in range(world):
        got = blocks[r].cpu().numpy()
        for k, p in enumerate(planets_of_rank(n_planets, world, r)):
            out[p] = got[k]
    return out


def run_planet_batch(sequences, frames_params, world: int = 1, rank: int = 0,
                     device=None, states=None):
    """Advance this rank's planets through ``frames_params`` (GPU).  ``sequences``
    are workloads.LodSequence objects for ALL planets of the batch,
    ``frames_params[p]`` is float64[frames, 23] for planet ``p``; the rank owns
    planets ``planets_of_rank(len(sequences), world, rank)`` and touches only
    those.  The planets of one rank advance in lockstep inside one cooperative
    launch (``pipeline.run_lod_sequence_batch``): a single planet's frame is
    latency bound and leaves the GPU mostly idle, a batch shares every grid
    barrier and round trip.  ``states`` continues pools returned by an earlier
    call (same rank) instead of initialising fresh ones.
    Returns (states, int64[owned, frames, STATS_WORDS]) -- the block
    :func:`gather_stats` assembles across ranks."""
    from . import _lib
    from .pipeline import run_lod_sequence_batch
    from .state import initialize

    owned = planets_of_rank(len(sequences), world, rank)
    if states is None:
        states = [initialize(sequences[p].mesh, sequences[p].depth, device=device) for p in owned]
    elif len(states) != len(owned):
        raise ValueError(f"rank {rank} owns {len(owned)} planets, got {len(states)} states")
    rows = run_lod_sequence_batch(states, [frames_params[p] for p in owned], raw=True)
    frames = rows[0].shape[0] if rows else 0
    block = np.zeros((len(owned), frames, _lib.STATS_WORDS), dtype=np.int64)
    for k, r in enumerate(rows):
        block[k] = r
    return states, block
