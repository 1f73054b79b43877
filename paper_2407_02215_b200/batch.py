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
    (all_gather of equally padded blocks), otherwise returns the local block
    re-indexed (single process)."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, dtype=np.int64)
    frames, words = local.shape[1], local.shape[2]
    out = np.zeros((n_planets, frames, words), dtype=np.int64)
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
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
                     device=None):
    """Advance this rank's planets frame by frame (GPU).  ``sequences`` are
    workloads.LodSequence objects, ``frames_params[p]`` is float64[frames, 23].
    The planets of one rank advance in lockstep inside one cooperative launch
    (``pipeline.run_lod_sequence_batch``): a single planet's frame is latency
    bound and leaves the GPU mostly idle, a batch shares every grid barrier and
    round trip.  Returns (states, int64[owned, frames, STATS_WORDS])."""
    from . import _lib
    from .pipeline import run_lod_sequence_batch
    from .state import initialize

    owned = planets_of_rank(len(sequences), world, rank)
    states = [initialize(sequences[p].mesh, sequences[p].depth, device=device) for p in owned]
    per_planet = run_lod_sequence_batch(states, [frames_params[p] for p in owned])
    rows = [[[s.splits_rejected_oom, s.merges_rejected_oom, s.splits_applied,
              s.merges_applied, s.split_allocs, s.merge_allocs, s.live_before,
              s.live_after] + [0] * (_lib.STATS_WORDS - 8) for s in stats] for stats in per_planet]
    return states, np.array(rows, dtype=np.int64).reshape(len(owned), -1, _lib.STATS_WORDS)
