"""GPU: the multi-GPU path of BASELINE config 5 as far as one GPU can take it:
`batch.run_planet_batch` against solo runs, `bench.py --workload batch` under
torch.distributed.run with the NCCL process group initialised (world size 1 on a one-GPU box,
2 when a second GPU is visible), and the planet-for-planet equality of the N = 1 and N = 2 lines."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2407_02215_b200 import _lib, batch, workloads
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_run_planet_batch_world1_and_world2_shares_equal_solo_runs():
    """run_planet_batch for world 1 (all planets) and for both ranks of a world of 2 (each on
    this GPU, one after the other): the stats blocks, gathered, equal one solo sequence run per
    planet; a second call continues the returned states."""
    import torch
    seqs = workloads.planet_batch(5, 18, 12)
    prms = [s.params() for s in seqs]
    first = [p[:12] for p in prms]
    second = [p[12:] for p in prms]
    with ParallelEngine() as eng:
        solo_states = [initialize(s.mesh, 18) for s in seqs]
        solo = np.array([[_row(r) for r in eng.run_lod_sequence(st, p)] for st, p in zip(solo_states, prms)])
    states, block = batch.run_planet_batch(seqs, first, world=1, rank=0)
    states, block2 = batch.run_planet_batch(seqs, second, world=1, rank=0, states=states)
    full = np.concatenate([batch.gather_stats(block, list(range(5)), 5, 1),
                           batch.gather_stats(block2, list(range(5)), 5, 1)], axis=1)
    assert full.shape == (5, 24, _lib.STATS_WORDS)
    assert np.array_equal(full[:, :, :8], solo)
    for p in range(5):
        for k in ("ids", "nexts", "prevs", "twins", "bits", "counters"):
            assert torch.equal(getattr(states[p], "d_" + k), getattr(solo_states[p], "d_" + k)), (p, k)
    parts = {}
    for rank in range(2):
        owned = batch.planets_of_rank(5, 2, rank)
        _, blk = batch.run_planet_batch(seqs, prms, world=2, rank=rank)
        assert blk.shape[0] == len(owned)
        for k, p in enumerate(owned):
            parts[p] = blk[k]
    assert np.array_equal(np.stack([parts[p] for p in range(5)])[:, :, :8], solo)
    with pytest.raises(ValueError):
        batch.run_planet_batch(seqs, prms, world=2, rank=0, states=states)   # 5 states for a rank that owns 3


def _row(s):
    return [s.splits_rejected_oom, s.merges_rejected_oom, s.splits_applied, s.merges_applied,
            s.split_allocs, s.merge_allocs, s.live_before, s.live_after]


def _bench(*flags, timeout=900):
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    proc = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *flags], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=timeout)
    assert proc.returncode == 0, (proc.stdout + proc.stderr)[-3000:]
    lines = [l for l in proc.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, proc.stdout[-2000:]
    return json.loads(lines[0]), proc.stderr


def test_bench_config5_under_torchrun_initialises_nccl():
    """`bench.py --workload batch` launched as one rank under torch.distributed.run: NCCL process
    group, barrier, max-over-ranks reductions and the final all_gather of the stats all run (world
    size 1), and the line equals the plain single-process run planet for planet."""
    plain, _ = _bench("--workload", "batch", "--steps", "6", "--warmup", "3")
    ranked, err = _bench("--workload", "batch", "--steps", "6", "--warmup", "3", "--torchrun-world1")
    assert plain["n_gpus"] == ranked["n_gpus"] == 1 and plain["scaling"] == "strong"
    assert "NCCL" in ranked["collective"] and "none" in plain["collective"]
    assert plain["stats_digest"] == ranked["stats_digest"]
    assert plain["config"]["planets"] == 8 and plain["planets_per_rank"] == [8]
    assert plain["gpu_launches"] == 1 and plain["e2e"]["h2d_bytes_per_step"] == 8 * 23 * 8
    assert len(plain["stats_digest"]["live_after_last_frame"]) == 8
    assert ranked["value"] > 0 and ranked["e2e"]["value"] > 0


def test_bench_config5_two_ranks_equal_one_rank_planet_for_planet():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (the round's boxes have one): covered at world size 1 above and by "
                    "tests/test_batch_gloo.py on CPU")
    one, _ = _bench("--workload", "batch", "--steps", "6", "--warmup", "3")
    two, _ = _bench("--gpus", "2", "--steps", "6", "--warmup", "3")
    assert two["n_gpus"] == 2 and two["planets_per_rank"] == [4, 4] and len(two["per_rank_device_ms"]) == 2
    assert one["stats_digest"] == two["stats_digest"]
