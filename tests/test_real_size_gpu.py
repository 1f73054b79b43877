"""GPU, BASELINE configurations at their REAL sizes, slot level, against the
oracle run at the SAME size (not a smaller pool): config 3 (Earth sweep, 2^26
slots, all 128 frames), config 5 (8 planets x 2^24 slots in one batch launch),
the long soak loop and the wide-grid (4 CTAs per SM) frame kernel at 1 M live
bisectors.  Arrays are compared on the device (the oracle's arrays are uploaded
one at a time) so that a 3.5 GB pool compares in about a second.

Reference behaviour matched: ``ParallelEngine(threads=1).update``,
pkg/src/cbtmesh/pipeline.py:204-322, compare set of SURVEY.md 8(c).
"""

import ctypes as C

import numpy as np
import pytest

from paper_2407_02215_b200 import _lib, halfedge, workloads
from paper_2407_02215_b200.lod import LodDecide
from paper_2407_02215_b200.pipeline import (MergeAll, ParallelEngine, UniformSplit,
                                            run_lod_sequence_batch)
from paper_2407_02215_b200.state import initialize

from tests.parity import stats_words

pytestmark = pytest.mark.gpu

RECORD_ARRAYS = ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter")


def _upload(arr, device):
    import torch
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).to(device)


def _first_diff(g, o):
    import torch
    bad = (g.reshape(g.shape[0], -1) != o.reshape(o.shape[0], -1)).any(dim=1)
    rows = torch.nonzero(bad).flatten()
    r = int(rows[0])
    return f"{rows.numel()} rows differ, first row {r}: gpu {g[r].tolist()} oracle {o[r].tolist()}"


def device_state_equal(st, op, tag, stats):
    """Every array of SURVEY 8(c) -- records, commands, reservations, counter,
    the active list, the consumed free-rank window, the bitfield and every
    level sum (reference heap layout through cbtm_export_nodes) -- compared on
    the device against the oracle's arrays."""
    import torch
    dev = st.device
    for k in RECORD_ARRAYS:
        o = _upload(getattr(op, k), dev)
        g = getattr(st, "d_" + k)
        if not torch.equal(g, o):
            raise AssertionError(f"{tag}: {k}: {_first_diff(g, o)}")
        del o
    n = stats.live_before
    o = _upload(op.cache_live[:n], dev)
    assert torch.equal(st.d_cache_live[:n], o), f"{tag}: cache_live[:n]"
    T = stats.reserved_slots
    A = stats.split_allocs + stats.merge_allocs
    if st.exact_free_cache:
        F = st.capacity - n
        o = _upload(op.cache_free[:F], dev)
        assert torch.equal(st.d_cache_free[:F], o), f"{tag}: cache_free[:F]"
    elif A:
        o = _upload(op.cache_free[T - A:T], dev)
        assert torch.equal(st.d_cache_free[T - A:T], o), f"{tag}: cache_free[T-A:T)"
    nodes = torch.empty(2 * st.capacity, dtype=torch.int32, device=dev)
    rc = _lib.load().cbtm_export_nodes(_lib.ptr(st.d_bits), _lib.ptr(st.d_counters), st.depth,
                                       _lib.ptr(nodes), st.stream())
    _lib.check(rc, "cbtm_export_nodes")
    o = _upload(op.nodes, dev)
    if not torch.equal(nodes, o):
        raise AssertionError(f"{tag}: cbt.nodes: {_first_diff(nodes, o)}")
    del nodes, o
    # indirect dispatch arguments written on the device by the index pass
    assert st.d_dispatch.tolist() == [(n + 255) // 256, 1, 1, n], f"{tag}: dispatch args"


def live_records_equal(st, op, tag, stats):
    """Cheap per-frame check: the active list and the records at the live
    slots (ids + the three neighbour links), gathered on the device."""
    import torch
    dev = st.device
    n = stats.live_before
    o_live = _upload(op.cache_live[:n], dev)
    assert torch.equal(st.d_cache_live[:n], o_live), f"{tag}: cache_live[:n]"
    live = np.flatnonzero(op.leaves)
    idx = torch.from_numpy(live).to(dev)
    for k in ("ids", "nexts", "prevs", "twins"):
        o = _upload(getattr(op, k)[live], dev)
        assert torch.equal(getattr(st, "d_" + k)[idx], o), f"{tag}: {k} at the live slots"
    assert int(st.d_counters[1].item()) == live.size == stats.live_after, f"{tag}: root count"


def test_config3_earth_sweep_2_26_slot_level_every_frame():
    """BASELINE config 3 at its real size against the oracle at 2^26: all 128
    frames' counters, the active list and the live records after every launch
    of 4 frames, every array of the pool every 8th frame."""
    import oracle
    from oracle import OraclePool, OracleVerdict
    seq = workloads.earth_sweep(depth=26, frames=64)
    prms = seq.params()
    st = initialize(seq.mesh, 26)
    op = OraclePool(seq.mesh, 26)
    threads = oracle.max_threads()
    peak = 0
    with ParallelEngine() as eng:
        for f0 in range(0, seq.n_frames, 4):
            rows = eng.run_lod_sequence(st, prms[f0:f0 + 4], first_epoch=f0)
            for j, r in enumerate(rows):
                # stage 2 as a linear scan: same arrays as the descents (pinned in test_oracle_golden)
                o, _ = op.update(OracleVerdict.lod(seq.mesh, prms[f0 + j]), threads=threads, fast_setup=True)
                assert stats_words(r) == tuple(int(x) for x in o), f"frame {f0 + j}: counters"
                assert r.poison == 0
                peak = max(peak, r.live_after)
            live_records_equal(st, op, f"frame {f0 + 3}", rows[-1])
            if (f0 + 4) % 8 == 0:
                device_state_equal(st, op, f"frame {f0 + 3}", rows[-1])
    assert peak > 60000 and rows[-1].live_after < 40000   # went down to the ground and back to space


def test_config3_2_26_exact_free_cache_per_frame_updates():
    """Same pool size through ParallelEngine.update (one launch per frame), with
    the whole free cache materialised like the reference does: 12 frames, every
    array including cache_free[0:F) every 4th frame."""
    import oracle
    from oracle import OraclePool, OracleVerdict
    seq = workloads.earth_sweep(depth=26, frames=64)
    prms = seq.params()
    st = initialize(seq.mesh, 26, exact_free_cache=True)
    op = OraclePool(seq.mesh, 26)
    threads = oracle.max_threads()
    with ParallelEngine() as eng:
        for f in range(12):
            r = eng.update(st, LodDecide(seq.config, seq.cameras[f], seq.mesh), epoch=f)
            o, _ = op.update(OracleVerdict.lod(seq.mesh, prms[f]), threads=threads, fast_setup=(f % 4 != 3))
            assert stats_words(r) == tuple(int(x) for x in o), f"frame {f}: counters"
            if f % 4 == 3:     # genuine stage-2 descents on the oracle side for the compared frames
                device_state_equal(st, op, f"frame {f}", r)


def test_config5_eight_planets_2_24_batch_vs_oracle():
    """BASELINE config 5 at its real size: 8 icosphere planets on 2^24-slot
    pools, paths rotated by p * 45 degrees, advanced in lockstep by
    cbtm_run_lod_sequence_batch.  Planets 0 and 5 are compared with the oracle
    at 2^24 (counters every frame, all arrays at frames 63 and 127), the other
    six with solo runs of the same sequence, array for array."""
    import torch
    import oracle
    from oracle import OraclePool, OracleVerdict
    seqs = workloads.planet_batch(8, 24, 64)
    prms = [s.params() for s in seqs]
    states = [initialize(s.mesh, 24) for s in seqs]
    first = run_lod_sequence_batch(states, [p[:64] for p in prms])
    threads = oracle.max_threads()
    oracles = {}
    for p in (0, 5):
        op = oracles[p] = OraclePool(seqs[p].mesh, 24)
        for f in range(64):
            o, _ = op.update(OracleVerdict.lod(seqs[p].mesh, prms[p][f]), threads=threads, fast_setup=True)
            assert stats_words(first[p][f]) == tuple(int(x) for x in o), f"planet {p} frame {f}"
        device_state_equal(states[p], op, f"planet {p} frame 63", first[p][63])
    second = run_lod_sequence_batch(states, [p[64:] for p in prms], first_epoch=64)
    for p in (0, 5):
        op = oracles[p]
        for f in range(64, 128):
            o, _ = op.update(OracleVerdict.lod(seqs[p].mesh, prms[p][f]), threads=threads, fast_setup=True)
            assert stats_words(second[p][f - 64]) == tuple(int(x) for x in o), f"planet {p} frame {f}"
        device_state_equal(states[p], op, f"planet {p} frame 127", second[p][63])
    del oracles
    with ParallelEngine() as eng:
        for p in (1, 2, 3, 4, 6, 7):
            solo = initialize(seqs[p].mesh, 24)
            rows = eng.run_lod_sequence(solo, prms[p])
            assert [stats_words(r) for r in rows] == [stats_words(r) for r in first[p] + second[p]], p
            for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter", "bits", "counters"):
                assert torch.equal(getattr(solo, "d_" + k), getattr(states[p], "d_" + k)), f"planet {p}: {k}"
            n = rows[-1].live_before
            assert torch.equal(solo.d_cache_live[:n], states[p].d_cache_live[:n]), f"planet {p}: cache_live"
            del solo
    # rotated paths really are different planets' worth of work, not eight copies
    assert len({tuple(r.live_after for r in first[p]) for p in range(8)}) > 1


def test_soak_camera_loop_d22():
    """Long ground<->space loop (640 frames, 5 periods) on a 2^22 pool, one launch
    per 160 frames, against the oracle: counters every frame, every array at the
    end of every launch (was tests/soak.py)."""
    import oracle
    from oracle import OraclePool, OracleVerdict
    import bench
    seq, down, cycle = bench.sweep_params(22, 0.0)
    prm = np.concatenate([down, bench.step_params(cycle, 0, 640 - len(down))])
    st = initialize(seq.mesh, 22)
    op = OraclePool(seq.mesh, 22)
    threads = oracle.max_threads()
    eng = ParallelEngine()
    ooms = 0
    for f0 in range(0, len(prm), 160):
        rows = eng.run_lod_sequence(st, prm[f0:f0 + 160], first_epoch=f0)
        for j, r in enumerate(rows):
            o, _ = op.update(OracleVerdict.lod(seq.mesh, prm[f0 + j]), threads=threads, fast_setup=True)
            assert stats_words(r) == tuple(int(x) for x in o), f"frame {f0 + j}"
            assert r.poison == 0
            ooms += r.splits_rejected_oom + r.merges_rejected_oom
        device_state_equal(st, op, f"frame {f0 + 159}", rows[-1])


def test_wide_grid_kernel_one_million_live():
    """The 4-CTAs-per-SM variant of the frame kernel (CBTM_POOL_WIDE_GRID, chosen by
    the python layer above 150 k live bisectors) against the oracle: icosphere
    subdivided uniformly to depth 12 in a 2^22 pool, one update per epoch -- up to
    490 k splits in a frame, reservation pressure (3d+4 per split exceeds the free
    count), ~1 M live -- then merged back down by MergeAll frames.  Every counter
    every frame, every array every 3rd frame (was tests/large_live_check.py)."""
    import oracle
    from oracle import OraclePool, OracleVerdict
    mesh = halfedge.icosphere(1.0, 1)
    st = initialize(mesh, 22)
    op = OraclePool(mesh, 22)
    threads = oracle.max_threads()
    plan = [(UniformSplit(12), OracleVerdict.uniform(12))] * 17 + [(MergeAll(), OracleVerdict.const(2))] * 5
    wide_frames = rejected = 0
    with ParallelEngine() as eng:
        for e, (gpu, cpu) in enumerate(plan):
            wide_frames += bool(st.c_pool().flags & _lib.POOL_WIDE_GRID)
            r = eng.update(st, gpu, epoch=e)
            o, _ = op.update(cpu, threads=threads, fast_setup=True)
            assert stats_words(r) == tuple(int(x) for x in o), f"epoch {e}"
            assert r.poison == 0
            rejected += r.splits_rejected_oom
            if e % 3 == 2 or e == len(plan) - 1:
                device_state_equal(st, op, f"epoch {e}", r)
    assert wide_frames >= 8, "the wide-grid kernel was not exercised"
    assert rejected > 0, "no reservation pressure"
    assert max(int(x) for x in (op.count(),)) > 0


def test_wide_grid_flag_in_one_launch_matches_narrow():
    """The same subdivision with all epochs inside ONE launch of each kernel
    variant (flag forced): identical counters and arrays."""
    import torch
    mesh = halfedge.icosphere(1.0, 1)
    a = initialize(mesh, 22)
    b = initialize(mesh, 22)
    eng = ParallelEngine()
    rows_a = eng.run_epochs(a, UniformSplit(11), 15)
    b._stats_np[7] = 10 ** 6            # the python layer reads the last published live count
    assert b.c_pool().flags & _lib.POOL_WIDE_GRID
    pool = b.c_pool()
    cv = UniformSplit(11).device_verdict(b)
    d_stats = torch.zeros((15, _lib.STATS_WORDS), dtype=torch.int64, device=b.device)
    _lib.check(_lib.load().cbtm_run_epochs(C.byref(pool), C.byref(cv), 15, _lib.ptr(d_stats), b.stream()),
               "cbtm_run_epochs")
    rows_b = d_stats.cpu().numpy()
    b._touched()
    assert [list(stats_words(r)) for r in rows_a] == [[int(rows_b[e, k]) for k in (0, 1, 2, 3, 4, 5, 6, 7)]
                                                       for e in range(15)]
    for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter", "bits", "counters"):
        assert torch.equal(getattr(a, "d_" + k), getattr(b, "d_" + k)), k


def test_dispatch_args_after_every_kind_of_update():
    """d_dispatch == [ceil(n/256), 1, 1, n] with n = the length of the active list
    the index pass just wrote (north_star subsystem 4), through cbtm_update,
    the begin/finish split (python callable) and the standalone cbtm_index."""
    import torch
    mesh = halfedge.dodecahedron()
    st = initialize(mesh, 14)
    with ParallelEngine() as eng:
        for e in range(6):
            r = eng.update(st, UniformSplit(5), epoch=e)
            n = r.live_before
            assert st.d_dispatch.tolist() == [(n + 255) // 256, 1, 1, n]
        r = eng.update(st, lambda bid: 2, epoch=6)
        assert st.d_dispatch.tolist() == [(r.live_before + 255) // 256, 1, 1, r.live_before]
    n = st.count()
    disp = torch.zeros(4, dtype=torch.int32, device=st.device)
    live = torch.empty(n, dtype=torch.int32, device=st.device)
    rc = _lib.load().cbtm_index(_lib.ptr(st.d_bits), _lib.ptr(st.d_counters), st.depth, _lib.ptr(live), 0,
                                _lib.ptr(disp), st.stream())
    _lib.check(rc, "cbtm_index")
    assert disp.tolist() == [(n + 255) // 256, 1, 1, n]
    assert np.array_equal(live.cpu().numpy(), st.live_slots())
