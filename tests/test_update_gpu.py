"""GPU parity: the CUDA update path (through the python drop-in, i.e. the C
ABI) against the C oracle and the reference's golden digests, frame by frame,
every array, bit for bit."""

import numpy as np
import pytest

from paper_2407_02215_b200 import halfedge, workloads
from paper_2407_02215_b200.pipeline import (KeepAll, MergeAll, ParallelEngine,
                                            SplitAll, UniformSplit)
from paper_2407_02215_b200.lod import LodDecide
from paper_2407_02215_b200.state import initialize

from tests import workloads as tw
from tests.parity import (assert_state_equal, golden_frame_check, load_golden,
                          stats_words)

pytestmark = pytest.mark.gpu


MODES = ["exact", "fast", "fast-staged", "exact-staged", "fast-descend"]


def run_pair(name, mesh, depth, frames, gpu_decide_of, orc_verdict_of, mode,
             max_depth=None, golden=True, check_every=1):
    """mode: exact = whole free cache materialised (whole-array parity);
    fast = only the consumed free-rank window; -staged = one kernel per stage
    instead of the persistent cooperative frame kernel; -descend = free ranks
    resolved by tree descent instead of the window table (the fallback taken
    when a frame's allocations span more than 4096 leaf blocks)."""
    from oracle import OraclePool
    exact = mode.startswith("exact")
    st = initialize(mesh, depth, exact_free_cache=exact, staged_launches=mode.endswith("staged"),
                    descend_free_ranks=mode.endswith("descend"))
    op = OraclePool(mesh, depth)
    if max_depth is not None:
        st.max_depth = max_depth
        op.max_depth = max_depth
    rec = load_golden(name) if golden else None
    host = assert_state_equal(st, op, f"{name}/init", exact)
    if rec:
        golden_frame_check(host, rec["init"], f"{name}/init", exact)
    with ParallelEngine(threads=1) as eng:
        for f in range(frames):
            s = eng.update(st, gpu_decide_of(f, st), epoch=f)
            o, _ = op.update(orc_verdict_of(f, op), threads=8)
            assert stats_words(s) == tuple(int(x) for x in o), f"{name}/{f}: stats"
            assert s.poison == 0
            if f % check_every == 0 or f == frames - 1:
                host = assert_state_equal(st, op, f"{name}/{f}", exact, s)
                if rec:
                    golden_frame_check(host, rec["frames"][f], f"{name}/{f}", exact)
                    assert {k: rec["frames"][f]["stats"][k] for k in rec["frames"][f]["stats"]} == \
                        dict(zip(("oom_splits", "oom_merges", "split_freed", "merge_freed",
                                  "split_alloc", "merge_alloc", "live_before", "live_after"),
                                 stats_words(s)))
    return st, op


@pytest.mark.parametrize("exact", MODES)
def test_config1_quad_uniform(exact):
    from oracle import OracleVerdict
    st, _ = run_pair("quad_d16_uniform12", halfedge.single_quad(), 16, 18,
                     lambda f, st: UniformSplit(12),
                     lambda f, op: OracleVerdict.uniform(12), exact)
    assert st.count() == 16384


@pytest.mark.parametrize("exact", MODES)
def test_const_sources(exact):
    from oracle import OracleVerdict
    run_pair("grid_d9_uniform2", halfedge.quad_grid(2, 2), 9, 3,
             lambda f, st: UniformSplit(2), lambda f, op: OracleVerdict.uniform(2), exact)
    run_pair("triangle_d4_splitall", halfedge.single_triangle(), 4, 6,
             lambda f, st: SplitAll(), lambda f, op: OracleVerdict.const(1), exact)
    consts = [SplitAll, MergeAll]
    run_pair("grid_d12_alternate", halfedge.quad_grid(2, 2), 12, 8,
             lambda f, st: consts[f % 2](), lambda f, op: OracleVerdict.const(1 + f % 2), exact)
    run_pair("dodeca_d9_keep", halfedge.dodecahedron(), 9, 2,
             lambda f, st: KeepAll(), lambda f, op: OracleVerdict.const(0), exact)
    run_pair("triangle_d4_depthlimit1", halfedge.single_triangle(), 4, 3,
             lambda f, st: SplitAll(), lambda f, op: OracleVerdict.const(1), exact,
             max_depth=1)


@pytest.mark.parametrize("case", tw.SOUP_CASES, ids=lambda c: f"{c[0]}_d{c[1]}")
@pytest.mark.parametrize("exact", MODES)
def test_random_soups_under_pressure(case, exact):
    """Explicit random verdicts, not budgeted: OOM rejections every frame, so
    the admission tail walk and the top-of-window slot placement are pinned."""
    from oracle import OracleVerdict
    mesh_name, depth, seed, frames = case

    def verdicts(f, n):
        sp, mp = tw.soup_schedule(f)
        return tw.random_verdicts(n, seed, f, sp, mp)

    def gpu_decide(f, st):
        ids = st.ids[st.live_slots()]          # ascending slot == cache_live order
        table = {int(i): int(v) for i, v in zip(ids, verdicts(f, len(ids)))}
        return lambda bid: table[bid]          # python-callable path of the API

    run_pair(f"soup_{mesh_name}_d{depth}_s{seed}", tw.MESHES[mesh_name](), depth, frames,
             gpu_decide, lambda f, op: OracleVerdict.explicit_array(verdicts(f, op.count())),
             exact)


def _lod_pair(seq):
    from oracle import OracleVerdict
    prms = seq.params()
    return (lambda f, st: LodDecide(seq.config, seq.cameras[f], seq.mesh),
            lambda f, op: OracleVerdict.lod(seq.mesh, prms[f]))


def test_config2_cube_sphere_flyin_exact():
    seq = workloads.cube_sphere_flyin(depth=20, frames=64)
    g, o = _lod_pair(seq)
    run_pair("cube_sphere_flyin_d20", seq.mesh, 20, seq.n_frames, g, o, "exact")


@pytest.mark.parametrize("mode", ["fast", "fast-staged", "fast-descend"])
def test_config2_cube_sphere_flyin_fast(mode):
    seq = workloads.cube_sphere_flyin(depth=20, frames=64)
    g, o = _lod_pair(seq)
    run_pair("cube_sphere_flyin_d20", seq.mesh, 20, seq.n_frames, g, o, mode, check_every=4)


def test_config3_stress_earth_sweep_d20():
    """Config 3's camera sweep on a 2^20 pool: 727k OOM rejections."""
    seq = workloads.earth_sweep(depth=20, frames=64)
    g, o = _lod_pair(seq)
    run_pair("earth_sweep_d20", seq.mesh, 20, seq.n_frames, g, o, "exact", check_every=4)


def test_config3_stress_earth_sweep_d20_fast_window():
    """Same sweep in the default mode: the free-rank window table (and its
    descent fallback) under heavy reservation pressure."""
    seq = workloads.earth_sweep(depth=20, frames=64)
    g, o = _lod_pair(seq)
    run_pair("earth_sweep_d20", seq.mesh, 20, seq.n_frames, g, o, "fast", check_every=8)


def test_config3_short_d22():
    seq = workloads.earth_sweep(depth=22, frames=16)
    g, o = _lod_pair(seq)
    run_pair("earth_sweep_d22_short", seq.mesh, 22, seq.n_frames, g, o, "fast", check_every=8)


def test_sequence_runner_matches_per_frame_updates():
    """cbtm_run_lod_sequence (no host sync between frames) == frame-by-frame."""
    seq = workloads.cube_sphere_flyin(depth=18, frames=24)
    a = initialize(seq.mesh, 18)
    b = initialize(seq.mesh, 18)
    c = initialize(seq.mesh, 18, staged_launches=True)
    with ParallelEngine() as eng:
        staged = eng.run_lod_sequence(c, seq.params())
        per_frame = [eng.update(a, LodDecide(seq.config, c, seq.mesh), epoch=i)
                     for i, c in enumerate(seq.cameras)]
        batched = eng.run_lod_sequence(b, seq.params())
    assert [stats_words(s) for s in per_frame] == [stats_words(s) for s in batched]
    assert [stats_words(s) for s in per_frame] == [stats_words(s) for s in staged]
    ha, hb, hc = a.to_host(), b.to_host(), c.to_host()
    for k in ha:
        if k != "cache_free":
            assert np.array_equal(ha[k], hb[k]), k
            assert np.array_equal(ha[k], hc[k]), k


def test_batch_kernel_equals_separate_sequences():
    """cbtm_run_lod_sequence_batch (several planets in lockstep inside one
    cooperative launch, BASELINE config 5) == one sequence run per planet.
    Mixed batch: pools of different depth and mesh, one of them small enough to
    run under reservation pressure (admission tail path) next to pools on the
    a-priori fast path."""
    from paper_2407_02215_b200.pipeline import run_lod_sequence_batch
    seqs = [workloads.cube_sphere_flyin(depth=18, frames=20),
            workloads.earth_sweep(depth=20, frames=20, rotate_deg=45.0),
            workloads.cube_sphere_flyin(depth=12, frames=20),      # tiny pool: constant OOM pressure
            workloads.earth_sweep(depth=22, frames=20, rotate_deg=90.0),
            workloads.earth_sweep(depth=16, frames=20)]
    prms = [s.params()[:20] for s in seqs]
    solo = [initialize(s.mesh, s.depth) for s in seqs]
    both = [initialize(s.mesh, s.depth) for s in seqs]
    with ParallelEngine() as eng:
        want = [eng.run_lod_sequence(st, p) for st, p in zip(solo, prms)]
    got = run_lod_sequence_batch(both, prms)
    assert any(w.splits_rejected_oom + w.merges_rejected_oom for w in want[2]), "pressure case lost its pressure"
    for p, (w, g) in enumerate(zip(want, got)):
        assert [stats_words(s) for s in w] == [stats_words(s) for s in g], f"planet {p}: stats"
        ha, hb = solo[p].to_host(), both[p].to_host()
        for k in ha:
            assert np.array_equal(ha[k], hb[k]), f"planet {p}: {k}"


def test_more_planets_than_one_launch_takes():
    """Eleven small planets: the batch API splits them into launches of at most
    MAX_BATCH pools; results equal separate runs."""
    from paper_2407_02215_b200 import _lib
    from paper_2407_02215_b200.pipeline import run_lod_sequence_batch
    assert _lib.MAX_BATCH < 11
    seqs = [workloads.cube_sphere_flyin(depth=13 + p % 3, frames=10) for p in range(11)]
    solo = [initialize(s.mesh, s.depth) for s in seqs]
    both = [initialize(s.mesh, s.depth) for s in seqs]
    with ParallelEngine() as eng:
        want = [eng.run_lod_sequence(st, s.params()) for st, s in zip(solo, seqs)]
    got = run_lod_sequence_batch(both, [s.params() for s in seqs])
    for p in range(11):
        assert [stats_words(s) for s in want[p]] == [stats_words(s) for s in got[p]], p
        assert np.array_equal(solo[p].to_host()["nodes"], both[p].to_host()["nodes"]), p
        assert np.array_equal(solo[p].ids, both[p].ids), p


def test_linger_mode_matches_plain_updates():
    """ParallelEngine(linger_us=...): frames handed to the listening frame kernel
    through the host-mapped mailbox (no launch) == one launch per frame.  Covers
    back-to-back frames (mailbox), a pause longer than the linger time (fresh
    launch), other stream work in between, and a changed pool parameter."""
    import time
    seq = workloads.cube_sphere_flyin(depth=18, frames=40)
    a = initialize(seq.mesh, 18)
    b = initialize(seq.mesh, 18)
    plain = ParallelEngine()
    fast = ParallelEngine(linger_us=3000.0)
    want = []
    for i, cam in enumerate(seq.cameras):    # (not interleaved with the lingering run: work queued on the
        if i == 30:                           #  same stream would wait for the listening kernel to give up)
            a.max_depth = 30
        want.append(plain.update(a, LodDecide(seq.config, cam, seq.mesh), epoch=i))
    posted = 0
    for i, cam in enumerate(seq.cameras):
        if i == 12:
            time.sleep(0.02)                 # far beyond the linger time: the kernel has gone
        if i == 20:
            assert b.count() == want[i].live_before   # stream work (a device->host read) while the kernel listens
        if i == 30:
            b.max_depth = 30                 # pool parameter baked into the listening kernel: must relaunch
        listening = time.perf_counter() < b._mb_listen_until and b._mb_pool is b.c_pool()
        sb = fast.update(b, LodDecide(seq.config, cam, seq.mesh), epoch=i)
        posted += listening
        assert stats_words(want[i]) == stats_words(sb), i
    assert posted >= 20, f"only {posted} of 40 frames went through the mailbox"
    ha, hb = a.to_host(), b.to_host()
    for k in ha:
        assert np.array_equal(ha[k], hb[k]), k


def test_run_epochs_in_one_launch_equals_per_frame_updates():
    """ParallelEngine.run_epochs with one device verdict source = cbtm_run_epochs (all epochs in one
    launch) on BASELINE config 1 (quad, 2^16 pool, uniform depth 12: 18 frames, reservation pressure
    from frame 10 on): same counters and state as one update per epoch, and the golden live counts."""
    a = initialize(halfedge.single_quad(), 16)
    b = initialize(halfedge.single_quad(), 16)
    with ParallelEngine() as eng:
        per_frame = [eng.update(a, UniformSplit(12), epoch=e) for e in range(18)]
        one_launch = eng.run_epochs(b, UniformSplit(12), 18)
    assert [stats_words(s) for s in per_frame] == [stats_words(s) for s in one_launch]
    assert one_launch[-1].live_after == 16384 and sum(s.splits_rejected_oom for s in one_launch) > 0
    rec = load_golden("quad_d16_uniform12")
    assert [s.live_after for s in one_launch] == [f["stats"]["live_after"] for f in rec["frames"]]
    ha, hb = a.to_host(), b.to_host()
    for k in ha:
        assert np.array_equal(ha[k], hb[k]), k
