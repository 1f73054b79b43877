"""GPU: the drop-in API behaves like the reference's (mirrors of the reference's
own pkg/tests/test_pipeline.py and test_lod.py cases, run through our package),
plus the device-side validator and the triangle export."""

import numpy as np
import pytest

from paper_2407_02215_b200 import bisector, halfedge, lod
from paper_2407_02215_b200.pipeline import (CSV_HEADER, EpochFactory, KeepAll, KernelDecide, MergeAll,
                                            ParallelEngine, SplitAll, UniformSplit, converged_epoch,
                                            evaluate_verdicts, write_stats_csv)
from paper_2407_02215_b200.state import (CapacityError, conformity_violations, initialize,
                                         pointer_violations)
from tests.workloads import pentagon_cluster

pytestmark = pytest.mark.gpu


def fig_id(label, depth, rank=4):
    return label + (1 << rank) * (1 << depth)


def assert_sound(st):
    assert pointer_violations(st) == []
    assert conformity_violations(st) == []
    dev = st.validate_device()
    assert dev["live"] == st.count()
    assert (dev["bad_ids"], dev["too_deep"], dev["dangling"], dev["no_reciprocal"], dev["depth_gaps"]) == (0,) * 5
    assert dev["first_bad_slot"] == -1


def test_keep_all_is_identity():
    st = initialize(halfedge.dodecahedron(), 9)
    before = st.neighbor_id_map()
    with ParallelEngine(threads=2) as eng:
        stats = eng.update(st, KeepAll())
    assert stats.live_before == stats.live_after == 60 and stats.structural_ops == 0
    assert len(stats.stage_times_us) == 9
    assert st.neighbor_id_map() == before


def test_figure_quad_merge_and_unanimous_consent():
    st = initialize(pentagon_cluster(), 6)
    with ParallelEngine() as eng:
        eng.update(st, lambda bid: 1 if bid == fig_id(7, 0) else 0)
        eng.update(st, lambda bid: 1 if bid == fig_id(14, 1) else 0)
        inset = st.live_ids()
        quad = {fig_id(l, 2) for l in (28, 29, 46, 47)}
        assert quad <= inset
        dissent = sorted(quad)[0]
        stats = eng.update(st, lambda bid: 2 if bid in quad - {dissent} else 0)
        assert stats.merges_applied == 0 and st.live_ids() == inset     # one member keeps: nobody merges
        stats = eng.update(st, lambda bid: 2 if bid in quad else 0)
    assert stats.merges_applied == 4
    assert st.live_ids() == (inset - quad) | {fig_id(14, 1), fig_id(23, 1)}
    assert_sound(st)


def test_split_wins_over_merge():
    st = initialize(pentagon_cluster(), 6)
    with ParallelEngine() as eng:
        eng.update(st, lambda bid: 1 if bid == fig_id(7, 0) else 0)
        quad = {fig_id(l, 1) for l in (14, 15, 2, 3)}
        verdicts = {bid: 2 for bid in quad}
        verdicts[fig_id(14, 1)] = 1
        stats = eng.update(st, lambda bid: verdicts.get(bid, 0))
    assert stats.merges_applied == 0 and stats.splits_applied > 0
    assert_sound(st)


def test_reserved_slots_disjoint_and_previously_free():
    st = initialize(halfedge.quad_grid(2, 2), 8)
    free_before = set(range(st.capacity)) - {int(s) for s in st.live_slots()}
    consumed = [int(s) for s in st.live_slots()]
    with ParallelEngine(threads=4) as eng:
        stats = eng.update(st, SplitAll())
    assert stats.splits_applied == 16
    claimed = []
    for s in consumed:
        cmd = int(st.commands[s])
        n = 2 + ((cmd >> 1) & 1) + ((cmd >> 2) & 1)
        claimed.extend(int(x) for x in st.reserved[s, :n])
    assert len(claimed) == len(set(claimed)) and set(claimed) <= free_before


def test_uniform_split_doubles_and_csv():
    st = initialize(halfedge.single_triangle(), 9)
    with ParallelEngine(threads=2) as eng:
        stats = eng.run_epochs(st, UniformSplit(3), 4)
    assert [s.live_after for s in stats] == [6, 12, 24, 24]
    assert converged_epoch(stats) == 3
    st = initialize(halfedge.quad_grid(2, 2), 9)
    with ParallelEngine() as eng:
        stats = eng.run_epochs(st, UniformSplit(2), 3)
    text = write_stats_csv(stats, no_timing=True)
    assert text.splitlines()[0] == CSV_HEADER
    assert text.splitlines()[1].split(",")[:7] == ["0", "16", "32", "16", "0", "0", "0"]
    with pytest.raises(ValueError):
        with ParallelEngine() as eng:
            eng.run_epochs(st, KeepAll(), 0)


def test_alternating_split_merge_returns_to_start():
    st = initialize(halfedge.quad_grid(2, 2), 12)
    with ParallelEngine() as eng:
        eng.update(st, UniformSplit(1))
        base = st.live_ids()
        stats = eng.run_epochs(st, EpochFactory(lambda e: SplitAll() if e % 2 == 0 else MergeAll()), 6)
    assert all(s.splits_rejected_oom == 0 and s.structural_ops > 0 for s in stats)
    assert st.live_ids() == base
    assert_sound(st)


def test_oom_rejection_is_safe_and_depth_limit_demotes():
    st = initialize(halfedge.single_triangle(), 4)
    with ParallelEngine() as eng:
        rejected = 0
        for _ in range(6):
            rejected += eng.update(st, SplitAll()).splits_rejected_oom
            assert_sound(st)
    assert rejected > 0 and st.count() <= 16
    st = initialize(halfedge.single_triangle(), 4)
    st.max_depth = 1
    with ParallelEngine() as eng:
        eng.update(st, SplitAll())
        stats = eng.update(st, SplitAll())
    assert stats.splits_applied == 0
    assert max(bisector.depth_of(b, st.rank) for b in st.live_ids()) == 1
    with pytest.raises(CapacityError):
        initialize(halfedge.dodecahedron(), 5)


def test_user_kernel_decide_subclass_and_clone():
    class EveryOther(KernelDecide):          # implements only the reference's fill protocol
        def fill(self, verdicts, state, count, start, end):
            for i in range(start, end):
                verdicts[i] = 1 if int(state.ids[state.cache_live[i]]) % 2 == 0 else 0

    st = initialize(halfedge.dodecahedron(), 10)
    twin = st.clone()
    with ParallelEngine() as eng:
        a = eng.update(st, EveryOther())
        b = eng.update(twin, lambda bid: 1 if bid % 2 == 0 else 0)
    assert a.splits_applied == b.splits_applied > 0
    assert st.live_ids() == twin.live_ids() and st.neighbor_id_map() == twin.neighbor_id_map()
    assert_sound(st)


def test_lod_decide_matches_python_decide_and_static_camera_converges():
    """reference test_lod.py:127-146 and :212-227"""
    mesh = halfedge.dodecahedron()
    cfg = lod.LodConfig(target_area_px=400.0)
    cam = lod.Camera([0.0, 0.2, 3.0], [0.0, -0.05, -1.0], [0, 1, 0], width=640, height=480)
    st = initialize(mesh, 14)
    dec = lod.LodDecide(cfg, cam, mesh)
    stats = []
    with ParallelEngine() as eng:
        for epoch in range(12):
            # device verdicts == the pure-python criterion, id by id, every epoch
            got = evaluate_verdicts(st, dec.device_verdict(st))
            ids = st.ids[st.cache_live[:st.count()]]
            want = np.array([lod.decide(cfg, cam, mesh, int(b)) for b in ids], dtype=np.int8)
            assert np.array_equal(got, want), epoch
            stats.append(eng.update(st, dec, epoch=epoch))
    assert converged_epoch(stats) is not None        # a static camera converges
    assert st.count() > 60
    assert_sound(st)


def test_triangle_export_matches_host_decode():
    st = initialize(halfedge.dodecahedron(), 17)     # headroom: no reservation pressure
    with ParallelEngine() as eng:
        stats = eng.run_epochs(st, UniformSplit(5), 7)
    assert converged_epoch(stats) is not None
    ids, tris = st.decode_live()
    assert len(ids) == st.count() == 60 * 32
    for k in range(0, len(ids), 97):
        want = bisector.decode_tri(int(ids[k]), st.rank, st.mesh.next, st.mesh.vert, st.mesh.positions)
        assert np.array_equal(tris[k].view(np.uint64), want.view(np.uint64))
    # areas add up to the surface of the dodecahedron (area conservation)
    area = 0.5 * np.linalg.norm(np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0]), axis=1).sum()
    roots = np.array([st.mesh.root_bisector_vertices(h) for h in range(60)])
    root_area = 0.5 * np.linalg.norm(np.cross(roots[:, 1] - roots[:, 0], roots[:, 2] - roots[:, 0]), axis=1).sum()
    assert abs(area - root_area) < 1e-9
    # device-resident export: same triangles in active-list (ascending slot) order, draw args on device,
    # and the active list it leaves behind is the current state's
    d_tris, d_draw = st.export_live_triangles()
    assert np.array_equal(d_tris.cpu().numpy().view(np.uint64), tris.view(np.uint64))
    assert d_draw.cpu().tolist() == [3 * len(ids), 1, 0, 0]
    assert np.array_equal(st.cache_live[:len(ids)], st.live_slots())
    assert np.array_equal(st.ids[st.live_slots()], ids)
    # a too small output buffer truncates instead of overrunning
    import torch
    small = torch.full((100, 3, 3), -1.0, dtype=torch.float64, device=st.device)
    part, d_draw = st.export_live_triangles(out=small)
    assert part.shape[0] == 100 and d_draw.cpu().tolist() == [300, 1, 0, 0]
    assert np.array_equal(part.cpu().numpy().view(np.uint64), tris[:100].view(np.uint64))


def test_triangle_export_deep_planet_ids_match_the_oracle_decode():
    """f1 where fp64 matters: BASELINE config 2 (cube-sphere fly-in, 2^20 pool) at frame 63 --
    75 k live bisectors down to depth 40 -- every exported triangle bit-compared with the oracle's
    restatement of nb_decode_tris (bisector.py:186-189), the draw arguments, and the order."""
    import oracle
    from paper_2407_02215_b200 import workloads
    seq = workloads.cube_sphere_flyin(depth=20, frames=64)
    st = initialize(seq.mesh, 20)
    with ParallelEngine() as eng:
        rows = eng.run_lod_sequence(st, seq.params())
    assert rows[-1].peak_depth >= 38
    d_tris, d_draw = st.export_live_triangles()
    n = st.count()
    live = st.live_slots()
    ids = st.ids[live]
    assert d_tris.shape == (n, 3, 3) and n > 70000
    depths = np.array([bisector.depth_of(int(b), st.rank) for b in ids])
    assert depths.max() >= 39 and (depths >= 30).sum() > 1000
    want = oracle.decode_tris(ids, st.rank, seq.mesh.next, seq.mesh.vert, seq.mesh.positions)
    got = d_tris.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert d_draw.cpu().tolist() == [3 * n, 1, 0, 0]
    assert np.array_equal(st.cache_live[:n], live)
    # and the python mirror of the decode agrees on the deepest ones
    for k in np.argsort(depths)[-20:]:
        host = bisector.decode_tri(int(ids[k]), st.rank, seq.mesh.next, seq.mesh.vert, seq.mesh.positions)
        assert np.array_equal(host.view(np.uint64), got[k].view(np.uint64))
    # the batch entry point of the reference's API runs the same kernel
    out = np.empty((n, 3, 3))
    bisector.nb_decode_tris(ids, st.rank, seq.mesh.next, seq.mesh.vert, seq.mesh.positions, out, 0, n)
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))


def test_device_validator_reports_corruption():
    st = initialize(halfedge.quad_grid(2, 2), 8)
    with ParallelEngine() as eng:
        eng.update(st, UniformSplit(2))
    assert_sound(st)
    victim = int(st.live_slots()[5])
    st.d_twins[victim] = int(np.setdiff1d(np.arange(st.capacity), st.live_slots())[0])   # dangling
    other = int(st.live_slots()[9])
    st.d_nexts[other] = int(st.live_slots()[0]) if int(st.nexts[other]) != int(st.live_slots()[0]) else int(st.live_slots()[1])
    st._touched()
    dev = st.validate_device()
    host = pointer_violations(st)
    assert dev["dangling"] == sum("dangling" in v for v in host) >= 1
    assert dev["no_reciprocal"] == sum("no reciprocal" in v for v in host)
    assert dev["depth_gaps"] == sum("depth gap" in v for v in host)
    assert dev["first_bad_slot"] >= 0


def test_peak_depth_is_reduced_on_the_device():
    """UpdateStats.peak_depth = deepest live bisector at the start of the frame -- the per-frame
    reduction cmd_animate does on the host (cli.py:232-237) -- for single updates and sequences."""
    from paper_2407_02215_b200 import workloads
    seq = workloads.cube_sphere_flyin(depth=16, frames=12)
    st = initialize(seq.mesh, 16)
    with ParallelEngine() as eng:
        for i, cam in enumerate(seq.cameras[:6]):
            want = max(bisector.depth_of(int(b), st.rank) for b in st.ids[st.live_slots()])
            s = eng.update(st, lod.LodDecide(seq.config, cam, seq.mesh), epoch=i)
            assert s.peak_depth == want, i
        before = max(bisector.depth_of(int(b), st.rank) for b in st.ids[st.live_slots()])
        rows = eng.run_lod_sequence(st, seq.params()[6:])
        assert rows[0].peak_depth == before
        after = max(bisector.depth_of(int(b), st.rank) for b in st.ids[st.live_slots()])
        assert eng.update(st, KeepAll()).peak_depth == after


def test_profile_engine_reports_all_device_phase_times():
    """ParallelEngine(profile=True) waits for the frame's complete row: the six device phase timers
    folded onto the reference's nine `stage_times_us` slots (pipeline.py:218-223), same counters as the
    default engine, which returns on the early row (phases 4-6 not timed yet, no poison count)."""
    from paper_2407_02215_b200 import workloads
    seq = workloads.cube_sphere_flyin(depth=16, frames=10)
    a = initialize(seq.mesh, 16)
    b = initialize(seq.mesh, 16)
    fast, prof = ParallelEngine(), ParallelEngine(profile=True)
    for i, cam in enumerate(seq.cameras):
        sa = fast.update(a, lod.LodDecide(seq.config, cam, seq.mesh), epoch=i)
        sb = prof.update(b, lod.LodDecide(seq.config, cam, seq.mesh), epoch=i)
        assert sa.csv_row(no_timing=True) == sb.csv_row(no_timing=True)
        assert all(t > 0 for t in sb.phase_ns), sb.phase_ns
        t = sb.stage_times_us
        assert len(t) == 9 and t[1] > 0 and t[3] > 0 and t[4] > 0 and t[5] > 0 and t[8] > 0
        assert sa.phase_ns[0] > 0 and sa.phase_ns[1] > 0 and sa.phase_ns[2] > 0
        assert sa.phase_ns[3:] == [0, 0, 0] or sa.phase_ns[5] > 0      # early row (or the complete one if it won the race)
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.to_host()["nodes"], b.to_host()["nodes"])
    # python-callable verdicts under profiling: stages 1-2 and the host's verdict evaluation are timed with
    # events, the stages behind it by the device's phase timers (same nine slots as timed() fills,
    # pipeline.py:218-223: t2 cache pointers, t4 verdicts + commands, t5 reserve, t6 fill, t9 reduction)
    s = prof.update(b, lambda bid: 0, epoch=99)
    t = s.stage_times_us
    assert s.structural_ops == 0 and t[1] > 0 and t[3] > 0 and t[4] > 0 and t[5] > 0 and t[8] > 0
    assert s.phase_ns[1] > 0 and s.phase_ns[5] > 0
