"""Floor of the per-frame path: the same K frames (1) inside one launch, (2) as K launches queued
without any host wait (device-timed: kernel + inter-launch gap), (3) one launch per frame with the
host waiting for the frame's counters (cbtm_update_wait), (4) through ParallelEngine.update."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.lod import LodDecide
from paper_2407_02215_b200.pipeline import ParallelEngine, lod_verdict
from paper_2407_02215_b200.state import initialize

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 26
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0     # bench.py times frames [warmup, warmup + K) of the cycle
seq, down, cycle = bench.sweep_params(depth, 0.0)
eng = ParallelEngine()
state = initialize(seq.mesh, depth)
eng.run_lod_sequence(state, down)
if first:
    eng.run_lod_sequence(state, bench.step_params(cycle, 0, first))
start = state.clone()
cams = seq.cameras
cam_cycle = cams[bench.SETUP_FRAMES - 1::-1] + cams[:bench.SETUP_FRAMES]
L = _lib.load()
K = 64
pc = time.perf_counter
cam_cycle = [cam_cycle[(first + j) % len(cam_cycle)] for j in range(K)]
decs = [LodDecide(seq.config, cam_cycle[j], seq.mesh) for j in range(K)]   # kept alive: their buffers are read below
prm = np.stack([d._prm for d in decs])
cvs = []
for j in range(K):
    cv = _lib.CVerdict()
    cv.mode = _lib.VERDICT_LOD
    cv.root_tris = _lib.ptr(start.d_root_tris)
    C.memmove(cv.prm, decs[j]._prm_c, 8 * 23)
    cvs.append(cv)
ev = lambda: torch.cuda.Event(enable_timing=True)
for trial in range(3):
    st = start.clone(); torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(); rows = eng.run_lod_sequence(st, prm); b.record(); torch.cuda.synchronize()
    one_launch = a.elapsed_time(b) * 1e3 / K
    want = [(r.live_before, r.live_after, r.splits_applied, r.merges_applied) for r in rows]

    st = start.clone(); torch.cuda.synchronize()
    pref = st.c_pool_ref(); stream = st.stream()
    a, b = ev(), ev()
    a.record()
    for j in range(K):
        L.cbtm_update(pref, cvs[j], stream)
    b.record(); torch.cuda.synchronize()
    queued = a.elapsed_time(b) * 1e3 / K
    assert int(st._stats_np[7]) == want[-1][1]

    st = start.clone(); torch.cuda.synchronize()
    pref = st.c_pool_ref(); stream = st.stream(); hp = st._stats_host_ptr
    t0 = pc()
    for j in range(K):
        L.cbtm_update_wait(pref, cvs[j], hp, 10**10, stream)
    torch.cuda.synchronize()
    waited = (pc() - t0) / K * 1e6
    assert int(st._stats_np[7]) == want[-1][1]

    st = start.clone(); torch.cuda.synchronize()
    t0 = pc()
    got = []
    for j in range(K):
        s = eng.update(st, LodDecide(seq.config, cam_cycle[j], seq.mesh), epoch=j)
        got.append((s.live_before, s.live_after, s.splits_applied, s.merges_applied))
    torch.cuda.synchronize()
    api = (pc() - t0) / K * 1e6
    assert got == want
    print(f"trial {trial}: one launch {one_launch:.1f} | K queued launches {queued:.1f} | launch + wait per frame {waited:.1f} | "
          f"ParallelEngine.update {api:.1f}   (us/frame)")
