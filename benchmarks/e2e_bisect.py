"""Which python-side piece of the per-frame path stretches the frame period?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.lod import LodDecide
from paper_2407_02215_b200.pipeline import ParallelEngine, UpdateStats, lod_verdict, _checked
from paper_2407_02215_b200.state import initialize

seq, down, cycle = bench.sweep_params(26, 0.0)
eng = ParallelEngine()
state = initialize(seq.mesh, 26)
eng.run_lod_sequence(state, down)
start = state.clone()
cams = seq.cameras
cam_cycle = cams[bench.SETUP_FRAMES - 1::-1] + cams[:bench.SETUP_FRAMES]
L = _lib.load()
K = 64
pc = time.perf_counter
decs = [LodDecide(seq.config, cam_cycle[j], seq.mesh) for j in range(K)]

def run(name, body):
    best = 1e9
    for rep in range(3):
        st = start.clone()
        torch.cuda.synchronize()
        t0 = pc()
        for j in range(K):
            body(st, j)
        torch.cuda.synchronize()
        best = min(best, (pc() - t0) / K * 1e6)
    print(f"{name:60s} {best:6.1f} us/frame")

def bare(st, j):
    cv = lod_verdict(st, decs[j]._prm_c)
    L.cbtm_update_wait(st.c_pool_ref(), cv, st._stats_host_ptr, 10**10, st.stream())
run("update_wait, prebuilt LodDecide", bare)

def two_calls(st, j):
    cv = lod_verdict(st, decs[j]._prm_c)
    seq0 = int(st._stats_np[_lib.STAT_SEQ])
    L.cbtm_update(st.c_pool_ref(), cv, st.stream())
    L.cbtm_wait_frame(st._stats_host_ptr, seq0 + 1, 10**10)
run("cbtm_update + cbtm_wait_frame (two calls)", two_calls)

cvs = []
for j in range(K):
    cv = _lib.CVerdict()
    cv.mode = _lib.VERDICT_LOD
    cv.root_tris = _lib.ptr(start.d_root_tris)
    C.memmove(cv.prm, decs[j]._prm_c, 8 * 23)
    cvs.append(cv)

def two_calls_distinct_cv(st, j):
    seq0 = int(st._stats_np[_lib.STAT_SEQ])
    L.cbtm_update(st.c_pool_ref(), cvs[j], st.stream())
    L.cbtm_wait_frame(st._stats_host_ptr, seq0 + 1, 10**10)
run("two calls, distinct CVerdict per frame (root_tris of the first state)", two_calls_distinct_cv)

def combined_distinct_cv(st, j):
    L.cbtm_update_wait(st.c_pool_ref(), cvs[j], st._stats_host_ptr, 10**10, st.stream())
run("update_wait, distinct CVerdict per frame", combined_distinct_cv)

def floor_like(st, j):
    if j == 0:
        floor_like.pref = C.byref(st.c_pool()); floor_like.stream = st.stream(); floor_like.hp = st._stats_host_ptr
        floor_like.seq0 = int(st._stats_np[_lib.STAT_SEQ])
    L.cbtm_update(floor_like.pref, C.byref(cvs[j]), floor_like.stream)
    L.cbtm_wait_frame(floor_like.hp, floor_like.seq0 + j + 1, 10**10)
run("as in e2e_floor: everything hoisted", floor_like)

def floor_stream(st, j):
    if j == 0:
        floor_like.pref = C.byref(st.c_pool()); floor_like.hp = st._stats_host_ptr
        floor_like.seq0 = int(st._stats_np[_lib.STAT_SEQ])
    L.cbtm_update(floor_like.pref, C.byref(cvs[j]), st.stream())
    L.cbtm_wait_frame(floor_like.hp, floor_like.seq0 + j + 1, 10**10)
run("hoisted except st.stream()", floor_stream)

def floor_pool(st, j):
    if j == 0:
        floor_like.stream = st.stream(); floor_like.hp = st._stats_host_ptr
        floor_like.seq0 = int(st._stats_np[_lib.STAT_SEQ])
    L.cbtm_update(st.c_pool_ref(), C.byref(cvs[j]), floor_like.stream)
    L.cbtm_wait_frame(floor_like.hp, floor_like.seq0 + j + 1, 10**10)
run("hoisted except st.c_pool_ref()", floor_pool)

def floor_seq(st, j):
    if j == 0:
        floor_like.pref = C.byref(st.c_pool()); floor_like.stream = st.stream(); floor_like.hp = st._stats_host_ptr
    seq0 = int(st._stats_np[_lib.STAT_SEQ])
    L.cbtm_update(floor_like.pref, C.byref(cvs[j]), floor_like.stream)
    L.cbtm_wait_frame(floor_like.hp, seq0 + 1, 10**10)
run("hoisted except the sequence word read per frame", floor_seq)

def plus_touch(st, j):
    bare(st, j)
    st._touched()
run("+ state._touched()", plus_touch)

def plus_stats(st, j):
    plus_touch(st, j)
    _checked(UpdateStats.from_device_words(st._stats_np.tolist(), j))
run("+ UpdateStats", plus_stats)

def plus_decide(st, j):
    d = LodDecide(seq.config, cam_cycle[j], seq.mesh)
    cv = lod_verdict(st, d._prm_c)
    L.cbtm_update_wait(st.c_pool_ref(), cv, st._stats_host_ptr, 10**10, st.stream())
    st._touched()
    _checked(UpdateStats.from_device_words(st._stats_np.tolist(), j))
run("+ LodDecide per frame", plus_decide)

def api(st, j):
    eng.update(st, LodDecide(seq.config, cam_cycle[j], seq.mesh), epoch=j)
run("ParallelEngine.update(LodDecide(...))", api)

def api_pre(st, j):
    eng.update(st, decs[j], epoch=j)
run("ParallelEngine.update(prebuilt)", api_pre)
