"""Where the end-to-end frame time goes on the host side (ParallelEngine.update, LOD source)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.lod import LodDecide
from paper_2407_02215_b200.pipeline import ParallelEngine, UpdateStats
from paper_2407_02215_b200.state import initialize

seq, down, cycle = bench.sweep_params(26, 0.0)
eng = ParallelEngine()
state = initialize(seq.mesh, 26)
eng.run_lod_sequence(state, down)
cams = seq.cameras
cam_cycle = cams[bench.SETUP_FRAMES - 1::-1] + cams[:bench.SETUP_FRAMES]
L = _lib.load()
K = 64
T = {k: 0.0 for k in ("decide", "pre", "launch", "wait", "post")}
pc = time.perf_counter
t_all0 = pc()
for j in range(K):
    t0 = pc()
    d = LodDecide(seq.config, cam_cycle[j % len(cam_cycle)], seq.mesh)
    t1 = pc()
    pool = state.c_pool(); stream = state.stream()
    seq_before = int(state._stats_np[_lib.STAT_SEQ])
    cv = d.device_verdict(state)
    t2 = pc()
    L.cbtm_update(C.byref(pool), C.byref(cv), stream)
    t3 = pc()
    L.cbtm_wait_frame(state._stats_host_ptr, seq_before + 1, 10**10)
    t4 = pc()
    words = state._stats_np.tolist()
    state._touched()
    s = UpdateStats.from_device_words(words, j)
    t5 = pc()
    T["decide"] += t1 - t0; T["pre"] += t2 - t1; T["launch"] += t3 - t2; T["wait"] += t4 - t3; T["post"] += t5 - t4
t_all = pc() - t_all0
print({k: round(v / K * 1e6, 2) for k, v in T.items()}, "total us/frame", round(t_all / K * 1e6, 2))
print("device phase sum us", sum(s.phase_ns) / 1e3)
