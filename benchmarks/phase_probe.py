"""Work vs barrier wait per phase of the frame kernel.  Needs a library built with -DCBTM_DEBUG_TIMING
(every CTA records when its work of a phase ends):
    nvcc ... -DCBTM_DEBUG_TIMING -o paper_2407_02215_b200/libcbtm.so paper_2407_02215_b200/csrc/cbtm.cu
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 26
seq, down, cycle = bench.sweep_params(depth, 0.0)
eng = ParallelEngine()
state = initialize(seq.mesh, depth)
eng.run_lod_sequence(state, down)
eng.run_lod_sequence(state, bench.step_params(cycle, 0, 8))
prm = bench.step_params(cycle, 8, 64)
L = _lib.load()
d_stats = torch.zeros((64, _lib.STATS_WORDS), dtype=torch.int64, device=state.device)
pool = state.c_pool()
_lib.check(L.cbtm_run_lod_sequence(C.byref(pool), _lib.ptr(state.d_root_tris), prm.ctypes.data, 64,
                                   _lib.ptr(d_stats), state.stream()), "seq")
torch.cuda.synchronize()
rows = d_stats.cpu().numpy()
print(f"{'phase':26s} {'total us':>9s} {'latest work end us':>19s} {'barrier + skew us':>18s}")
for k, name in enumerate(_lib.PHASE_NAMES):
    tot, work = rows[:, 16 + k].mean() / 1e3, rows[:, 22 + k].mean() / 1e3
    print(f"{name:26s} {tot:9.2f} {work:19.2f} {tot - work:18.2f}")
for k, name in enumerate(("reserve: latest CTA enters", "reserve: window block found", "reserve: slots expanded")):
    print(f"{name:26s} {'':9s} {rows[:, 28 + k].mean() / 1e3:19.2f}")
print(f"{'frame':26s} {rows[:, 16:22].sum(axis=1).mean() / 1e3:9.2f}")
