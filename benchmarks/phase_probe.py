import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, torch, ctypes as C
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize
seq, down, cycle = bench.sweep_params(26, 0.0)
eng = ParallelEngine()
state = initialize(seq.mesh, 26)
eng.run_lod_sequence(state, down)
eng.run_lod_sequence(state, bench.step_params(cycle, 0, 8))
prm = bench.step_params(cycle, 8, 64)
L = _lib.load()
d_stats = torch.zeros((64, _lib.STATS_WORDS), dtype=torch.int64, device=state.device)
pool = state.c_pool()
rc = L.cbtm_run_lod_sequence(C.byref(pool), _lib.ptr(state.d_root_tris), prm.ctypes.data, 64, _lib.ptr(d_stats), state.stream())
torch.cuda.synchronize()
rows = d_stats.cpu().numpy()
names = ["P2:classified(cta0)", "P2:last lookback", "P2:last scattered", "P2:admin total", "P2:admin descent", "P2:admin done", "P3:agreed", "P3:lookback", "P3:expanded", "P3:reserved"]
print("phases us:", rows[:, 16:22].mean(axis=0) / 1e3)
for k, nm in enumerate(names):
    print(f"{nm:24s} mean {rows[:, 22 + k].mean() / 1e3:7.2f} us  max {rows[:, 22 + k].max() / 1e3:7.2f}")
