"""Finer timeline of the frame kernel (debug build, -DCBTM_DEBUG_TIMING compiled into /tmp): latest arrival
of any CTA at a dozen points of the frame, averaged over the frames of a sequence run.
    python benchmarks/probe_phases.py [depth]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C
import numpy as np
import torch
from paper_2407_02215_b200 import _lib, build

dbg = "/tmp/libcbtm_dbg.so"
subprocess.check_call([build.nvcc_path(), *[f for f in build.NVCC_FLAGS if f not in ("-Xptxas", "-v")], "-DCBTM_DEBUG_TIMING",
                       "-o", dbg, os.path.join(build.CSRC, "cbtm.cu"), "-ccbin", "/usr/bin/g++"])
_lib.LIB_PATH = dbg
L = _lib.load()
L.cbtm_debug_probes.argtypes = [C.c_void_p, C.c_int]
import bench
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 26
seq, down, cycle = bench.sweep_params(depth, 0.0)
eng = ParallelEngine()
state = initialize(seq.mesh, depth)
eng.run_lod_sequence(state, down)
eng.run_lod_sequence(state, bench.step_params(cycle, 0, 8))
buf = np.zeros((128, 32), dtype=np.uint64)
L.cbtm_debug_probes(buf.ctypes.data, 1)
K = 64
rows = eng.run_lod_sequence(state, bench.step_params(cycle, 8, K))
torch.cuda.synchronize()
L.cbtm_debug_probes(buf.ctypes.data, 1)
t = buf[:K].astype(np.int64)
names = {0: "frame start", 7: "  index: work done (latest CTA)", 1: "P2 start (classify)", 8: "  gathers issued", 9: "  verdicts + needs known",
         10: "  commands scattered", 2: "P3 start (agree)", 12: "  window table built (CTA nb-1)", 13: "  agreement done (latest CTA)",
         3: "P4 start (reserve)", 14: "  prefix known", 15: "  window block found", 27: "  first block's bits arrived (latest warp)", 28: "  blocks expanded (latest warp)", 16: "  slots expanded", 17: "  reserve done",
         4: "P5 start (apply)", 18: "  neighbour bundles arrived (splits and merges, latest warp)", 19: "  parents arrived", 25: "  splits: stores issued", 21: "  merges: members arrived", 26: "  merges: stores issued", 20: "  apply done", 5: "P6 start (reduce)", 22: "  reduce done", 6: "frame end (after last barrier)"}
order = [0, 7, 1, 8, 9, 10, 2, 12, 13, 3, 14, 15, 27, 28, 16, 17, 4, 21, 18, 19, 25, 26, 20, 5, 22, 6]
print(f"2^{depth} pool, {K} frames, live {np.mean([r.live_before for r in rows]):.0f}: us since frame start (mean over frames)")
prev = None
for k in order:
    ok = t[:, k] > 0
    rel = (t[ok, k] - t[ok, 0]) / 1e3
    print(f"{names[k]:62s} {rel.mean():7.2f}" + (f"   (+{rel.mean() - prev:5.2f})" if prev is not None else ""))
    prev = rel.mean()
