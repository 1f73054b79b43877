import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize
seq, down, cycle = bench.sweep_params(26, 0.0)
eng = ParallelEngine()
st = initialize(seq.mesh, 26)
eng.run_lod_sequence(st, down)
eng.run_lod_sequence(st, bench.step_params(cycle, 0, 8))
rows = eng.run_lod_sequence(st, bench.step_params(cycle, 8, 120))
rows = eng.run_lod_sequence(st, bench.step_params(cycle, 128, 128))
print("live  chunks  index classify agree reserve apply reduce  total(us)")
for r in rows[::4]:
    ph = [x / 1e3 for x in r.phase_ns]
    print(f"{r.live_before:6d} {(r.live_before + 255) // 256:4d}   " + " ".join(f"{x:6.2f}" for x in ph) + f"  {sum(ph):6.2f}  S {r.splits_applied} M {r.merges_applied}")
