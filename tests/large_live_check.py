"""Scale check (script, not collected by pytest): uniform subdivision of the icosphere to depth 13 in a 2^24 pool
-- up to 2 M live bisectors, up to 1 M splits in one frame, allocation windows of thousands of leaf blocks --
GPU (all epochs in one launch) against the CPU oracle: counters every frame, every array at the end; then
steady-state frame time at that size.

    python tests/large_live_check.py [--target 13] [--depth 24]
"""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from oracle import OraclePool, OracleVerdict
from paper_2407_02215_b200 import halfedge
from paper_2407_02215_b200.pipeline import KeepAll, ParallelEngine, UniformSplit
from paper_2407_02215_b200.state import initialize

ap = argparse.ArgumentParser()
ap.add_argument("--target", type=int, default=13)
ap.add_argument("--depth", type=int, default=24)
args = ap.parse_args()
mesh = halfedge.icosphere(1.0, 1)
epochs = args.target + 6
st = initialize(mesh, args.depth)
eng = ParallelEngine()
rows = eng.run_epochs(st, UniformSplit(args.target), epochs)
op = OraclePool(mesh, args.depth)
bad = 0
for e in range(epochs):
    s, _ = op.update(OracleVerdict.uniform(args.target), threads=oracle.max_threads(), fast_setup=True)
    r = rows[e]
    got = (r.splits_rejected_oom, r.merges_rejected_oom, r.splits_applied, r.merges_applied, r.split_allocs,
           r.merge_allocs, r.live_before, r.live_after)
    if got != tuple(int(x) for x in s):
        bad += 1
        print("epoch", e, got, tuple(int(x) for x in s))
host = st.to_host()
diff = [k for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter", "cache_live", "nodes")
        if not np.array_equal(host[k], getattr(op, k))]
print(f"live after each epoch: {[r.live_after for r in rows]}")
print(f"{bad} epochs with different counters; arrays that differ: {diff}; poison {sum(r.poison for r in rows)}")
# steady state: KeepAll frames at full size, device-timed
K = 32
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
eng.run_epochs(st, KeepAll(), 4)
a.record()
keep = eng.run_epochs(st, KeepAll(), K)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / K
n = keep[-1].live_after
print(f"steady state: {n} live bisectors, {ms * 1e3:.1f} us per KeepAll frame, {n / ms / 1e6:.1f} G bisectors/s; "
      f"phases us: {[round(x / 1e3, 1) for x in keep[-1].phase_ns]}")
big = max(rows, key=lambda r: r.splits_applied)
print(f"largest frame: {big.splits_applied} splits, {big.split_allocs} slots allocated, "
      f"{sum(big.phase_ns) / 1e3:.1f} us; phases us: {[round(x / 1e3, 1) for x in big.phase_ns]}")
sys.exit(1 if bad or diff else 0)
