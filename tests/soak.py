"""Soak: a long camera loop (ground <-> space, many periods) on the GPU in one launch per 512 frames against the
CPU oracle frame by frame (counters) and array by array at the end.  Not part of the test suite (minutes).

    python tests/soak.py [--depth 22] [--frames 2048]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import oracle
from oracle import OraclePool, OracleVerdict
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize

ap = argparse.ArgumentParser()
ap.add_argument("--depth", type=int, default=22)
ap.add_argument("--frames", type=int, default=2048)
args = ap.parse_args()
seq, down, cycle = bench.sweep_params(args.depth, 0.0)
prm = np.concatenate([down, bench.step_params(cycle, 0, args.frames - len(down))])
st = initialize(seq.mesh, args.depth, exact_free_cache=False)
eng = ParallelEngine()
rows = []
for f0 in range(0, len(prm), 512):
    rows += eng.run_lod_sequence(st, prm[f0:f0 + 512], first_epoch=f0)
op = OraclePool(seq.mesh, args.depth)
threads = oracle.max_threads()
bad = 0
for f in range(len(prm)):
    s, _ = op.update(OracleVerdict.lod(seq.mesh, prm[f]), threads=threads, fast_setup=True)
    r = rows[f]
    got = (r.splits_rejected_oom, r.merges_rejected_oom, r.splits_applied, r.merges_applied, r.split_allocs,
           r.merge_allocs, r.live_before, r.live_after)
    if got != tuple(int(x) for x in s):
        bad += 1
        if bad < 5:
            print("frame", f, got, tuple(int(x) for x in s))
host = st.to_host()
diff = [k for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter", "cache_live", "nodes")
        if not np.array_equal(host[k], getattr(op, k))]
print(f"soak: {len(prm)} frames at 2^{args.depth}: {bad} frames with different counters, arrays that differ: {diff}; "
      f"live {rows[-1].live_after}, max live {max(r.live_after for r in rows)}, poison {sum(r.poison for r in rows)}, "
      f"oom {sum(r.splits_rejected_oom + r.merges_rejected_oom for r in rows)}")
sys.exit(1 if bad or diff else 0)
