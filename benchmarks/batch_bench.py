"""BASELINE config 5 on one GPU: P independent icosphere planets (2^24-slot pools, camera paths
rotated by p * 45 degrees) advanced (a) one after the other and (b) in lockstep inside one
cooperative launch (cbtm_run_lod_sequence_batch).  Device-timed with CUDA events.

    python benchmarks/batch_bench.py [--planets 8] [--depth 24] [--frames 64]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.pipeline import ParallelEngine, run_lod_sequence_batch
from paper_2407_02215_b200.state import initialize

ap = argparse.ArgumentParser()
ap.add_argument("--planets", type=int, default=8)
ap.add_argument("--depth", type=int, default=24)
ap.add_argument("--frames", type=int, default=64)
args = ap.parse_args()
P, K = args.planets, args.frames
dev = torch.device("cuda", 0)
L = _lib.load()
eng = ParallelEngine()
seqs, downs, cycles = zip(*[bench.sweep_params(args.depth, 45.0 * p) for p in range(P)])
timed = [bench.step_params(c, 8, K) for c in cycles]


def fresh():
    states = [initialize(s.mesh, args.depth, device=dev) for s in seqs]
    run_lod_sequence_batch(states, list(downs))
    run_lod_sequence_batch(states, [bench.step_params(c, 0, 8) for c in cycles])
    return states


def timed_run(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


states = fresh()
pools = (_lib.CPool * P)(*[s.c_pool() for s in states])
roots = (C.c_void_p * P)(*[_lib.ptr(s.d_root_tris) for s in states])
pinned = [torch.from_numpy(t).pin_memory() for t in timed]
prms = (C.c_void_p * P)(*[p.data_ptr() for p in pinned])
d_stats = [torch.zeros((K, _lib.STATS_WORDS), dtype=torch.int64, device=dev) for _ in range(P)]
souts = (C.c_void_p * P)(*[_lib.ptr(d) for d in d_stats])
st = states[0].stream()
ms_batch = timed_run(lambda: _lib.check(L.cbtm_run_lod_sequence_batch(pools, P, roots, prms, K, souts, st), "batch"))
rows_b = [d.cpu().numpy().copy() for d in d_stats]

states2 = fresh()
pools2 = [s.c_pool() for s in states2]


def one_by_one():
    for q in range(P):
        _lib.check(L.cbtm_run_lod_sequence(C.byref(pools2[q]), _lib.ptr(states2[q].d_root_tris), pinned[q].data_ptr(), K,
                                           _lib.ptr(d_stats[q]), st), "seq")


ms_seq = timed_run(one_by_one)
rows_s = [d.cpu().numpy() for d in d_stats]
same = all(np.array_equal(a[:, :12], b[:, :12]) for a, b in zip(rows_b, rows_s)) and all(
    torch.equal(getattr(x, "d_" + k), getattr(y, "d_" + k)) for x, y in zip(states, states2)
    for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "bits", "counters"))
units = int(sum(r[:, 6].sum() for r in rows_b))
print(json.dumps({
    "workload": f"config 5: {P} icosphere planets, 2^{args.depth}-slot pools, {K} frames of the ground<->space sweep each",
    "identical_results": bool(same),
    "batched_ms_per_frame_step": ms_batch / K, "sequential_ms_per_frame_step": ms_seq / K,
    "batched_bisectors_per_s": units / (ms_batch * 1e-3), "sequential_bisectors_per_s": units / (ms_seq * 1e-3),
    "speedup": ms_seq / ms_batch,
    "phase_us_batched": {n: float(rows_b[0][:, _lib.STAT_PHASE_NS + k].mean()) / 1e3 for k, n in enumerate(_lib.PHASE_NAMES)},
    "live_per_planet_mean": float(np.mean([r[:, 6].mean() for r in rows_b]))}))
