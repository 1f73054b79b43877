"""Small, fixed launch sequences for ncu captures (profiles/): one target per invocation.

    python benchmarks/ncu_targets.py frames      # k_frames<2>: 2^26 Earth sweep, 3 frames per launch, 3 launches
    python benchmarks/ncu_targets.py wide        # k_frames<4>: 1 M live bisectors (2^22 pool), 2 frames per launch
    python benchmarks/ncu_targets.py batch       # k_frames_batch: 8 planets x 2^24, 3 frames per launch
    python benchmarks/ncu_targets.py reduce D    # k_sum_reduce on a random 2^D bitfield (stamped tree), 3 launches
    python benchmarks/ncu_targets.py index D     # k_index<false>, decode-all (both lists), 2 launches
    python benchmarks/ncu_targets.py decode D    # k_decode<true>: 2^20 random ranks, 3 launches
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import torch
import bench
from paper_2407_02215_b200 import _lib, halfedge
from paper_2407_02215_b200.pipeline import KeepAll, ParallelEngine, UniformSplit, run_lod_sequence_batch
from paper_2407_02215_b200.state import initialize

target = sys.argv[1]
D = int(sys.argv[2]) if len(sys.argv) > 2 else 28
dev = torch.device("cuda", 0)
L = _lib.load()
eng = ParallelEngine()
stream = torch.cuda.current_stream(dev).cuda_stream

if target == "frames":
    seq, down, cycle = bench.sweep_params(26, 0.0)
    st = initialize(seq.mesh, 26)
    eng.run_lod_sequence(st, down)
    for k in range(3):
        eng.run_lod_sequence(st, bench.step_params(cycle, 3 * k, 3))
elif target == "wide":
    st = initialize(halfedge.icosphere(1.0, 1), 22)
    for e in range(13):
        eng.update(st, UniformSplit(12), epoch=e)      # one launch per epoch: the wide grid takes over above 150 k live
    assert st.c_pool().flags & _lib.POOL_WIDE_GRID
    for k in range(3):
        eng.run_epochs(st, KeepAll(), 2)
elif target == "batch":
    seqs, downs, cycles = zip(*[bench.sweep_params(24, 45.0 * p) for p in range(8)])
    states = [initialize(s.mesh, 24) for s in seqs]
    run_lod_sequence_batch(states, list(downs))
    for k in range(3):
        run_lod_sequence_batch(states, [bench.step_params(c, 3 * k, 3) for c in cycles])
else:
    bits = bench.random_bits(torch, dev, D, 1000 * D + 50)
    cnt = torch.zeros(L.cbtm_counter_words(D), dtype=torch.int32, device=dev)
    ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
    assert L.cbtm_sum_reduce(bits.data_ptr(), cnt.data_ptr(), D, ws.data_ptr(), 1024, stream) == 0   # builds + stamps
    torch.cuda.synchronize()
    if target == "reduce":
        for k in range(3):
            assert L.cbtm_sum_reduce(bits.data_ptr(), cnt.data_ptr(), D, ws.data_ptr(), 1024, stream) == 0
    elif target == "index":
        n = 1 << D
        live = torch.empty(n, dtype=torch.int32, device=dev)
        free = torch.empty(n, dtype=torch.int32, device=dev)
        for k in range(2):
            assert L.cbtm_index(bits.data_ptr(), cnt.data_ptr(), D, live.data_ptr(), free.data_ptr(), 0, stream) == 0
    elif target == "decode":
        ones = int(cnt[1].item())
        K = 1 << 20
        ranks = torch.randint(0, ones, (K,), dtype=torch.int64, device=dev)
        out = torch.empty(K, dtype=torch.int32, device=dev)
        for k in range(3):
            assert L.cbtm_decode_ones(bits.data_ptr(), cnt.data_ptr(), D, ranks.data_ptr(), K, out.data_ptr(), stream) == 0
    else:
        raise SystemExit(f"unknown target {target}")
torch.cuda.synchronize()
print("done", target)
