"""Timeline of a back-to-back series of k_sum_reduce launches (the series bench.py times as one CUDA
graph): where do the microseconds between the launches go?  Needs a library built with
-DCBTM_DEBUG_TIMING (into /tmp, the in-tree library is not touched):

    python benchmarks/reduce_chain_probe.py [depth ...]

Four launches on four cold copies, captured as one graph; per launch: first CTA entry, median release
from griddepcontrol.wait, first / last tile landed, last tile counted, all in us since the first
launch's first entry (%globaltimer)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C
import numpy as np
import torch
from paper_2407_02215_b200 import _lib, build

dbg = "/tmp/libcbtm_dbg.so"
cmd = [build.nvcc_path(), *[f for f in build.NVCC_FLAGS if f not in ("-Xptxas", "-v")], "-DCBTM_DEBUG_TIMING", "-o", dbg,
       os.path.join(build.CSRC, "cbtm.cu"), "-ccbin", "/usr/bin/g++"]
subprocess.check_call(cmd)
_lib.LIB_PATH = dbg
L = _lib.load()
L.cbtm_debug_reduce_stamps.argtypes = [C.c_void_p, C.c_int]
from benchmarks.cbt_microbench import device_bits, flush_l2
dev = torch.device("cuda", 0)
flush = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
ws = torch.zeros(2048, dtype=torch.uint8, device=dev)
base = (ws.data_ptr() + 1023) // 1024 * 1024
NL = int(os.environ.get("CHAIN", "4"))     # launches per series; the debug build keeps the stamps of the LAST four (slots by ticket address)
WARM = "--warm" in sys.argv     # no L2 flush between the repetitions: everything the launches read sits in L2
for depth in [int(a) for a in sys.argv[1:] if a.isdigit()] or [24, 26, 28]:
    bits = [device_bits(depth, 0.5, False, dev)]
    bits += [bits[0].clone() for _ in range(NL - 1)]
    cnts = [torch.zeros(L.cbtm_counter_words(depth), dtype=torch.int32, device=dev) for _ in range(NL)]
    side = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        for k in range(NL):
            assert L.cbtm_sum_reduce(bits[k].data_ptr(), cnts[k].data_ptr(), depth, base + 256 * k, 256, side.cuda_stream) == 0
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=side):
            for k in range(NL):
                assert L.cbtm_sum_reduce(bits[k].data_ptr(), cnts[k].data_ptr(), depth, base + 256 * k, 256,
                                         torch.cuda.current_stream().cuda_stream) == 0
    torch.cuda.synchronize()
    for rep in range(4):
        if not WARM:
            flush_l2(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize()
    tiles = max(1, (1 << depth) >> 17)
    st = np.zeros((4 * 2048, 5), dtype=np.uint64)
    assert L.cbtm_debug_reduce_stamps(st.ctypes.data, 4 * 2048) == 0
    rows = [st[(k % 4) * 2048:(k % 4 + 1) * 2048] for k in range(NL - 4, NL)]
    rows = [r[r[:, 0] > 0] for r in rows]
    t0 = min(int(r[:, 0].min()) for r in rows)
    sm_load = np.bincount(rows[-1][:, 4].astype(np.int64), minlength=148)
    print(f"D={depth}: {tiles} tiles, {len(rows[0])} CTAs, graph of {NL}: {a.elapsed_time(b) * 1e3 / NL:.2f} us per launch; "
          f"CTAs per SM of launch 1: min {sm_load[sm_load > 0].min()} max {sm_load.max()} on {int((sm_load > 0).sum())} SMs")
    for k, r in enumerate(rows, NL - 4):
        rel = (r[:, :4].astype(np.int64) - t0) / 1e3
        print(f"   launch {k}: entry {rel[:, 0].min():6.2f}..{rel[:, 0].max():6.2f}  released {rel[:, 1].min():6.2f}/"
              f"{np.median(rel[:, 1]):6.2f}/{rel[:, 1].max():6.2f}  first tile {rel[:, 2].min():6.2f}/{np.median(rel[:, 2]):6.2f}/"
              f"{rel[:, 2].max():6.2f}  counted {rel[:, 3].min():6.2f}/{np.median(rel[:, 3]):6.2f}/{rel[:, 3].max():6.2f}")
    del bits, cnts
