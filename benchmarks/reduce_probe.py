"""Where does k_sum_reduce spend its time?  Needs a library built with -DCBTM_DEBUG_TIMING (into
/tmp, the in-tree library is not touched):  python benchmarks/reduce_probe.py [depth ...]
Per CTA: kernel entry, release from griddepcontrol.wait, first tile landed, last tile counted."""
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
ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream(dev).cuda_stream
for depth in [int(a) for a in sys.argv[1:]] or [26, 28, 30]:
    bits = device_bits(depth, 0.5, False, dev)
    cnt = torch.zeros(L.cbtm_counter_words(depth), dtype=torch.int32, device=dev)
    for rep in range(4):
        flush_l2(flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        assert L.cbtm_sum_reduce(bits.data_ptr(), cnt.data_ptr(), depth, ws.data_ptr(), 1024, stream) == 0
        b.record()
        torch.cuda.synchronize()
    tiles = max(1, (1 << depth) >> 17)
    n = min(tiles, 2048)
    st = np.zeros((4 * 2048, 5), dtype=np.uint64)
    assert L.cbtm_debug_reduce_stamps(st.ctypes.data, 4 * 2048) == 0
    slot = (ws.data_ptr() >> 8) & 3     # the stamps of a launch go to the slot its ticket pointer selects
    st = st[slot * 2048:slot * 2048 + n]
    st = st[st[:, 0] > 0]
    t0 = st[:, 0].min()
    rel = (st[:, :4].astype(np.int64) - int(t0)) / 1e3
    print(f"D={depth}: {len(st)} CTAs, event time {a.elapsed_time(b) * 1e3:.1f} us; us since the first CTA's entry:")
    for k, name in enumerate(("entry", "released", "first tile landed", "last tile counted")):
        c = rel[:, k]
        print(f"   {name:18s} min {c.min():6.2f}  p10 {np.percentile(c, 10):6.2f}  median {np.median(c):6.2f}  "
              f"p90 {np.percentile(c, 90):6.2f}  max {c.max():6.2f}")
    sm = st[:, 4].astype(np.int64)
    per_sm_end = np.array([rel[sm == s, 3].max() for s in np.unique(sm)])
    print(f"   per-SM finish: min {per_sm_end.min():.2f} median {np.median(per_sm_end):.2f} max {per_sm_end.max():.2f} "
          f"({len(per_sm_end)} SMs used)")
    del bits, cnt
