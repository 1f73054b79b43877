"""Host cost of one cbtm_update call, piece by piece."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.lod import LodDecide
from paper_2407_02215_b200.pipeline import ParallelEngine, lod_verdict
from paper_2407_02215_b200.state import initialize

if os.environ.get("CBTM_DEBUG_LIB"):
    import subprocess
    from paper_2407_02215_b200 import build
    dbg = "/tmp/libcbtm_dbg.so"
    subprocess.check_call([build.nvcc_path(), *[f for f in build.NVCC_FLAGS if f not in ("-Xptxas", "-v")], "-DCBTM_DEBUG_TIMING",
                           "-o", dbg, os.path.join(build.CSRC, "cbtm.cu"), "-ccbin", "/usr/bin/g++"])
    _lib._lib = None
    _lib.LIB_PATH = dbg
seq, down, cycle = bench.sweep_params(24, 0.0)
eng = ParallelEngine()
st = initialize(seq.mesh, 24)
eng.run_lod_sequence(st, down)
L = _lib.load()
pc = time.perf_counter
N = 2000
t0 = pc()
for _ in range(N):
    L.cbtm_abi_version()
print(f"ctypes call, no arguments:            {(pc() - t0) / N * 1e6:.2f} us")
t0 = pc()
for _ in range(N):
    L.cbtm_workspace_bytes(20)
print(f"ctypes call, one int argument:        {(pc() - t0) / N * 1e6:.2f} us")
cv = lod_verdict(st, LodDecide(seq.config, seq.cameras[70], seq.mesh)._prm_b)
pref = st.c_pool_ref(); stream = st.stream(); hp = st._stats_host_ptr
t0 = pc()
for _ in range(N):
    L.cbtm_wait_frame(hp, 0, 1000)
print(f"cbtm_wait_frame (already there):      {(pc() - t0) / N * 1e6:.2f} us")
for K in (8, 64):
    torch.cuda.synchronize()
    t0 = pc()
    for _ in range(K):
        L.cbtm_update(pref, cv, stream)
    dt = pc() - t0
    torch.cuda.synchronize()
    print(f"cbtm_update, {K} calls queued:          {dt / K * 1e6:.2f} us per call")
    if os.environ.get("CBTM_DEBUG_LIB"):
        L.cbtm_debug_launch_ns.restype = C.c_longlong
        print(f"   of which inside cudaLaunchKernelExC: {L.cbtm_debug_launch_ns(1) / 1e3:.2f} us")
torch.cuda.synchronize()
t0 = pc()
for _ in range(64):
    L.cbtm_update_begin(pref, stream)
dt = pc() - t0
torch.cuda.synchronize()
print(f"cbtm_update_begin (plain launch):     {dt / 64 * 1e6:.2f} us per call")
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    s2 = st.stream()
    for K in (8, 64):
        torch.cuda.synchronize()
        t0 = pc()
        for _ in range(K):
            L.cbtm_update(pref, cv, s2)
        dt = pc() - t0
        torch.cuda.synchronize()
        print(f"cbtm_update on a non-default stream, {K} calls queued: {dt / K * 1e6:.2f} us per call")
    t0 = pc()
    for _ in range(64):
        L.cbtm_update_begin(pref, s2)
    dt = pc() - t0
    torch.cuda.synchronize()
    print(f"cbtm_update_begin on a non-default stream:            {dt / 64 * 1e6:.2f} us per call")
