"""Runs the standalone CBT kernels a few times at one depth (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02215_b200 import _lib
depth = int(sys.argv[1]) if len(sys.argv) > 1 else 30
what = sys.argv[2] if len(sys.argv) > 2 else "reduce"
L = _lib.load()
dev = torch.device("cuda", 0)
n = 1 << depth
gen = torch.Generator(device=dev); gen.manual_seed(depth)
bits = torch.randint(-2 ** 63, 2 ** 63 - 1, (max(n // 64, 16),), dtype=torch.int64, device=dev, generator=gen)
cnt = torch.zeros(L.cbtm_counter_words(depth), dtype=torch.int32, device=dev)
ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(dev).cuda_stream
for _ in range(3):
    assert L.cbtm_sum_reduce(bits.data_ptr(), cnt.data_ptr(), depth, ws.data_ptr(), 1024, st) == 0
if what == "index":
    live = torch.empty(n, dtype=torch.int32, device=dev)
    free = torch.empty(n, dtype=torch.int32, device=dev)
    for _ in range(3):
        assert L.cbtm_index(bits.data_ptr(), cnt.data_ptr(), depth, live.data_ptr(), free.data_ptr(), 0, st) == 0
torch.cuda.synchronize()
print("ok", int(cnt[1]))
