import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_02215_b200 import _lib
L = _lib.load()
dev = torch.device("cuda", 0)
for depth in (26, 28, 30):
    n = 1 << depth
    bits = [torch.randint(-2 ** 63, 2 ** 63 - 1, (n // 64,), dtype=torch.int64, device=dev) for _ in range(4)]
    cnt = torch.zeros(L.cbtm_counter_words(depth), dtype=torch.int32, device=dev)
    ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    best = []
    for r in range(8):
        flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(4):
            L.cbtm_sum_reduce(bits[k].data_ptr(), cnt.data_ptr(), depth, ws.data_ptr(), 1024, st)
        b.record(); torch.cuda.synchronize()
        best.append(a.elapsed_time(b) / 4)
        ws.zero_()
    print(depth, "us per launch (b2b of 4, cold):", round(sorted(best)[len(best)//2] * 1e3, 2))
