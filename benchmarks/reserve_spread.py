"""How many leaf blocks does the free-rank interval of one chunk (256 consecutive live ranks) span?
The reserve phase expands those blocks a warp each; python benchmarks/reserve_spread.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize
seq, down, cycle = bench.sweep_params(26, 0.0)
eng = ParallelEngine()
st = initialize(seq.mesh, 26)
eng.run_lod_sequence(st, down)
eng.run_lod_sequence(st, bench.step_params(cycle, 0, 8))
prev = 7
for f in (8, 20, 40, 60):
    rows = eng.run_lod_sequence(st, bench.step_params(cycle, prev + 1, f - prev))
    prev = f
    r = rows[-1]
    n = r.live_before
    live = st.d_cache_live[:n].to(torch.int64)
    cmd = st.d_commands[live].cpu().numpy().astype(np.uint32)
    res = st.d_reserved.view(-1, 4)[live].cpu().numpy()
    sm = cmd & 7
    na = np.where(sm != 0, 2 + ((sm >> 1) & 1) + ((sm >> 2) & 1), 0)
    own = (sm == 0) & ((cmd & 8) != 0) & ((cmd & 32) != 0)          # merge owners (requested; agreed ones allocate)
    spans, totals = [], []
    for c in range(0, n, 256):
        blocks = set()
        tot = 0
        for k in range(c, min(n, c + 256)):
            cnt = na[k] if na[k] else 0
            for q in range(cnt):
                blocks.add(int(res[k, q]) >> 10)
            tot += cnt
        if tot:
            spans.append(len(blocks)); totals.append(tot)
    spans = np.array(spans); totals = np.array(totals)
    print(f"frame {f}: live {n}, chunks that allocate by splits {len(spans)}; slots per chunk mean {totals.mean():.0f} max {totals.max()}; "
          f"leaf blocks spanned per chunk: mean {spans.mean():.1f} p90 {np.percentile(spans, 90):.0f} max {spans.max()}")
