import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench
from paper_2407_02215_b200 import _lib
from paper_2407_02215_b200.pipeline import ParallelEngine
from paper_2407_02215_b200.state import initialize
seq, down, cycle = bench.sweep_params(26, 0.0)
eng = ParallelEngine()
st = initialize(seq.mesh, 26)
eng.run_lod_sequence(st, down)
eng.run_lod_sequence(st, bench.step_params(cycle, 0, 8))
for f in (8, 20, 40, 60):
    rows = eng.run_lod_sequence(st, bench.step_params(cycle, f, 1)) if f == 8 else eng.run_lod_sequence(st, bench.step_params(cycle, prev + 1, f - prev))
    prev = f
    r = rows[-1]
    n = r.live_before
    live = st.d_cache_live[:n].to(torch.int64)
    cmd = st.d_commands[live].cpu().numpy().astype(np.uint32)
    split = (cmd & 7) != 0
    merge = ((cmd & 7) == 0) & ((cmd & 8) != 0)       # MERGE bit (requested; agreed ones are a subset)
    cons = split | merge
    nch = (n + 255) // 256
    per = np.add.reduceat(cons.astype(np.int64), np.arange(0, n, 256))
    persm = np.zeros(148, np.int64)
    for c in range(nch):
        persm[(c % 296) % 148] += per[c]      # CTA bid -> SM (bid mod 148, approx)
    print(f"frame {f}: live {n}, splits {split.sum()}, merge requests {merge.sum()}, applied S {r.splits_applied} M {r.merges_applied}; "
          f"consumed per chunk: mean {per.mean():.1f} max {per.max()} p90 {np.percentile(per,90):.0f}; per SM: mean {persm.mean():.0f} max {persm.max()}")
