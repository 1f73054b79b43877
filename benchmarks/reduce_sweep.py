#!/usr/bin/env python
"""Full sum reduction (k_sum_reduce) against the HBM roofline, D = 20..30, cold and batched
(8 back-to-back launches on 8 cold copies, L2 flushed by reads between repetitions), in both
modes of the kernel: `delta` (stamped tree: per-tile atomic deltas into the levels above the
tile roots) and `rebuild` (unstamped tree: last-CTA pass).

    python benchmarks/reduce_sweep.py [--depths 20 22 24 26 28 30] [--batch 16] [--env CBTM_REDUCE_NO_PREFETCH ...]

--env runs the sweep once more per measurement hook of the library (CBTM_REDUCE_NO_PREFETCH,
CBTM_REDUCE_NO_PDL: read once per process, hence a subprocess each).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def sweep(depths, reps, out, batch_override=0):
    import torch
    from paper_2407_02215_b200 import _lib
    from benchmarks.cbt_microbench import device_bits, flush_l2
    dev = torch.device("cuda", 0)
    L = _lib.load()
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ws = torch.zeros(1024, dtype=torch.uint8, device=dev)
    lut = torch.tensor([bin(i).count("1") for i in range(256)], dtype=torch.int64, device=dev)
    rows = []
    for depth in depths:
        n = 1 << depth
        nb = batch_override or (8 if depth <= 28 else 4)
        bits = device_bits(depth, 0.5, False, dev)
        want = 0
        for lo in range(0, bits.numel(), 1 << 22):
            want += int(lut[bits[lo:lo + (1 << 22)].view(torch.uint8).to(torch.int64)].sum().item())
        bits_k = [bits] + [bits.clone() for _ in range(nb - 1)]
        cnt_k = [torch.zeros(L.cbtm_counter_words(depth), dtype=torch.int32, device=dev) for _ in range(nb)]
        nbytes = n // 8 + 4 * L.cbtm_counter_words(depth)

        def launch(k):
            assert L.cbtm_sum_reduce(bits_k[k].data_ptr(), cnt_k[k].data_ptr(), depth, ws.data_ptr(), 1024, stream) == 0

        res = {}
        # the batch as ONE CUDA graph (the programmatic-dependent-launch edges are captured with it):
        # the GPU runs the launches back to back, the host's per-call cost (ctypes + launch, ~3 us)
        # is out of the picture
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            gstream = side.cuda_stream
            for k in range(nb):      # warm-up outside capture
                assert L.cbtm_sum_reduce(bits_k[k].data_ptr(), cnt_k[k].data_ptr(), depth, ws.data_ptr(), 1024, gstream) == 0
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=side):
                for k in range(nb):
                    assert L.cbtm_sum_reduce(bits_k[k].data_ptr(), cnt_k[k].data_ptr(), depth, ws.data_ptr(), 1024,
                                             torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        for mode in ("rebuild", "delta"):
            for batch in (1, nb, -nb):
                samples = []
                for r in range(reps + 3):
                    if mode == "rebuild":
                        for c in cnt_k:
                            c[0] = 0        # no stamp: the last CTA rebuilds the upper levels
                    flush_l2(flush)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    if batch < 0:
                        graph.replay()
                    else:
                        for k in range(batch):
                            launch(k)
                    b.record()
                    torch.cuda.synchronize()
                    if r >= 3:
                        samples.append(a.elapsed_time(b) * 1e3 / abs(batch))
                res[(mode, batch)] = float(np.median(samples))
            for c in cnt_k:
                assert int(c[1].item()) == want, (depth, mode, int(c[1].item()), want)
                assert torch.equal(c, cnt_k[0])
        # the delta path must also follow a CHANGED bitfield: flip bits, reduce again, compare with a rebuild
        bits_k[0][::7] ^= 0x5A5A5A5A
        launch(0)
        ref = torch.zeros_like(cnt_k[0])
        assert L.cbtm_sum_reduce(bits_k[0].data_ptr(), ref.data_ptr(), depth, ws.data_ptr(), 1024, stream) == 0
        assert torch.equal(ref, cnt_k[0]), f"delta update disagrees with a rebuild at D={depth}"
        row = {"depth": depth, "bytes": nbytes, "batch": nb}
        for (mode, batch), us in res.items():
            tag = f"{mode}_{'graph' if batch < 0 else 'batched' if batch > 1 else 'single'}"
            row[tag + "_us"] = us
            row[tag + "_frac"] = nbytes / us / 1e3 / peak
        rows.append(row)
        print(f"D={depth:2d} {nbytes / 1e6:7.1f} MB | delta: single {row['delta_single_us']:6.1f} us ({row['delta_single_frac']:.2f})"
              f" batched {row['delta_batched_us']:6.1f} us ({row['delta_batched_frac']:.2f}) graph {row['delta_graph_us']:6.1f} us "
              f"({row['delta_graph_frac']:.2f}) | rebuild: single "
              f"{row['rebuild_single_us']:6.1f} us ({row['rebuild_single_frac']:.2f}) batched {row['rebuild_batched_us']:6.1f} us "
              f"({row['rebuild_batched_frac']:.2f}) graph {row['rebuild_graph_us']:6.1f} us ({row['rebuild_graph_frac']:.2f})", flush=True)
        del bits, bits_k, cnt_k
        torch.cuda.empty_cache()
    if out:
        with open(out, "w") as fh:
            json.dump({"peak_gbs": peak, "rows": rows}, fh, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depths", type=int, nargs="+", default=[20, 22, 24, 26, 28, 30])
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--env", nargs="*", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=0, help="launches (and cold copies) per series; default 8, 4 beyond 2^28")
    args = ap.parse_args()
    sweep(args.depths, args.reps, args.out, args.batch)
    for hook in args.env or []:
        print(f"--- {hook}=1", flush=True)
        env = dict(os.environ, **{hook: "1"})
        subprocess.run([sys.executable, os.path.abspath(__file__), "--reps", str(args.reps), "--batch", str(args.batch),
                        "--depths", *map(str, args.depths)], env=env, check=False)


if __name__ == "__main__":
    main()
