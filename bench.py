#!/usr/bin/env python
"""bench.py -- per-frame bisector update on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload earth|batch]

A *step* is one full nine-stage update (index + classify + admit + split/merge +
bitfield + sum reduction) for one camera frame.

workload `earth` (default at N = 1): BASELINE config 3, ONE Earth-scale icosphere planet
  on a 2^26-slot pool, LOD camera sweeping between the ground (10 m) and space (3 R).
  Untimed setup flies the camera down to the ground (64 frames); the warm-up and timed
  steps ride the ground<->space sweep (period 128 frames), so the pool keeps splitting
  and merging for any K.
workload `batch` (default at N > 1): BASELINE config 5, EIGHT independent icosphere
  planets on 2^24-slot pools (paths rotated by p * 45 degrees), planet p on rank p mod N
  (`batch.run_planet_batch`); a step advances every planet by one frame; the planets of a
  rank run in lockstep inside one launch; no data-path collective, one final all_gather
  of the per-frame stats (NCCL).  Total work is fixed: strong scaling.
`--gpus N` without a torchrun environment re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU).

Reported on ONE JSON line (rank 0):
  value / ms_per_step  device-timed (CUDA events on the launch stream) K-step run with the
                       camera parameters already resident in HBM, no host synchronisation
                       between frames
  e2e                  the same K frames through the public python API with host inputs:
                       earth: `ParallelEngine().update(state, LodDecide(config, camera, mesh))`
                       per frame (default engine, nothing subtracted: the clock runs from
                       before the first update until the stream has drained after the last);
                       batch: `pipeline.run_lod_sequence_batch` (parameters uploaded, stats
                       downloaded inside the timed region)
  roofline             earth: the persistent frame kernel k_frames (the only kernel of the
                       timed region) against the HBM roofline, algorithmic bytes as
                       SURVEY.md 8(d) defines them; `traffic` from the ncu capture recorded in
                       profiles/kframes_traffic.json.  cbt_kernels_d26 / config4 time the
                       full-pool CBT kernels (sum reduction, decode-all) alone, where they
                       are HBM bound, next to the CPU port on the same bitfield
  cpu_baseline         the REAL reference (`cbtmesh` from baseline/_ref, all host threads)
                       on a bounded sample of the same frames, from the same pool state
                       (kind "reference"); `cpu_port` = the C/OpenMP port of the reference
                       path (oracle/) on more frames; `cpu_reference` = the reference at
                       1 thread and all threads, also on BASELINE config 2

--impl reference runs the reference's CPU implementation of the path on the same workload:
the real `cbtmesh.pipeline.ParallelEngine(threads=cpu_count)` when baseline/_ref is present
(kind "reference"), else the C port (kind "port").  CPU only, none of the CUDA code.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "update ms/frame & bisectors/s (classify+split/merge+CBT reduce+index)"
UNIT = "bisectors/s"
SETUP_FRAMES = 64
BATCH_PLANETS = 8
BATCH_DEPTH = 24
DTYPE = "int32/u64 + f64 classifier"


def sweep_params(depth: int, rotate_deg: float):
    """(sequence, descent prm[64,23], cyclic sweep prm[128,23])."""
    from paper_2407_02215_b200 import workloads
    seq = workloads.earth_sweep(depth=depth, frames=SETUP_FRAMES, rotate_deg=rotate_deg)
    prm = seq.params()
    down = prm[:SETUP_FRAMES]
    cycle = np.concatenate([down[::-1], down])  # ascent, then descent again
    return seq, down, cycle


def step_params(cycle: np.ndarray, first: int, count: int) -> np.ndarray:
    idx = (first + np.arange(count)) % cycle.shape[0]
    return np.ascontiguousarray(cycle[idx])


def step_cameras(seq, first: int, count: int) -> list:
    cams = seq.cameras
    cam_cycle = cams[SETUP_FRAMES - 1::-1] + cams[:SETUP_FRAMES]
    return [cam_cycle[(first + j) % len(cam_cycle)] for j in range(count)]


def load_peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(depth: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of k_frames per frame, from the ncu
    capture recorded (with the commit it was taken at) in profiles/kframes_traffic.json."""
    path = os.path.join(ROOT, "profiles", "kframes_traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
        row = rec["pools"][str(depth)]
        return row["dram_bytes_per_frame"], (f"{rec['source']} at commit {rec['commit']}: "
                                             f"{row['note']}")
    except (OSError, KeyError, ValueError):
        return None, "no ncu capture on record for this pool depth (profiles/kframes_traffic.json)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.rows = []
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def wait_first(self, seconds: float):
        """Block until nvidia-smi has delivered its first sample (or give up)."""
        t0 = time.time()
        while self.proc is not None and not self.rows and time.time() - t0 < seconds:
            time.sleep(0.01)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for name, cell in zip(names, r[5:9]):
                if cell.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU arms: the real reference (baseline/_ref) and the C port (oracle/)
# ---------------------------------------------------------------------------

def oracle_pool_from_host(mesh, depth, host_arrays):
    from oracle import OraclePool
    op = OraclePool(mesh, depth)
    for k, v in host_arrays.items():
        getattr(op, k)[...] = v
    return op


def port_sample(op, mesh, prms, threads):
    """Time len(prms) genuine frames of the C port; returns (seconds, stats rows)."""
    from oracle import OracleVerdict
    rows, total = [], 0.0
    for prm in prms:
        t0 = time.perf_counter()
        s, _ = op.update(OracleVerdict.lod(mesh, prm), threads=threads)
        total += time.perf_counter() - t0
        rows.append([int(x) for x in s])
    return total, rows


def reference_available() -> bool:
    from baseline import ref_timing
    return ref_timing.available()


def host_arrays_of_oracle(op) -> dict:
    return {k: getattr(op, k) for k in ("ids", "nexts", "prevs", "twins", "commands", "reserved", "counter",
                                        "cache_live", "cache_free", "nodes")}


def workload_config(args, n_gpus, workload):
    if workload == "batch":
        return {"workload": f"planet_batch: {BATCH_PLANETS} icosphere planets (H=240), pools 2^{BATCH_DEPTH} slots, camera "
                            f"paths rotated by p*45 deg, LOD camera ground(10 m)<->space(3R) sweep 1920x1080, 49 px target; "
                            f"{SETUP_FRAMES} untimed descent frames then steps ride the 128-frame cycle",
                "pool_depth": BATCH_DEPTH, "planets": BATCH_PLANETS,
                "parallelism": f"planet p on rank p mod {n_gpus} (round robin), the planets of a rank in lockstep in one "
                               "launch, no collective on the data path, one final all_gather of the stats",
                "l2": "pool state (8 x 0.83 GB) exceeds L2"}
    return {"workload": f"earth_sweep icosphere H=240, pool 2^{args.depth} slots, LOD camera "
                        f"ground(10 m)<->space(3R) sweep 1920x1080, 49 px target; "
                        f"{SETUP_FRAMES} untimed descent frames then steps ride the 128-frame cycle",
            "pool_depth": args.depth, "planets": n_gpus,
            "parallelism": "1 planet per GPU, no collective on the data path",
            "l2": "pool state (3.3 GB) exceeds L2; roofline kernels timed with L2 flushed"}


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path, CPU only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from oracle import OraclePool, OracleVerdict
    threads = oracle.max_threads()
    workload = resolve_workload(args, int(os.environ.get("WORLD_SIZE", str(args.gpus))))
    depth = BATCH_DEPTH if workload == "batch" else args.depth
    planets = range(BATCH_PLANETS) if workload == "batch" else range(1)
    use_ref = reference_available() and not args.port_only
    if use_ref:
        from baseline import ref_timing
        ref_timing.load()
        jit_s = ref_timing.warm_jit(threads)
    seconds, units, port_seconds, port_units = 0.0, 0, 0.0, 0
    W, K = args.warmup, args.steps
    for p in planets:
        seq, down, cycle = sweep_params(depth, 45.0 * p)
        op = OraclePool(seq.mesh, depth)
        for prm in down:  # untimed setup: fast-forward with the port (linear-scan stage 2)
            op.update(OracleVerdict.lod(seq.mesh, prm), threads=threads, fast_setup=True)
        for prm in step_params(cycle, 0, W):
            op.update(OracleVerdict.lod(seq.mesh, prm), threads=threads, fast_setup=True)
        timed = step_params(cycle, W, K)
        if use_ref:
            st = ref_timing.state_from_arrays(seq.mesh, depth, host_arrays_of_oracle(op))
            # one untimed frame on a scratch copy is not affordable at 2^26 (3.5 GB): the JIT is warm, the
            # first timed frame pays only the page faults of the fresh state
            per_frame, ref_rows = ref_timing.time_frames(st, seq.mesh, seq.config, step_cameras(seq, W, K), threads)
            seconds += sum(per_frame)
            units += sum(r[6] for r in ref_rows)
            del st
        n_port = K if not use_ref else min(K, 4)
        sec, rows = port_sample(op, seq.mesh, timed[:n_port], threads)
        # (under reservation pressure the reference at threads > 1 admits in scheduler order --
        #  pipeline.py:7-9 -- so counters are only comparable on frames without rejections)
        pressure = any(r[0] or r[1] for r in rows + (ref_rows[:n_port] if use_ref else []))
        if use_ref and not pressure and rows != ref_rows[:n_port]:
            raise SystemExit("bench.py: the C port and the real reference disagree on the timed frames")
        port_seconds += sec
        port_units += sum(r[6] for r in rows)
        del op
    port = {"value": port_units / port_seconds, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": "the C/OpenMP port of the reference path (oracle/) on the first timed frames of every planet"}
    if use_ref:
        value = units / seconds
        cpu = {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": f"{K} full frames per planet through the unmodified cbtmesh.pipeline.ParallelEngine(threads={threads})"
                         f".update + LodDecide (baseline/_ref), numba kernels JIT-warmed first ({jit_s:.0f} s, untimed); "
                         "setup and warm-up frames fast-forwarded with the C port (identical state, verified on the "
                         "timed frames)",
               "port": port}
    else:
        value, seconds = port["value"], port_seconds
        cpu = dict(port, sample=f"{K} full frames per planet (C/OpenMP port of the reference path: baseline/_ref absent)")
    steps_total = K * len(planets) if workload == "batch" else K
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": K, "warmup": W,
        "ms_per_step": 1e3 * seconds / max(1, K), "higher_is_better": True,
        "scaling": "strong" if workload == "batch" else "weak", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic", "config": workload_config(args, 1 if workload == "earth" else args.gpus, workload),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "frames_timed": steps_total,
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# roofline helpers (GPU)
# ---------------------------------------------------------------------------

def _clean_l2_flush(torch, flush):
    """Evict with READS of a buffer larger than L2 (a write flush leaves ~126 MB
    of dirty lines whose write-back competes with the timed kernel)."""
    flush.view(torch.int64).sum()


def _time_graph(torch, device, flush, launch, copies, reps=15):
    """Median ms per launch of `launch(k, stream)`, k = 0..copies-1, captured as ONE CUDA graph
    (programmatic-dependent-launch edges included) and replayed between a CUDA-event pair: every
    k works on its own cold copy of the data, the GPU runs the launches back to back and the
    host's per-call cost is out of the picture.  L2 flushed by reads before every replay."""
    side = torch.cuda.Stream(device=device)
    with torch.cuda.stream(side):
        for k in range(copies):
            launch(k, side.cuda_stream)
    torch.cuda.synchronize(device)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        for k in range(copies):
            launch(k, torch.cuda.current_stream(device).cuda_stream)
    torch.cuda.synchronize(device)
    samples = []
    for _ in range(reps + 2):
        _clean_l2_flush(torch, flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graph.replay()
        b.record()
        torch.cuda.synchronize(device)
        samples.append(a.elapsed_time(b) / copies)
    return float(np.median(samples[2:]))


def _time_single(torch, device, flush, launch, reps=7):
    samples = []
    stream = torch.cuda.current_stream(device).cuda_stream
    for _ in range(reps + 1):
        _clean_l2_flush(torch, flush)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        launch(0, stream)
        b.record()
        torch.cuda.synchronize(device)
        samples.append(a.elapsed_time(b))
    return float(np.median(samples[1:]))


def cbt_kernel_probe(L, torch, device, depth, bits, peak, cpu_pool=None, cpu_threads=1):
    """The two full-pool CBT kernels of BASELINE config 4 on the given bitfield, cold, against the
    HBM roofline: k_sum_reduce (graph-batched, per launch) and k_index with both lists (decode-all).
    With `cpu_pool` (an OraclePool of the same depth) the C port runs the same two operations on
    the same bits (reference layout: uint32[2N] heap, one root-to-leaf descent per rank)."""
    n = 1 << depth
    flush = torch.zeros(512 << 20, dtype=torch.uint8, device=device)
    copies = 8 if depth <= 28 else 4
    bits_k = [bits] + [bits.clone() for _ in range(copies - 1)]
    cnts = [torch.zeros(L.cbtm_counter_words(depth), dtype=torch.int32, device=device) for _ in range(copies)]
    ws = torch.zeros(1024, dtype=torch.uint8, device=device)

    def reduce(k, stream):
        assert L.cbtm_sum_reduce(bits_k[k].data_ptr(), cnts[k].data_ptr(), depth, ws.data_ptr(), 1024, stream) == 0

    red_ms = _time_graph(torch, device, flush, reduce, copies)
    red_single_ms = _time_single(torch, device, flush, reduce)
    # a longer series (32 launches on 32 cold copies): the first launch of a series has nothing to overlap
    # with and the graph launch itself costs a few microseconds -- an eighth of that is in `us` above
    long_series = None
    if depth <= 28:
        copies32 = 32
        bits_k += [bits.clone() for _ in range(copies32 - copies)]
        cnts += [cnts[0].clone() for _ in range(copies32 - copies)]
        long_ms = _time_graph(torch, device, flush, reduce, copies32, reps=9)
        del bits_k[copies:], cnts[copies:]
        torch.cuda.empty_cache()
        long_series = {"launches": copies32, "us": long_ms * 1e3}
    ones = int(cnts[0][1].item())
    live = torch.empty(n, dtype=torch.int32, device=device)
    free = torch.empty(n, dtype=torch.int32, device=device)

    def index(k, stream):
        assert L.cbtm_index(bits.data_ptr(), cnts[0].data_ptr(), depth, live.data_ptr(), free.data_ptr(), 0, stream) == 0

    idx_ms = _time_single(torch, device, flush, index, reps=5)
    # back to back (one graph of 4 launches on the same buffers: every launch writes 4 N bytes, far more than
    # the L2 holds, so each one starts cold): without the launch overhead of a lone, event-timed kernel
    idx_series_ms = _time_graph(torch, device, flush, index, 4, reps=5)
    # spot check: the compacted lists are sorted and partition the pool
    assert bool((live[1:ones] > live[:ones - 1]).all()) and bool((free[1:n - ones] > free[:n - ones - 1]).all())
    red_bytes = n // 8 + 4 * L.cbtm_counter_words(depth)
    all_bytes = n // 8 + 4 * n
    out = {"leaves": n, "occupancy": ones / n,
           "reduce": {"us": red_ms * 1e3, "GB/s": red_bytes / red_ms / 1e6, "frac": red_bytes / red_ms / 1e6 / peak,
                      "algorithmic_bytes": red_bytes, "single_launch_us": red_single_ms * 1e3,
                      "series_of_32": None if long_series is None else dict(
                          long_series, frac=red_bytes / (long_series["us"] * 1e-6) / 1e9 / peak),
                      "timing": f"{copies} launches on {copies} cold copies as one CUDA graph, per launch, median of 15"},
           "decode_all": {"us": idx_ms * 1e3, "GB/s": all_bytes / idx_ms / 1e6,
                          "frac": all_bytes / idx_ms / 1e6 / peak, "algorithmic_bytes": all_bytes,
                          "series_of_4": {"us": idx_series_ms * 1e3, "frac": all_bytes / idx_series_ms / 1e6 / peak},
                          "timing": "single launch, CUDA events, median of 5"}}
    if cpu_pool is not None:
        import ctypes as C
        import oracle
        host_bits = bits.cpu().numpy().view(np.uint8)
        cpu_pool.nodes[n:] = np.unpackbits(host_bits, bitorder="little")[:n]
        t0 = time.perf_counter()
        oracle.sum_reduce_nodes(cpu_pool.nodes, depth, cpu_threads)
        t_red = time.perf_counter() - t0
        assert int(cpu_pool.nodes[1]) == ones
        t0 = time.perf_counter()
        oracle.lib().orc_cache_pointers(C.byref(cpu_pool._cpool()), ones, n - ones, 0, max(ones, n - ones), cpu_threads)
        t_idx = time.perf_counter() - t0
        same = (np.array_equal(cpu_pool.cache_live[:ones], live[:ones].cpu().numpy())
                and np.array_equal(cpu_pool.cache_free[:n - ones], free[:n - ones].cpu().numpy()))
        if not same:
            raise SystemExit("bench.py: decode-all on the GPU and on the CPU port disagree")
        out["cpu_port"] = {"cores": cpu_threads, "reduce_ms": t_red * 1e3, "decode_all_ms": t_idx * 1e3,
                           "reduce_speedup": t_red / (red_ms * 1e-3), "decode_all_speedup": t_idx / (idx_ms * 1e-3),
                           "layout": "reference heap uint32[2N] (8 B/slot): sum_reduce_array + one descent per rank "
                                     "(k_cache_pointers); outputs verified equal to the GPU lists"}
    del bits_k, cnts, live, free, flush
    torch.cuda.empty_cache()
    return out


def random_bits(torch, device, depth, seed):
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    return torch.randint(-2 ** 63, 2 ** 63 - 1, ((1 << depth) // 64,), dtype=torch.int64, device=device, generator=gen)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def resolve_workload(args, world):
    if args.workload != "auto":
        return args.workload
    return "batch" if world > 1 else "earth"


def dist_setup(torch):
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback for the product path)")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} wants cuda:{local} but only {torch.cuda.device_count()} device(s) are visible")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    under_torchrun = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    if under_torchrun:  # also at world size 1: the NCCL gather path is the same code
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        dist.init_process_group("nccl", device_id=device)

    def barrier():
        if under_torchrun:
            dist.barrier()
        torch.cuda.synchronize(device)

    return dist, world, rank, local, device, under_torchrun, barrier


def run_gpu_earth(args):
    import ctypes as C
    import torch

    from paper_2407_02215_b200 import _lib
    from paper_2407_02215_b200.lod import LodDecide
    from paper_2407_02215_b200.pipeline import ParallelEngine
    from paper_2407_02215_b200.state import initialize

    dist, world, rank, local, device, grouped, barrier = dist_setup(torch)
    seq, down, cycle = sweep_params(args.depth, 45.0 * rank)
    K, W = args.steps, args.warmup
    eng = ParallelEngine()
    # clocks are sampled from before the setup frames until after the e2e run: the device-timed
    # region itself is a few ms, shorter than nvidia-smi's sampling period
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    state = initialize(seq.mesh, args.depth, device=device, staged_launches=args.staged)
    eng.run_lod_sequence(state, down)                       # setup: fly to the ground
    eng.run_lod_sequence(state, step_params(cycle, 0, W))   # warm-up steps
    timed_prm = step_params(cycle, W, K)

    start_host = None
    if rank == 0 and world == 1 and not args.no_cpu:
        start_host = state.to_host()
    e2e_state = state.clone()
    draw_state = state.clone() if rank == 0 and not args.no_draw_leg else None

    # ---- device-timed run: K frames, parameters resident, no host sync ----
    L = _lib.load()
    d_stats = torch.zeros((K, _lib.STATS_WORDS), dtype=torch.int64, device=device)
    pinned = torch.from_numpy(timed_prm).pin_memory()
    pool = state.c_pool()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if rank == 0:
        sampler.wait_first(2.0)
    barrier()
    ev0.record()
    rc = L.cbtm_run_lod_sequence(C.byref(pool), _lib.ptr(state.d_root_tris), pinned.data_ptr(), K,
                                 _lib.ptr(d_stats), state.stream())
    ev1.record()
    barrier()
    _lib.check(rc, "cbtm_run_lod_sequence")
    state._touched()
    gpu_ms = ev0.elapsed_time(ev1)
    rows = d_stats.cpu().numpy()
    units = int(rows[:, 6].sum())

    # ---- e2e: the same frames through the public API, default engine, per-frame host<->device ----
    # Every frame: LodDecide(config, camera, mesh) -> ParallelEngine.update -> UpdateStats on the host
    # (184 B of camera parameters in, 256 B of counters out, one cooperative launch).  Nothing is
    # subtracted: the clock stops when the stream has drained after the last frame.
    cams = step_cameras(seq, W, K)
    for cam in cams[:3]:            # warm the per-frame launch path on a scratch copy
        eng.update(state, LodDecide(seq.config, cam, seq.mesh))
    barrier()
    t0 = time.perf_counter()
    e2e_rows = []
    for j in range(K):
        s = eng.update(e2e_state, LodDecide(seq.config, cams[j], seq.mesh), epoch=j)
        e2e_rows.append((s.splits_rejected_oom, s.merges_rejected_oom, s.splits_applied, s.merges_applied,
                         s.split_allocs, s.merge_allocs, s.live_before, s.live_after))
    e2e_state.synchronize()
    barrier()
    e2e_s = time.perf_counter() - t0
    if e2e_rows != [tuple(int(x) for x in rows[j, :8]) for j in range(K)]:
        raise SystemExit("bench.py: e2e run and device-timed run report different counters (parity failure)")

    # ---- the paper's frame: update, then everything a draw call needs ----
    # Every frame: update as above, then cbtm_export_live_triangles on the same stream (index of the NEW
    # state, fp64 decode of every live bisector into a device vertex buffer, indirect draw arguments
    # written on the device).  Shows that other GPU work runs between the frame kernels: update()
    # returns when the frame's counters are decided, the export is queued behind the rest of the frame.
    draw = None
    if rank == 0 and not args.no_draw_leg:
        cap = 1 << 18
        vbuf = torch.empty((cap, 3, 3), dtype=torch.float64, device=device)
        dargs = torch.zeros(4, dtype=torch.int32, device=device)
        dpool = draw_state.c_pool()

        def frame(j):
            s = eng.update(draw_state, LodDecide(seq.config, cams[j], seq.mesh), epoch=j)
            _lib.check(L.cbtm_export_live_triangles(C.byref(dpool), _lib.ptr(draw_state.d_root_tris), _lib.ptr(vbuf), cap,
                                                    _lib.ptr(dargs), draw_state.stream()), "cbtm_export_live_triangles")
            return s
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        for j in range(K):
            s = frame(j)
        draw_state.synchronize()
        draw_s = time.perf_counter() - t0
        if int(dargs[0]) != 3 * s.live_after or s.live_after != int(rows[K - 1, 7]):
            raise SystemExit("bench.py: draw arguments of the last frame do not match its live count")
        draw = {"ms_per_step": 1e3 * draw_s / K, "value": units / draw_s, "unit": UNIT,
                "vertex_buffer_bytes_last_frame": 72 * s.live_after,
                "mode": "per frame: ParallelEngine().update(...) then cbtm_export_live_triangles (k_index of the new "
                        "state + fp64 decode of all live bisectors + indirect draw args, device resident) on the same "
                        "stream; wall clock over K frames including the drain"}
        del vbuf
    clocks = sampler.stop() if rank == 0 else None

    # ---- max over ranks ----
    t = torch.tensor([gpu_ms, e2e_s * 1e3, float(units)], dtype=torch.float64, device=device)
    if grouped:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        gpu_ms, e2e_ms, units_all = float(tmax[0]), float(tmax[1]), float(tsum[2])
        gathered = [torch.zeros_like(d_stats) for _ in range(world)]
        dist.all_gather(gathered, d_stats)  # the only collective: final stats gather
    else:
        e2e_ms, units_all = e2e_s * 1e3, float(units)
    if rank != 0:
        if grouped:
            dist.destroy_process_group()
        return 0

    # ---- roofline: k_frames, the one kernel of the timed region ----
    peak, peak_src = load_peaks()
    N = 1 << args.depth
    n_f, S_f, M_f, A_f = (rows[:, c].astype(np.float64) for c in (6, 2, 3, 9))
    # B_frame = B_reduce + N/8 + 4(n + A) + 16 n + 90 S + 50 M, B_reduce = N/4
    alg_bytes = float((N / 4 + N / 8 + 4 * (n_f + A_f) + 16 * n_f + 90 * S_f + 50 * M_f).sum())
    achieved = alg_bytes / (gpu_ms * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(args.depth)
    roofline = {
        "bound": "hbm", "kernel": "k_frames (persistent cooperative frame kernel, all six phases)",
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "traffic_source": traffic_src,
        "algorithmic_bytes_per_frame": alg_bytes / K, "kernel_ms": gpu_ms, "launches": 1, "frames_per_launch": K,
        "timing": "CUDA events on the launch stream around the one launch that runs the K timed frames",
        "peak_source": peak_src,
        "note": "algorithmic bytes per SURVEY.md 8(d) (full-bitfield reduction and indexation every frame: "
                "N/4 + N/8 + 4(n+A) + 16n + 90S + 50M).  The kernel moves far less than that -- indexation "
                "skips empty leaf blocks from their counters and the in-frame reduction only recounts the "
                "leaf blocks the frame touched (traffic << algorithmic) -- and is bound by the latency of "
                "~35 dependent L2 round trips and 6 grid barriers per frame, not by HBM; the two full-pool "
                "CBT kernels are measured against the roofline in cbt_kernels_d26 / config4"}

    # ---- CPU baselines on bounded samples, from the same start state ----
    cpu = cpu_port = cpu_reference = None
    cpu_pool = None
    if start_host is not None:
        import oracle
        threads = oracle.max_threads()
        n_port = min(K, args.cpu_frames)
        op = cpu_pool = oracle_pool_from_host(seq.mesh, args.depth, start_host)
        sec, port_rows = port_sample(op, seq.mesh, timed_prm[:n_port], threads)
        for j in range(n_port):
            if port_rows[j] != [int(x) for x in rows[j, :8]]:
                raise SystemExit(f"bench.py: GPU and CPU-port stats differ at timed frame {j}: "
                                 f"{rows[j, :8].tolist()} vs {port_rows[j]}")
        cpu_port = {"value": sum(r[6] for r in port_rows) / sec, "unit": UNIT, "cores": threads, "kind": "port",
                    "ms_per_frame": 1e3 * sec / n_port,
                    "sample": f"first {n_port} timed frames from the same pool state (stats verified equal to the "
                              "GPU's), C/OpenMP port of the reference path (oracle/): OpenMP over stage 2 / "
                              "classifier / stage 9"}
        cpu = cpu_port
        if reference_available() and not args.port_only:
            cpu_reference = reference_legs(args, seq, start_host, cams, rows, threads)
            allt = cpu_reference["config3"]["all_threads"]
            cpu = {"value": allt["bisectors_per_s"], "unit": UNIT, "cores": threads, "kind": "reference",
                   "ms_per_frame": allt["ms_per_frame_mean"],
                   "sample": f"first {allt['frames']} timed frames from the same pool state (stats verified equal to the "
                             f"GPU's) through the unmodified cbtmesh ParallelEngine(threads={threads}).update + LodDecide "
                             "(baseline/_ref), numba JIT-warmed first; see cpu_reference for 1 thread and config 2, "
                             "cpu_port for the C/OpenMP port"}

    # ---- full-pool CBT kernels against the roofline (config 4), next to the CPU port ----
    cbt26 = cbt_kernel_probe(L, torch, device, args.depth, state.d_bits, peak) if args.depth <= 28 else None
    config4 = None
    if not args.no_config4:
        import oracle
        config4 = {}
        for d in (26, 28, 30):
            bits = random_bits(torch, device, d, 1000 * d + 50)
            use_cpu = d == 26 and cpu_pool is not None and args.depth == 26
            config4[f"d{d}"] = cbt_kernel_probe(L, torch, device, d, bits, peak, cpu_pool if use_cpu else None,
                                                oracle.max_threads() if use_cpu else 1)
            del bits
            torch.cuda.empty_cache()

    e2e_value = units_all / (e2e_ms * 1e-3)
    line = {
        "metric": METRIC, "value": units_all / (gpu_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": gpu_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic", "config": workload_config(args, world, "earth"),
        "live_bisectors_per_frame": {"mean": float(rows[:, 6].mean()), "max": int(rows[:, 6].max())},
        "ops_in_run": {"splits": int(rows[:, 2].sum()), "merges": int(rows[:, 3].sum()),
                       "oom": int(rows[:, 0].sum() + rows[:, 1].sum())},
        "phase_us": {name: float(rows[:, _lib.STAT_PHASE_NS + k].mean()) / 1e3
                     for k, name in enumerate(_lib.PHASE_NAMES)},
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms / K,
                "h2d_bytes_per_step": 8 * _lib.PRM_WORDS, "d2h_bytes_per_step": 8 * _lib.STATS_WORDS,
                "mode": "ParallelEngine().update(state, LodDecide(config, camera, mesh)) per frame: default engine, one "
                        "cooperative launch per frame, wall clock from before the first update until the stream has "
                        "drained after the last, nothing subtracted",
                "note": "pool state is device-resident by design; per-frame host input is the camera (184 B, passed as "
                        "launch parameters), per-frame output the 32 counters the kernel writes straight into mapped "
                        "host memory as soon as they are decided (after the agreement phase), so the host side of "
                        "the next frame overlaps with the rest of this one"},
        # persistent path: ONE cooperative launch (k_frames) runs all K frames, six phases each;
        # staged path: index, classify, admit, scatter, agree, reserve, apply, upper_reduce, publish per frame
        "e2e_update_plus_draw_export": draw,
        "gpu_launches": 9 * K if args.staged else 1,
        "launch_mode": "staged" if args.staged else "persistent (1 cooperative launch, 6 phases x K frames); e2e: K launches",
        "roofline": roofline,
        "cbt_kernels_d26": cbt26,
        "config4": config4,
        "cpu_baseline": cpu,
        "cpu_port": cpu_port,
        "cpu_reference": cpu_reference,
        "clocks": clocks,
    }
    print(json.dumps(line))
    if grouped:
        dist.destroy_process_group()
    return 0


def reference_legs(args, seq, start_host, cams, gpu_rows, threads):
    """The real reference beside the GPU: config 3 from the same pool state (a few frames at all
    threads, fewer at 1 thread) and the whole BASELINE config 2 fly-in (2^20 pool, 64 frames)."""
    from baseline import ref_timing
    from paper_2407_02215_b200 import workloads
    ref_timing.load()
    jit_s = ref_timing.warm_jit(threads)
    out = {"kind": "reference", "jit_warmup_s": jit_s, "cores": threads,
           "method": "cbtmesh.pipeline.ParallelEngine(threads=T).update with LodDecide, perf_counter_ns around update "
                     "(cli.py:285-289); unmodified package from baseline/_ref"}
    st = ref_timing.state_from_arrays(seq.mesh, args.depth, start_host)
    legs = {}
    for name, T, frames in (("all_threads", threads, args.ref_frames), ("one_thread", 1, max(1, args.ref_frames - 1))):
        work = st if name == "one_thread" else ref_timing.clone_state(st)
        per_frame, ref_rows = ref_timing.time_frames(work, seq.mesh, seq.config, cams[:frames], T)
        for j in range(frames):
            if ref_rows[j] != [int(x) for x in gpu_rows[j, :8]]:
                raise SystemExit(f"bench.py: GPU and real-reference stats differ at timed frame {j}: "
                                 f"{gpu_rows[j, :8].tolist()} vs {ref_rows[j]}")
        legs[name] = {"threads": T, "frames": frames, "ms_per_frame_mean": 1e3 * sum(per_frame) / frames,
                      "ms_per_frame": [1e3 * x for x in per_frame],
                      "bisectors_per_s": sum(r[6] for r in ref_rows) / sum(per_frame)}
        del work
    del st
    out["config3"] = legs
    if not args.no_config2:
        fly = workloads.cube_sphere_flyin(depth=20, frames=64)
        legs2 = {}
        for name, T in (("all_threads", threads), ("one_thread", 1)):
            from cbtmesh import sequential as ref_seq
            st2 = ref_seq.initialize(ref_timing.ref_mesh_of(fly.mesh), 20)
            per_frame, ref_rows = ref_timing.time_frames(st2, fly.mesh, fly.config, fly.cameras, T)
            legs2[name] = {"threads": T, "frames": len(per_frame), "ms_per_frame_median": 1e3 * float(np.median(per_frame)),
                           "total_ms": 1e3 * sum(per_frame), "bisectors_per_s": sum(r[6] for r in ref_rows) / sum(per_frame),
                           "peak_live": max(r[7] for r in ref_rows)}
        out["config2"] = legs2
    return out


def run_gpu_batch(args):
    """BASELINE config 5: 8 planets x 2^24 slots over the ranks (strong scaling)."""
    import torch

    from paper_2407_02215_b200 import _lib, batch, workloads

    dist, world, rank, local, device, grouped, barrier = dist_setup(torch)
    K, W = args.steps, args.warmup
    P = BATCH_PLANETS
    owned = batch.planets_of_rank(P, world, rank)
    seqs, downs, cycles = zip(*[sweep_params(BATCH_DEPTH, 45.0 * p) for p in range(P)])
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    t_setup = time.perf_counter()
    states, _ = batch.run_planet_batch(seqs, list(downs), world, rank, device)                       # setup
    states, _ = batch.run_planet_batch(seqs, [step_params(c, 0, W) for c in cycles], world, rank, device, states)  # warm-up
    timed = [step_params(c, W, K) for c in cycles]
    e2e_states = [s.clone() for s in states]
    setup_s = time.perf_counter() - t_setup

    # ---- device-timed: this rank's planets, K frames in lockstep in one launch per group ----
    import ctypes as C
    L = _lib.load()
    k = len(owned)
    d_stats = [torch.zeros((K, _lib.STATS_WORDS), dtype=torch.int64, device=device) for _ in owned]
    pinned = [torch.from_numpy(timed[p]).pin_memory() for p in owned]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if rank == 0:
        sampler.wait_first(2.0)
    barrier()
    ev0.record()
    launches = 0
    for g0 in range(0, k, _lib.MAX_BATCH):
        g = range(g0, min(k, g0 + _lib.MAX_BATCH))
        pools = (_lib.CPool * len(g))(*[states[q].c_pool() for q in g])
        roots = (C.c_void_p * len(g))(*[_lib.ptr(states[q].d_root_tris) for q in g])
        prms = (C.c_void_p * len(g))(*[pinned[q].data_ptr() for q in g])
        souts = (C.c_void_p * len(g))(*[_lib.ptr(d_stats[q]) for q in g])
        _lib.check(L.cbtm_run_lod_sequence_batch(pools, len(g), roots, prms, K, souts, states[g0].stream()),
                   "cbtm_run_lod_sequence_batch")
        launches += 1
    ev1.record()
    barrier()
    gpu_ms = ev0.elapsed_time(ev1) if k else 0.0
    for s in states:
        s._touched()
    local_rows = np.stack([d.cpu().numpy() for d in d_stats]) if k else np.zeros((0, K, _lib.STATS_WORDS), np.int64)

    # ---- e2e: the public batch API with host parameter arrays (uploaded inside, stats downloaded inside) ----
    barrier()
    t0 = time.perf_counter()
    _, e2e_block = batch.run_planet_batch(seqs, timed, world, rank, device, e2e_states)
    torch.cuda.synchronize(device)
    barrier()
    e2e_s = time.perf_counter() - t0
    clocks = sampler.stop() if rank == 0 else None
    cols = [c for c in range(13) if c != _lib.STAT_FRAME]   # (the frame counter of a cloned pool restarts)
    if not np.array_equal(e2e_block[:, :, cols], local_rows[:, :, cols]):
        raise SystemExit("bench.py: batch API run and device-timed run report different counters (parity failure)")

    # ---- the one collective: final gather of the per-frame stats (NCCL all_gather) ----
    full = batch.gather_stats(local_rows, owned, P, world, device=device if grouped else None)
    t = torch.tensor([gpu_ms, e2e_s * 1e3], dtype=torch.float64, device=device)
    per_rank_ms = [gpu_ms]
    if grouped:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank_ms = [float(x[0]) for x in allt]
        gpu_ms, e2e_ms = float(tmax[0]), float(tmax[1])
    else:
        e2e_ms = e2e_s * 1e3
    if rank != 0:
        if grouped:
            dist.destroy_process_group()
        return 0
    units_all = float(full[:, :, 6].sum())
    peak, peak_src = load_peaks()
    N = 1 << BATCH_DEPTH
    n_f, S_f, M_f, A_f = (full[:, :, c].astype(np.float64) for c in (6, 2, 3, 9))
    alg_bytes = float((N / 4 + N / 8 + 4 * (n_f + A_f) + 16 * n_f + 90 * S_f + 50 * M_f).sum())
    achieved = alg_bytes / world / (gpu_ms * 1e-3) / 1e9   # per GPU
    line = {
        "metric": METRIC, "value": units_all / (gpu_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": gpu_ms / K, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic", "config": workload_config(args, world, "batch"),
        "per_rank_device_ms": per_rank_ms, "planets_per_rank": [len(batch.planets_of_rank(P, world, r)) for r in range(world)],
        "live_bisectors_per_planet_frame": {"mean": float(full[:, :, 6].mean()), "max": int(full[:, :, 6].max())},
        "ops_in_run": {"splits": int(full[:, :, 2].sum()), "merges": int(full[:, :, 3].sum()),
                       "oom": int(full[:, :, 0].sum() + full[:, :, 1].sum())},
        "stats_digest": {"live_after_last_frame": full[:, -1, 7].tolist(),
                         "counter_sum": int(full[:, :, :10].sum())},
        "phase_us": {name: float(local_rows[0, :, _lib.STAT_PHASE_NS + j].mean()) / 1e3
                     for j, name in enumerate(_lib.PHASE_NAMES)},
        "e2e": {"value": units_all / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms / K,
                "h2d_bytes_per_step": 8 * _lib.PRM_WORDS * P, "d2h_bytes_per_step": 8 * _lib.STATS_WORDS * P,
                "mode": "batch.run_planet_batch -> pipeline.run_lod_sequence_batch with host float64[K,23] parameter "
                        "arrays per planet: parameter upload, K lockstep frames, stats download, all inside the clock"},
        "gpu_launches": launches, "launch_mode": "k_frames_batch: one cooperative launch per rank runs K frames of its planets",
        "collective": ("NCCL all_gather of the int64[planets, K, 32] stats (torch.distributed)" if grouped
                       else "none (single process; the gather is a local re-index)"),
        "roofline": {"bound": "hbm", "kernel": "k_frames_batch", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes_per_step": alg_bytes / K,
                     "note": "per GPU; latency-bound like the single-planet frame (see the earth workload's roofline note)"},
        "cpu_baseline": None, "setup_s": setup_s,
        "clocks": clocks,
    }
    print(json.dumps(line))
    if grouped:
        dist.destroy_process_group()
    return 0


def respawn_under_torchrun(args) -> int:
    """`--gpus N` from a plain shell: one rank per GPU under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="graft", choices=["graft", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "earth", "batch"],
                    help="earth = BASELINE config 3 (default at N = 1), batch = config 5 (default at N > 1)")
    ap.add_argument("--depth", type=int, default=26)
    ap.add_argument("--cpu-frames", type=int, default=8, help="frames of the C port timed beside the GPU")
    ap.add_argument("--ref-frames", type=int, default=3, help="frames of the real reference timed beside the GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--port-only", action="store_true", help="CPU legs: only the C port, not the real reference")
    ap.add_argument("--no-config2", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--no-draw-leg", action="store_true", help="skip the update + triangle export leg")
    ap.add_argument("--torchrun-world1", action="store_true",
                    help="run under torch.distributed.run even at N = 1 (exercises NCCL init + the gather)")
    ap.add_argument("--staged", action="store_true",
                    help="one kernel launch per pipeline stage (for ncu launch lists); default is the "
                         "persistent cooperative frame kernel")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.torchrun_world1):
        return respawn_under_torchrun(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if resolve_workload(args, world) == "batch":
        return run_gpu_batch(args)
    return run_gpu_earth(args)


if __name__ == "__main__":
    sys.exit(main())
