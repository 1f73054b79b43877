#!/usr/bin/env python
"""Turn ncu outputs brought back in gpurun_out/ into the small text summaries
committed under profiles/.

  launch list : python benchmarks/summarize_ncu.py launches gpurun_out/launches.csv [first_frame last_frame]
  full report : python benchmarks/summarize_ncu.py details gpurun_out/prof.ncu-rep
"""

from __future__ import annotations

import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_active.avg",
        "gpc__cycles_elapsed.max",
        # atomic traffic (north_star: "atomic throughput against B200 peak")
        "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_op_atom.sum",
        "lts__t_requests_op_red.sum", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
        "smsp__inst_executed_op_global_atom.sum", "smsp__inst_executed_op_global_red.sum",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_lsu.sum",
        "smsp__inst_executed.sum", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_membar_per_warp_active.pct"]


def launches(path, first=None, last=None):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    ours = [(r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("cbtm::", ""),
             float(r["Metric Value"]))
            for r in rows if r["Metric Name"] == "gpu__time_duration.sum" and "cbtm::" in r["Kernel Name"]]
    frames, cur = [], None
    for name, ns in ours:
        if name == "k_index":
            cur = []
            frames.append(cur)
        if cur is not None:
            cur.append((name, ns))
    first = 0 if first is None else first
    last = len(frames) if last is None else last
    sel = frames[first:last]
    agg = collections.OrderedDict()
    for fr in sel:
        for name, ns in fr:
            agg[name] = agg.get(name, 0.0) + ns / len(sel)
    total = sum(agg.values())
    print(f"# ncu launch list {path}: frames {first}..{last - 1} of {len(frames)} "
          f"(gpu__time_duration, cold cache, serialised -- compare shares, not absolutes)")
    print(f"# mean per frame: {total / 1e3:.1f} us over {len(sel)} frames")
    for name, ns in agg.items():
        print(f"{name:<16s} {ns / 1e3:8.2f} us  {100 * ns / total:5.1f} %")


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {k: hdr.index(k) for k in KEYS if k in hdr}
    name_i = hdr.index("Kernel Name")
    seen = collections.OrderedDict()
    for r in rows[2:]:
        seen.setdefault(r[name_i].split("(")[0], []).append(r)
    print(f"# ncu --set full summary of {path} (last captured launch of each kernel; {len(rows) - 2} launches captured)")
    for kname, rs in seen.items():
        print(f"\n## {kname}  ({len(rs)} launches)")
        r = rs[-1]   # the last captured launch of the kernel (warm code, steady state)
        for k, i in idx.items():
            print(f"  {k:<62s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], *(int(x) for x in sys.argv[3:5]))
    else:
        details(sys.argv[2])
