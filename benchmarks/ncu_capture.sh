#!/bin/bash
# ncu captures of the final kernels (run under gpurun from the repo root; outputs in gpurun_out/).
#   bash benchmarks/ncu_capture.sh r2
# Then, here: python benchmarks/summarize_ncu.py details gpurun_out/<tag>_<name>.ncu-rep > profiles/<tag>_<name>_ncu.txt
set -u
TAG=${1:-r2}
OUT=gpurun_out
ATOM=lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,smsp__inst_executed_op_global_atom.sum,smsp__inst_executed_op_global_red.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
NCU="ncu --set full --clock-control none --metrics $ATOM"
summarize() { python benchmarks/summarize_ncu.py details $OUT/${TAG}_$1.ncu-rep > $OUT/${TAG}_$1_ncu.txt 2>&1; [ "${2:-}" = keep ] || rm -f $OUT/${TAG}_$1.ncu-rep; }
# launch list of the bench command (device time per launch; cold cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 > $OUT/${TAG}_launches_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches_staged.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-config4 --staged > $OUT/${TAG}_launches_staged.log 2>&1
$NCU --import-source on -k regex:k_frames -s 1 -c 2 -f -o $OUT/${TAG}_kframes2 python benchmarks/ncu_targets.py frames > $OUT/${TAG}_ncu_frames.log 2>&1
summarize kframes2 keep
$NCU -k regex:k_frames -s 14 -c 2 -f -o $OUT/${TAG}_kframes4 python benchmarks/ncu_targets.py wide > $OUT/${TAG}_ncu_wide.log 2>&1
summarize kframes4
$NCU -k regex:k_frames_batch -s 1 -c 2 -f -o $OUT/${TAG}_kbatch python benchmarks/ncu_targets.py batch > $OUT/${TAG}_ncu_batch.log 2>&1
summarize kbatch
for D in 26 28 30; do
  $NCU -k regex:k_sum_reduce -s 1 -c 2 -f -o $OUT/${TAG}_reduce_d$D python benchmarks/ncu_targets.py reduce $D > $OUT/${TAG}_ncu_reduce$D.log 2>&1
  summarize reduce_d$D
done
$NCU -k regex:k_index -c 2 -f -o $OUT/${TAG}_index_d30 python benchmarks/ncu_targets.py index 30 > $OUT/${TAG}_ncu_index.log 2>&1
summarize index_d30
$NCU -k regex:k_decode -c 2 -f -o $OUT/${TAG}_decode_d28 python benchmarks/ncu_targets.py decode 28 > $OUT/${TAG}_ncu_decode.log 2>&1
summarize decode_d28
ls -la $OUT/ | tail -40; du -sh $OUT
