#!/bin/bash
# compute-sanitizer passes over the hot path (run under gpurun from the repo root; logs in gpurun_out/):
#   memcheck  out-of-bounds / misaligned global + shared accesses
#   racecheck shared-memory hazards inside a CTA
#   synccheck divergent barriers
#   initcheck reads of uninitialised device memory (bounded: torch allocations are reported as uninitialised
#             until written, so only the smoke workload is run under it)
# Workloads: __graft_entry__.smoke() (split / merge / LOD frames on small pools, every array against the
# oracle) and the CBT kernel tests (reduce rebuild + delta up to 2^21, decode, index).
set -u
OUT=gpurun_out
TAG=${1:-r2b}
SAN=/usr/local/cuda/bin/compute-sanitizer
for TOOL in memcheck racecheck synccheck; do
  timeout 900 $SAN --tool $TOOL --error-exitcode 9 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
      > $OUT/${TAG}_sanitize_${TOOL}_smoke.log 2>&1
  echo "$TOOL smoke rc=$?" | tee -a $OUT/${TAG}_sanitize_summary.txt
  timeout 900 $SAN --tool $TOOL --error-exitcode 9 --print-limit 20 python -m pytest tests/test_cbt_gpu.py -x -q \
      -k "not 24 and not 26 and not 28 and not largest" > $OUT/${TAG}_sanitize_${TOOL}_cbt.log 2>&1
  echo "$TOOL cbt rc=$?" | tee -a $OUT/${TAG}_sanitize_summary.txt
done
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed\|smoke ok" $OUT/${TAG}_sanitize_*.log | tee -a $OUT/${TAG}_sanitize_summary.txt
# wider pass (memcheck + racecheck): every update path of the frame kernels (pressure / admission tail, staged launches,
# batch kernel, linger mode, begin/finish split), the mesh ingest and the API tests
if [ "${2:-}" = wide ]; then
  for TOOL in memcheck racecheck; do
    timeout 3000 $SAN --tool $TOOL --error-exitcode 9 --print-limit 20 python -m pytest tests/test_update_gpu.py tests/test_api_gpu.py \
        tests/test_mesh_gpu.py -x -q > $OUT/${TAG}_sanitize_${TOOL}_update.log 2>&1
    echo "$TOOL update/api/mesh rc=$?" | tee -a $OUT/${TAG}_sanitize_summary.txt
    tail -3 $OUT/${TAG}_sanitize_${TOOL}_update.log | tee -a $OUT/${TAG}_sanitize_summary.txt
  done
fi
