# batch kernel with 2 / 3 / 4 co-resident CTAs per SM (register budget 128 / 85 / 64)
cd $GRAFT_REPO_ROOT
cp paper_2407_02215_b200/libcbtm.so /tmp/libcbtm_release.so
for C in 2 3 4 5; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --shared -Xcompiler -fPIC -DCBTM_BATCH_CTAS_PER_SM=$C -o paper_2407_02215_b200/libcbtm.so paper_2407_02215_b200/csrc/cbtm.cu -ccbin /usr/bin/g++
  echo "== BATCH_CTAS_PER_SM=$C"
  python bench.py --workload batch --steps 32 | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(d['ms_per_step'], d['phase_us'])"
done
cp /tmp/libcbtm_release.so paper_2407_02215_b200/libcbtm.so
