set -e
cd $GRAFT_REPO_ROOT
cp paper_2407_02215_b200/libcbtm.so /tmp/libcbtm_release.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --shared -Xcompiler -fPIC -DCBTM_DEBUG_TIMING -o paper_2407_02215_b200/libcbtm.so paper_2407_02215_b200/csrc/cbtm.cu -ccbin /usr/bin/g++
python benchmarks/phase_probe.py 26 > gpurun_out/r2_phase_probe.log 2>&1
cp /tmp/libcbtm_release.so paper_2407_02215_b200/libcbtm.so
