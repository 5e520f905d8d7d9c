#!/bin/bash
# Only the cycle-accounting diagnostic builds (tools/gpu_prof.sh).
set -e
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DPNCE_WATCHDOG -shared -Xcompiler -fPIC"
SRC="paper_2206_05506_b200/csrc/pnce_kernels.cu paper_2206_05506_b200/csrc/pnce_synth.cu"
mkdir -p tools/bin
$B -DPNCE_DIAG_PROF -o tools/bin/libpnce_diag_prof.so $SRC &
$B -DPNCE_DIAG_PROF -DPNCE_DIAG_NO_STORE -o tools/bin/libpnce_diag_prof_nostore.so $SRC &
wait
