#!/bin/bash
# Diagnostic: no circulant (B) loads -- isolates the raw-input pipeline.
set -e
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DPNCE_WATCHDOG -shared -Xcompiler -fPIC"
SRC="paper_2206_05506_b200/csrc/pnce_kernels.cu paper_2206_05506_b200/csrc/pnce_synth.cu"
mkdir -p tools/bin
$B -DPNCE_DIAG_NO_B -o tools/bin/libpnce_diag_no_b.so $SRC &
$B -DPNCE_DIAG_NO_B -DPNCE_DIAG_NO_STORE -o tools/bin/libpnce_diag_no_b_no_store.so $SRC &
$B -DPNCE_DIAG_NO_STORE -o tools/bin/libpnce_diag_no_store.so $SRC &
wait
