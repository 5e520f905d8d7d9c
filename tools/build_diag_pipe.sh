#!/bin/bash
# Diagnostic pipeline-stage removals (results are garbage; timing only).
set -e
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DPNCE_WATCHDOG -shared -Xcompiler -fPIC"
SRC="paper_2206_05506_b200/csrc/pnce_kernels.cu paper_2206_05506_b200/csrc/pnce_synth.cu"
mkdir -p tools/bin
$B -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_CONV -o tools/bin/libpnce_diag_ns_noconv.so $SRC &
$B -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_CONV -DPNCE_DIAG_NO_RAW -o tools/bin/libpnce_diag_ns_noconv_noraw.so $SRC &
$B -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_CONV -DPNCE_DIAG_NO_RAW -DPNCE_DIAG_NO_B -o tools/bin/libpnce_diag_ns_noinput.so $SRC &
$B -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_CONV -DPNCE_DIAG_NO_RAW -DPNCE_DIAG_NO_FULLWAIT -o tools/bin/libpnce_diag_mma_only.so $SRC &
wait
