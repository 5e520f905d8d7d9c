#!/bin/bash
# Diagnostic builds of the correlator (never used by the product path).
set -e
B="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DPNCE_WATCHDOG -shared -Xcompiler -fPIC"
SRC="paper_2206_05506_b200/csrc/pnce_kernels.cu paper_2206_05506_b200/csrc/pnce_synth.cu"
mkdir -p tools/bin
$B -DPNCE_DIAG_NO_STORE -o tools/bin/libpnce_diag_no_store.so $SRC &
$B -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_RAW -DPNCE_DIAG_NO_CONV -o tools/bin/libpnce_diag_pipe_only.so $SRC &
$B -DPNCE_DIAG_TRACE -o tools/bin/libpnce_diag_trace.so $SRC &
$B -DPNCE_DIAG_TRACE -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_RAW -DPNCE_DIAG_NO_CONV -o tools/bin/libpnce_diag_trace_pipe.so $SRC &
wait
$B -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_RAW -DPNCE_DIAG_NO_CONV -DPNCE_DIAG_NO_FULLWAIT -o tools/bin/libpnce_diag_mma_only.so $SRC
$B -DPNCE_DIAG_TRACE -DPNCE_DIAG_NO_STORE -DPNCE_DIAG_NO_RAW -DPNCE_DIAG_NO_CONV -DPNCE_DIAG_NO_FULLWAIT -o tools/bin/libpnce_diag_trace_mma.so $SRC
$B -DPNCE_DIAG_PROF -o tools/bin/libpnce_diag_prof.so $SRC &
$B -DPNCE_DIAG_PROF -DPNCE_DIAG_NO_STORE -o tools/bin/libpnce_diag_prof_nostore.so $SRC &
wait
