#!/bin/bash
# Bounds-checked diagnostic build (PNCE_DIAG_CHECKS): device-side PNCE_CHECK on global/shared accesses.
set -e
mkdir -p tools/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -DPNCE_WATCHDOG \
  -DPNCE_DIAG_CHECKS -shared -Xcompiler -fPIC -o tools/bin/libpnce_diag_checks.so \
  paper_2206_05506_b200/csrc/pnce_kernels.cu paper_2206_05506_b200/csrc/pnce_synth.cu
