#!/bin/bash
# Build the library at a git revision (default HEAD) into tools/bin/libpnce_<rev>.so for A/B runs.
set -e
REV=${1:-HEAD}
D=$(mktemp -d)
mkdir -p $D/paper_2206_05506_b200/csrc $D/include
for f in pnce_kernels.cu pnce_synth.cu pnce_internal.h sm100_ptx.cuh; do
  git show $REV:paper_2206_05506_b200/csrc/$f > $D/paper_2206_05506_b200/csrc/$f
done
git show $REV:include/pnce_b200.h > $D/include/pnce_b200.h
mkdir -p tools/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -DPNCE_WATCHDOG \
  -shared -Xcompiler -fPIC -o tools/bin/libpnce_$(echo $REV | tr -c 'a-zA-Z0-9\n' _).so \
  $D/paper_2206_05506_b200/csrc/pnce_kernels.cu $D/paper_2206_05506_b200/csrc/pnce_synth.cu
rm -rf $D
