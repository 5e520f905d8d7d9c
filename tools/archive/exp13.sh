#!/bin/bash
mkdir -p gpurun_out
T="--frames 4096 --gemm-frames 4096 --steps 1 --warmup 3 --no-e2e --no-cpu --no-quality"
for m in 0 3; do
  PNCE_TUNE_PACKED_MODE=$m PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/prof_p$m.bin timeout -s KILL 200 python bench.py $T > gpurun_out/prof_p$m.log 2>&1; echo prof$m=$?
  PNCE_TUNE_PACKED_MODE=$m PNCE_LIB=tools/bin/libpnce_diag_prof_nostore.so PNCE_PROF_FILE=gpurun_out/prof_ns_p$m.bin timeout -s KILL 200 python bench.py $T > gpurun_out/prof_ns_p$m.log 2>&1; echo profns$m=$?
done
