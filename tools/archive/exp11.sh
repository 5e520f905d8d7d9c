#!/bin/bash
mkdir -p gpurun_out
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality"
for m in 1 2; do
  PNCE_TUNE_FUSED_MODE=$m PNCE_TUNE_RAW_PREFETCH=0 PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/prof_m$m.bin timeout -s KILL 200 python bench.py $T > gpurun_out/prof_m$m.log 2>&1; echo prof$m=$?; grep -o '"us_per_frame": [0-9.]*' gpurun_out/prof_m$m.log | head -1
  PNCE_TUNE_FUSED_MODE=$m PNCE_TUNE_RAW_PREFETCH=0 PNCE_LIB=tools/bin/libpnce_diag_prof_nostore.so PNCE_PROF_FILE=gpurun_out/prof_ns_m$m.bin timeout -s KILL 200 python bench.py $T > gpurun_out/prof_ns_m$m.log 2>&1; echo profns$m=$?; grep -o '"us_per_frame": [0-9.]*' gpurun_out/prof_ns_m$m.log | head -1
done
