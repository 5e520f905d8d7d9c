#!/bin/bash
mkdir -p gpurun_out
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality --file-frames 0"
for d in 0 6000 11000; do
  PNCE_TUNE_DESYNC_NS=$d PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/prof_d$d.bin timeout -s KILL 200 python bench.py $T > gpurun_out/prof_d$d.log 2>&1; echo d$d=$?; grep -o '"us_per_frame": [0-9.]*' gpurun_out/prof_d$d.log | head -1
done
