#!/bin/bash
# Cycle accounting of the tensor16 launch (the last launch of the quality legs).
mkdir -p gpurun_out
COMMON="--steps 1 --warmup 3 --no-e2e --no-cpu --latency-reps 0 --cfg4-frames 0 --antenna-reps 0 --file-frames 0 --frames 2048 --no-gemm-leg"
for lib in prof prof_nostore; do
  PNCE_LIB=tools/bin/libpnce_diag_$lib.so PNCE_PROF_FILE=gpurun_out/$lib.t16.bin timeout -s KILL 200 python bench.py $COMMON > gpurun_out/$lib.t16.log 2>&1; echo "$lib t16=$?"
  python tools/prof_view.py gpurun_out/$lib.t16.bin
done
