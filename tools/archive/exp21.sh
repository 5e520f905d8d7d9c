#!/bin/bash
# Cycle accounting of the scored kernel (G=256 default, and G=512) and the plain kernel.
mkdir -p gpurun_out
L=tools/bin/libpnce_diag_prof.so
PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_scored.bin timeout -s KILL 200 python tools/prof_scored.py
python tools/prof_view.py gpurun_out/prof_scored.bin
PNCE_TUNE_SCORED_G=512 PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_scored512.bin timeout -s KILL 200 python tools/prof_scored.py
python tools/prof_view.py gpurun_out/prof_scored512.bin
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality --file-frames 0"
PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_plain.bin timeout -s KILL 200 python bench.py $T > /dev/null 2>&1
python tools/prof_view.py gpurun_out/prof_plain.bin
