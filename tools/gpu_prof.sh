#!/bin/bash
# Cycle accounting (PNCE_DIAG_PROF builds) of the fused kernel and the packed GEMM leg.
mkdir -p gpurun_out
[ -f tools/bin/libpnce_diag_prof.so ] || bash tools/build_diag_prof.sh > gpurun_out/build_diag.log 2>&1
COMMON="--steps 1 --warmup 3 --no-e2e --no-cpu --latency-reps 0 --cfg4-frames 0 --antenna-reps 0 --file-frames 0"
for lib in prof prof_nostore; do
  PNCE_LIB=tools/bin/libpnce_diag_$lib.so PNCE_PROF_FILE=gpurun_out/$lib.fused.bin timeout -s KILL 200 python bench.py --frames 4096 --no-gemm-leg --no-quality $COMMON > gpurun_out/$lib.fused.log 2>&1; echo "$lib fused=$?"
  python tools/prof_view.py gpurun_out/$lib.fused.bin
  PNCE_LIB=tools/bin/libpnce_diag_$lib.so PNCE_PROF_FILE=gpurun_out/$lib.gemm.bin timeout -s KILL 200 python bench.py --frames 4096 --gemm-frames 4096 --no-quality $COMMON > gpurun_out/$lib.gemm.log 2>&1; echo "$lib gemm=$?"
  python tools/prof_view.py gpurun_out/$lib.gemm.bin
done
