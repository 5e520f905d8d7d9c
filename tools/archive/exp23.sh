#!/bin/bash
mkdir -p gpurun_out
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality --file-frames 0"
PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace.bin timeout -s KILL 200 python bench.py $T > gpurun_out/trace.log 2>&1; echo trace=$?
python tools/trace_view.py gpurun_out/trace.bin
