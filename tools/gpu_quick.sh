#!/bin/bash
# Quick GPU round: smoke, GPU tests, default bench, traced run of the fused kernel.
mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -5 gpurun_out/gpu_tests.log
timeout -s KILL 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo "bench=$?"; tail -c 2500 gpurun_out/bench.log
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality"
PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace.bin timeout -s KILL 200 python bench.py $T > gpurun_out/trace.log 2>&1; echo trace=$?
timeout -s KILL 120 tools/bin/load_probe > gpurun_out/load_probe.txt 2>&1; echo probe=$?; cat gpurun_out/load_probe.txt
