#!/bin/bash
# Pipelined-LDG converters (mode 1) vs TMA-staged (mode 2): parity under both, speed, trace.
mkdir -p gpurun_out
PNCE_TUNE_FUSED_MODE=1 timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_m1.log 2>&1; echo "tests_m1=$?"; tail -3 gpurun_out/gpu_tests_m1.log
A="--frames 4096 --gemm-frames 2048 --steps 5 --no-e2e --no-cpu --no-quality"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%  tensor %.1f%% | gemm us/frame %.3f tensor %.1f%%'%(d['us_per_frame'],100*d['roofline']['frac'],100*d['roofline']['tensor_frac'],d['gemm_leg']['us_per_frame'],100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run tma PNCE_TUNE_FUSED_MODE=2
run ldg PNCE_TUNE_FUSED_MODE=1
run ldg_ab3 PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_AB_STAGES=3
run ldg_nostore PNCE_TUNE_FUSED_MODE=1 PNCE_LIB=tools/bin/libpnce_diag_no_store.so
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality"
PNCE_TUNE_FUSED_MODE=1 PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace_m1.bin timeout -s KILL 200 python bench.py $T > gpurun_out/trace.log 2>&1; echo trace=$?
