#!/bin/bash
# L2 prefetch of raw chunks (TMA and LDG converter modes); distance sweep; trace.
mkdir -p gpurun_out
A="--frames 4096 --gemm-frames 1024 --steps 5 --no-e2e --no-cpu --no-quality"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%  tensor %.1f%% | gemm us/frame %.3f tensor %.1f%%'%(d['us_per_frame'],100*d['roofline']['frac'],100*d['roofline']['tensor_frac'],d['gemm_leg']['us_per_frame'],100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run tma_pf0 PNCE_TUNE_FUSED_MODE=2 PNCE_TUNE_RAW_PREFETCH=0
run tma_pf4 PNCE_TUNE_FUSED_MODE=2 PNCE_TUNE_RAW_PREFETCH=4
run tma_pf8 PNCE_TUNE_FUSED_MODE=2 PNCE_TUNE_RAW_PREFETCH=8
run tma_pf16 PNCE_TUNE_FUSED_MODE=2 PNCE_TUNE_RAW_PREFETCH=16
run ldg_pf0 PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_RAW_PREFETCH=0
run ldg_pf8 PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_RAW_PREFETCH=8
run ldg_pf16 PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_RAW_PREFETCH=16
run tma_ab2_pf8 PNCE_TUNE_FUSED_MODE=2 PNCE_TUNE_AB_STAGES=2 PNCE_TUNE_RAW_PREFETCH=8
run tma_nostore_pf8 PNCE_TUNE_FUSED_MODE=2 PNCE_LIB=tools/bin/libpnce_diag_no_store.so
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality"
PNCE_TUNE_FUSED_MODE=1 PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace_m1.bin timeout -s KILL 200 python bench.py $T > gpurun_out/trace.log 2>&1; echo trace=$?
PNCE_TUNE_FUSED_MODE=2 PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace_m2.bin timeout -s KILL 200 python bench.py $T > gpurun_out/trace.log 2>&1; echo trace=$?
