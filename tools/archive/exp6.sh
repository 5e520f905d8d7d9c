#!/bin/bash
A="--frames 4096 --gemm-frames 2048 --steps 5 --no-e2e --no-cpu"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%  tensor %.1f%% | gemm us/frame %.3f tensor %.1f%%'%(d['us_per_frame'],100*d['roofline']['frac'],100*d['roofline']['tensor_frac'],d['gemm_leg']['us_per_frame'],100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run default X=1
run ab4 PNCE_TUNE_AB_STAGES=4
run ab2 PNCE_TUNE_AB_STAGES=2
run no_store PNCE_LIB=tools/bin/libpnce_diag_no_store.so
run pipe_only PNCE_LIB=tools/bin/libpnce_diag_pipe_only.so
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu"
PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace_full.bin python bench.py $T > /dev/null
