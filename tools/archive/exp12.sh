#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -3 gpurun_out/gpu_tests.log
A="--frames 4096 --gemm-frames 4096 --steps 5 --no-e2e --no-cpu --no-quality"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%  tensor %.1f%% | gemm us/frame %.3f tensor %.1f%%'%(d['us_per_frame'],100*d['roofline']['frac'],100*d['roofline']['tensor_frac'],d['gemm_leg']['us_per_frame'],100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run packed_ldg X=1
run packed_tma PNCE_TUNE_PACKED_MODE=0
run packed_ldg_512 PNCE_TUNE_GROUP_PACKED_LDG=512
