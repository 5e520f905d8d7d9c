#!/bin/bash
# Desync sweep + packed grouping, then launch list + full ncu capture of the fused kernel.
mkdir -p gpurun_out
A="--frames 4096 --gemm-frames 2048 --steps 5 --no-e2e --no-cpu --no-quality"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%  tensor %.1f%% | gemm us/frame %.3f tensor %.1f%%'%(d['us_per_frame'],100*d['roofline']['frac'],100*d['roofline']['tensor_frac'],d['gemm_leg']['us_per_frame'],100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run default X=1
run desync5 PNCE_TUNE_DESYNC_NS=5000
run desync10 PNCE_TUNE_DESYNC_NS=10000
run desync14 PNCE_TUNE_DESYNC_NS=14000
run packed256 PNCE_TUNE_GROUP_PACKED=256
run no_store PNCE_LIB=tools/bin/libpnce_diag_no_store.so
run pipe_only PNCE_LIB=tools/bin/libpnce_diag_pipe_only.so
B="--frames 512 --gemm-frames 512 --steps 1 --warmup 3 --no-e2e --no-cpu --no-quality"
timeout -s KILL 200 python bench.py $B > gpurun_out/plain_ncu2.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_correlate -s 3 -c 2 -o gpurun_out/prof_v6 python bench.py $B > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
