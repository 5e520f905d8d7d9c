#!/bin/bash
A="--frames 4096 --gemm-frames 4096 --steps 5 --no-e2e --no-cpu"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%  tensor %.1f%% | gemm us/frame %.3f tensor %.1f%%'%(d['us_per_frame'],100*d['roofline']['frac'],100*d['roofline']['tensor_frac'],d['gemm_leg']['us_per_frame'],100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run default X=1
run ldg PNCE_TUNE_FUSED_MODE=1
run raw3 PNCE_TUNE_RAW_STAGES=3

run raw4ab2 PNCE_TUNE_RAW_STAGES=4 PNCE_TUNE_AB_STAGES=2
run packed512 PNCE_TUNE_GROUP_PACKED=512
run nostore PNCE_LIB=tools/bin/libpnce_diag_nostore.so
run nostore_raw3 PNCE_LIB=tools/bin/libpnce_diag_nostore.so PNCE_TUNE_RAW_STAGES=3
