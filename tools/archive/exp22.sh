#!/bin/bash
# Packed GEMM leg: 256-column groups with two TMEM accumulators (A re-read per group).
A="--frames 512 --gemm-frames 4096 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); g=d['gemm_leg']; print('gemm %.3f us/frame  %.1f%% burst  %.1f%% sustained' % (g['us_per_frame'], 100*g['frac_of_bf16_peak'], 100*g['frac_of_bf16_sustained']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run base X=1
run g256 PNCE_TUNE_GROUP_PACKED=256
run g256_pol0 PNCE_TUNE_GROUP_PACKED=256 PNCE_TUNE_RAW_POL=0
run g256_pol2 PNCE_TUNE_GROUP_PACKED=256 PNCE_TUNE_RAW_POL=2
run g256_epi4 PNCE_TUNE_GROUP_PACKED=256 PNCE_TUNE_EPI8=0
run g384 PNCE_TUNE_GROUP_PACKED=384
run base2 X=1
