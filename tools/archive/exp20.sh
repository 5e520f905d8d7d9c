#!/bin/bash
# Raw-row L2 policy with several lag-row groups (scored G=256, tensor16, plain G=256).
A="--frames 4096 --gemm-frames 1024 --scored-frames 2048 --steps 5 --no-e2e --no-cpu --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f hbm %.1f%% | gemm %.3f | scored %.3f | t16 %.3f' % (d['us_per_frame'],100*d['roofline']['frac'], d['gemm_leg']['us_per_frame'], d['estimate_quality']['scored_us_per_frame'], d['tensor16_leg']['us_per_frame']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run pol_default X=1
run pol0 PNCE_TUNE_RAW_POL=0
run pol2 PNCE_TUNE_RAW_POL=2
run g256_pol1 PNCE_TUNE_GROUP_FUSED=256
run g256_pol0 PNCE_TUNE_GROUP_FUSED=256 PNCE_TUNE_RAW_POL=0
run g256_pol2 PNCE_TUNE_GROUP_FUSED=256 PNCE_TUNE_RAW_POL=2
