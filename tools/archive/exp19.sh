#!/bin/bash
A="--frames 4096 --gemm-frames 1024 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%% | gemm %.3f' % (d['us_per_frame'],100*d['roofline']['frac'], d['gemm_leg']['us_per_frame']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run base X=1
run g256 PNCE_TUNE_GROUP_FUSED=256
run g256_ldg PNCE_TUNE_GROUP_FUSED=256 PNCE_TUNE_FUSED_MODE=1
run base2 X=1
