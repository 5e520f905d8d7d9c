#!/bin/bash
mkdir -p gpurun_out
A="--frames 1024 --gemm-frames 4096 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f | gemm %.3f %.1f%%' % (d['us_per_frame'], d['gemm_leg']['us_per_frame'], 100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run base X=1
run epi8 PNCE_TUNE_EPI8=1
run desync PNCE_TUNE_DESYNC_NS=8000
run base2 X=1
run epi8_2 PNCE_TUNE_EPI8=1
