#!/bin/bash
A="--frames 4096 --gemm-frames 4096 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0 --cfg4-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 300 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f | gemm %.3f' % (d['us_per_frame'], d['gemm_leg']['us_per_frame']))
    elif 'rror' in l: print(l.strip()[:300])
"; }
run d0 X=1
run d5us PNCE_TUNE_DESYNC_NS=5000
run d10us PNCE_TUNE_DESYNC_NS=10000
run d3us PNCE_TUNE_DESYNC_NS=3000
run d0b X=1
