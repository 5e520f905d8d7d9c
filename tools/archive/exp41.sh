#!/bin/bash
A="--frames 2048 --gemm-frames 512 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0 --cfg4-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f hbm %.1f%%' % (d['us_per_frame'],100*d['roofline']['frac']))
    elif 'rror' in l or 'pnce:' in l: print(l.strip()[:300])
"; }
run quad PNCE_VERBOSE=1
run pair PNCE_TUNE_QUAD=0
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
