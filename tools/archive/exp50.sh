#!/bin/bash
A="--frames 1024 --gemm-frames 512 --steps 3 --no-cpu --no-quality --file-frames 0 --cfg4-frames 0 --e2e-frames 64"
for g in 512 256 128; do
PNCE_TUNE_GROUP_FUSED=$g timeout -s KILL 300 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('G=$g fused %.3f us/frame |' % d['us_per_frame'], json.dumps({k:v for k,v in d['latency'].items() if k!='note'}))
    elif 'rror' in l: print(l.strip()[:300])
"
done
