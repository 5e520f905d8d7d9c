#!/bin/bash
# 4-CTA quad kernel (two pairs share the converted row tile, double-buffered 256-col accumulators)
timeout -s KILL 120 python __graft_entry__.py smoke 2>&1 | tail -2
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
A="--frames 4096 --gemm-frames 512 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0 --cfg4-frames 0"
for qd in 1 0 1; do
PNCE_TUNE_QUAD=$qd timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('quad=$qd fused %.3f hbm %.1f%%' % (d['us_per_frame'],100*d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
"
done
