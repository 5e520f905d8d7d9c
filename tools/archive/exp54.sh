#!/bin/bash
timeout -s KILL 900 python -m pytest tests/test_gpu_knobs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
A="--frames 1024 --gemm-frames 512 --steps 3 --no-cpu --no-quality --file-frames 0 --cfg4-frames 0 --e2e-frames 64"
for n in 1 0 1; do
PNCE_TUNE_NARROW=$n timeout -s KILL 300 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('narrow=$n fused %.3f us/frame | latency device %.1f us (min %.1f), e2e %.1f us' % (d['us_per_frame'], d['latency']['device_us_median'], d['latency']['device_us_min'], d['latency']['e2e_us_median']))
    elif 'rror' in l: print(l.strip()[:300])
"
done
