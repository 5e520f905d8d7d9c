#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_gpu_tensor16.py tests/test_gpu_knobs.py -q -x 2>&1 | tail -2
A="--frames 1024 --gemm-frames 512 --scored-frames 512 --steps 5 --no-e2e --no-cpu --file-frames 0 --cfg4-frames 0"
for g in 160 256 160; do
PNCE_TUNE_T16_G=$g timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('t16 G=$g: %.3f us/frame' % d['tensor16_leg']['us_per_frame'], d['tensor16_leg']['saturations'], d['tensor16_leg']['nonfinite'])
    elif 'rror' in l: print(l.strip()[:300])
"
done
