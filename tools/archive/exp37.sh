#!/bin/bash
timeout -s KILL 900 python -m pytest tests/test_gpu_knobs.py -q -x 2>&1 | tail -3
timeout -s KILL 300 python bench.py --frames 1024 --gemm-frames 1024 --steps 5 --no-e2e --no-cpu --file-frames 0 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps(d['cfg4_leg'], indent=1))
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
"
