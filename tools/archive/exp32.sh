#!/bin/bash
# A-reuse (convert a row tile once, other lag-row groups TMA the fp16 A stages from an L2 scratch).
timeout -s KILL 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for r in 1 0; do
  echo "=== PNCE_TUNE_A_REUSE=$r"
  PNCE_TUNE_A_REUSE=$r timeout -s KILL 300 python tools/cfg4_time.py 512
  PNCE_TUNE_A_REUSE=$r timeout -s KILL 200 python bench.py --frames 4096 --gemm-frames 512 --scored-frames 4096 --steps 5 --no-e2e --no-cpu --file-frames 0 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('cfg3 fused %.3f | scored %.3f | t16 %.3f' % (d['us_per_frame'], d['estimate_quality']['scored_us_per_frame'], d['tensor16_leg']['us_per_frame']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"
done
