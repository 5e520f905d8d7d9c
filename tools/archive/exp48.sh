#!/bin/bash
# setmaxnreg: register reallocation to the epilogue (scored drain double-buffered), A/B vs previous build
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
A="--frames 4096 --gemm-frames 4096 --scored-frames 2048 --steps 5 --no-e2e --no-cpu --file-frames 0 --cfg4-frames 256"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 300 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['cfg4_leg']; print('fused %.3f | gemm %.3f | scored %.3f | t16 %.3f | cfg4 fused %.2f gemm %.2f' % (d['us_per_frame'], d['gemm_leg']['us_per_frame'], d['estimate_quality']['scored_us_per_frame'], d['tensor16_leg']['us_per_frame'], c['fused']['us_per_frame'], c['gemm']['us_per_frame']))
    elif 'rror' in l: print(l.strip()[:300])
"; }
run new X=1
run prev PNCE_LIB=tools/bin/libpnce_prev.so
run new2 X=1
run prev2 PNCE_LIB=tools/bin/libpnce_prev.so
