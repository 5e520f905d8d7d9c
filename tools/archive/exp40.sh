#!/bin/bash
A="--frames 2048 --gemm-frames 512 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0 --cfg4-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f hbm %.1f%%' % (d['us_per_frame'],100*d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:300])
"; }
run quad X=1
run quad_nocopy PNCE_LIB=tools/bin/libpnce_diag_quad_nocopy.so
run quad_nostore PNCE_LIB=tools/bin/libpnce_diag_no_store.so
run pair_nostore PNCE_LIB=tools/bin/libpnce_diag_no_store.so PNCE_TUNE_QUAD=0
