#!/bin/bash
mkdir -p gpurun_out
A="--frames 4096 --gemm-frames 1024 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%' % (d['us_per_frame'],100*d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run first X=1
run normal PNCE_TUNE_RAW_POLICY=1
run first2 X=1
run normal2 PNCE_TUNE_RAW_POLICY=1
B="--frames 512 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality --file-frames 0"
for pol in 0 1; do
PNCE_TUNE_RAW_POLICY=$pol timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_correlate -s 3 -c 1 --csv python bench.py $B > gpurun_out/ncu_pol$pol.csv 2>/dev/null; echo ncu$pol=$?; grep k_correlate gpurun_out/ncu_pol$pol.csv | cut -c1-60,200-
done
