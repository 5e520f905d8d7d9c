#!/bin/bash
A="--frames 4096 --gemm-frames 4096 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f hbm %.1f%% | gemm %.3f (%.1f%%)' % (d['us_per_frame'],100*d['roofline']['frac'], d['gemm_leg']['us_per_frame'], 100*d['gemm_leg']['frac_of_bf16_peak']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run base X=1
run ab4 PNCE_TUNE_AB_STAGES=4
run ab2 PNCE_TUNE_AB_STAGES=2
run base2 X=1
timeout -s KILL 600 python tools/cfg5_sweep.py > gpurun_out/cfg5_sweep.txt 2>&1; echo cfg5=$?; tail -5 gpurun_out/cfg5_sweep.txt
