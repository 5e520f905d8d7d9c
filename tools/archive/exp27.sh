#!/bin/bash
# Split drain (first N half of the accumulator released early) on/off; truth ring for scored.
timeout -s KILL 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
A="--frames 4096 --gemm-frames 4096 --scored-frames 2048 --steps 5 --no-e2e --no-cpu --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f hbm %.1f%% | gemm %.3f (%.1f%%) | scored %.3f | t16 %.3f | clk %s' % (d['us_per_frame'],100*d['roofline']['frac'], d['gemm_leg']['us_per_frame'], 100*d['gemm_leg']['frac_of_bf16_peak'], d['estimate_quality']['scored_us_per_frame'], d['tensor16_leg']['us_per_frame'], d['clocks']['sm_mhz']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run split X=1
run nosplit PNCE_TUNE_SPLIT_DRAIN=0
run split2 X=1
run nosplit2 PNCE_TUNE_SPLIT_DRAIN=0
run split_s2g512 PNCE_TUNE_TRUTH_SLOTS=2 PNCE_TUNE_SCORED_G=512
run split_s0 PNCE_TUNE_TRUTH_SLOTS=0
