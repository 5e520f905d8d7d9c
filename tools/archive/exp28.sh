#!/bin/bash
# Scored: split drain with G=512 (+ truth ring slots) vs G=256 double-buffered.
timeout -s KILL 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
A="--frames 1024 --gemm-frames 512 --scored-frames 4096 --steps 5 --no-e2e --no-cpu --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused %.3f | scored %.3f' % (d['us_per_frame'], d['estimate_quality']['scored_us_per_frame']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run g256_s3 X=1
run g512_s2 PNCE_TUNE_SCORED_G=512 PNCE_TUNE_TRUTH_SLOTS=2
run g512_s0 PNCE_TUNE_SCORED_G=512 PNCE_TUNE_TRUTH_SLOTS=0
run g512_s2_nosplit PNCE_TUNE_SCORED_G=512 PNCE_TUNE_TRUTH_SLOTS=2 PNCE_TUNE_SPLIT_DRAIN=0
run g512_s3 PNCE_TUNE_SCORED_G=512 PNCE_TUNE_TRUTH_SLOTS=3
run g256_s0 PNCE_TUNE_TRUTH_SLOTS=0
