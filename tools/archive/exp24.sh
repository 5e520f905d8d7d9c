#!/bin/bash
# Scored kernel warp split (4 conv + 8 epi vs 8 conv + 4 epi) x group width.
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; }
run base X=1
run conv8 PNCE_TUNE_SCORED_CONV8=1
run g512 PNCE_TUNE_SCORED_G=512
run g512_conv8 PNCE_TUNE_SCORED_G=512 PNCE_TUNE_SCORED_CONV8=1
