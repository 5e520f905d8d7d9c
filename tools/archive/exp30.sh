#!/bin/bash
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; }
run base X=1
run conv8_s3 PNCE_TUNE_SCORED_CONV8=1 PNCE_TUNE_TRUTH_SLOTS=3
run conv8_s2 PNCE_TUNE_SCORED_CONV8=1 PNCE_TUNE_TRUTH_SLOTS=2
run conv8_s4 PNCE_TUNE_SCORED_CONV8=1 PNCE_TUNE_TRUTH_SLOTS=4
run conv8_g512_s2 PNCE_TUNE_SCORED_CONV8=1 PNCE_TUNE_TRUTH_SLOTS=2 PNCE_TUNE_SCORED_G=512
run base2 X=1
