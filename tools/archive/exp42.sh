#!/bin/bash
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; }
run g256_s3 X=1
run g256_s3_ab4 PNCE_TUNE_AB_STAGES=4
run g256_s2_ab4 PNCE_TUNE_AB_STAGES=4 PNCE_TUNE_TRUTH_SLOTS=2
run g512_s2 PNCE_TUNE_SCORED_G=512 PNCE_TUNE_TRUTH_SLOTS=2
run g256_s0 PNCE_TUNE_TRUTH_SLOTS=0
run g256_s3b X=1
