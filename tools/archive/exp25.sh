#!/bin/bash
# Scored drain: truth through a per-thread LDGSTS ring (slots 0 = register path, 2, 3, 4) x group width.
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "scor or mse or truth or link" 2>&1 | tail -2
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; }
run s0 PNCE_TUNE_TRUTH_SLOTS=0
run s2 PNCE_TUNE_TRUTH_SLOTS=2
run s3 PNCE_TUNE_TRUTH_SLOTS=3
run s4 PNCE_TUNE_TRUTH_SLOTS=4
run s3_g512 PNCE_TUNE_TRUTH_SLOTS=3 PNCE_TUNE_SCORED_G=512
run s4_g512 PNCE_TUNE_TRUTH_SLOTS=4 PNCE_TUNE_SCORED_G=512
run s2_g512 PNCE_TUNE_TRUTH_SLOTS=2 PNCE_TUNE_SCORED_G=512
