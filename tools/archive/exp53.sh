#!/bin/bash
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; }
run tma_reuse X=1
run ldg_g256 PNCE_TUNE_FUSED_MODE=1
run ldg_g512 PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_SCORED_G=512
run tma_g512 PNCE_TUNE_SCORED_G=512
run tma_reuse2 X=1
