#!/bin/bash
# cfg4' fused: raw-ring depth x A-stage reuse, two passes
for pass in 1 2; do
for spec in "X=1" "PNCE_TUNE_RAW_STAGES=3" "PNCE_TUNE_RAW_STAGES=4" "PNCE_TUNE_A_REUSE=0" "PNCE_TUNE_A_REUSE=0 PNCE_TUNE_RAW_STAGES=2" "PNCE_TUNE_A_REUSE=0 PNCE_TUNE_RAW_STAGES=3" "PNCE_TUNE_A_REUSE=0 PNCE_TUNE_RAW_STAGES=4"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/prof_cfg4.py 256 2>&1 | tail -1)"
done
done
