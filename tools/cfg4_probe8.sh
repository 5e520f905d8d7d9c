#!/bin/bash
# cfg4' scored: reuse / truth ring / group width
for spec in "X=1" "PNCE_TUNE_A_REUSE=0" "PNCE_TUNE_TRUTH_SLOTS=0" "PNCE_TUNE_SCORED_EPI=4" "PNCE_TUNE_A_REUSE=0 PNCE_TUNE_RAW_STAGES=3"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/prof_cfg4.py 128 scored 2>&1 | tail -1)"
done
