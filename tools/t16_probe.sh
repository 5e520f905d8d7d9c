#!/bin/bash
# tensor16 cfg3: A/B stage depth
for pass in 1 2; do
for spec in "X=1" "PNCE_TUNE_AB_STAGES=4" "PNCE_TUNE_AB_STAGES=5" "PNCE_TUNE_AB_STAGES=6" "PNCE_TUNE_AB_STAGES=4 PNCE_TUNE_A_REUSE=0" "PNCE_TUNE_A_REUSE=0"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/t16_time.py 2048 2>&1 | tail -1)"
done
done
