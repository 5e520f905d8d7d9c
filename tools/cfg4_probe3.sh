#!/bin/bash
# cfg4' fused: A/B stage depth vs raw ring depth
for envs in "X=1" "PNCE_TUNE_AB_STAGES=4" "PNCE_TUNE_AB_STAGES=2" "X=1" "PNCE_TUNE_AB_STAGES=4"; do
  echo "$envs: $(env $envs timeout -s KILL 300 python tools/prof_cfg4.py 256 2>&1 | tail -1)"
done
