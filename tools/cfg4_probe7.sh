#!/bin/bash
# cfg4' fused (LDG converters): L2 prefetch distance of the converters' rows
for pass in 1 2; do
for spec in "X=1" "PNCE_TUNE_LDG_PF=1" "PNCE_TUNE_LDG_PF=2" "PNCE_TUNE_LDG_PF=4" "PNCE_TUNE_LDG_PF=8"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/prof_cfg4.py 256 2>&1 | tail -1)"
done
done
