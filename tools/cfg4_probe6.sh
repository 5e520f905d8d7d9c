#!/bin/bash
# cfg4': LDG converters (FUSED_MODE=1) vs the TMA raw ring, plain and scored, A/B stage depth
for pass in 1 2; do
for spec in "fused X=1" "fused PNCE_TUNE_FUSED_MODE=1" "fused PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_AB_STAGES=3" "scored X=1" "scored PNCE_TUNE_FUSED_MODE=1"; do
  set -- $spec
  m=$1; shift
  echo "$m $*: $(env "$@" timeout -s KILL 300 python tools/prof_cfg4.py 256 $m 2>&1 | tail -1)"
done
done
