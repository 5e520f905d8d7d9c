#!/bin/bash
# cfg4': stage-depth sensitivity (packed GEMM at 3 A/B stages; fused with a 2- or 3-chunk raw ring)
for spec in "packed X=1" "packed PNCE_TUNE_AB_STAGES=3" "fused X=1" "fused PNCE_TUNE_RAW_STAGES=2" "fused PNCE_TUNE_RAW_STAGES=3" "fused PNCE_TUNE_A_REUSE=0 PNCE_TUNE_RAW_STAGES=3"; do
  set -- $spec
  m=$1; shift
  echo "$m $*: $(env "$@" timeout -s KILL 300 python tools/prof_cfg4.py 256 $m 2>&1 | tail -1)"
done
