#!/bin/bash
# cfg4' fused under the epilogue-warp split (EPI8: 4 converter + 8 epilogue warps)
for envs in "X=1" "PNCE_TUNE_EPI8=1" "PNCE_TUNE_EPI8=1 PNCE_TUNE_A_REUSE=0" "X=1" "PNCE_TUNE_EPI8=1"; do
  echo "$envs: $(env $envs timeout -s KILL 300 python tools/prof_cfg4.py 256 2>&1 | tail -1)"
done
