#!/bin/bash
# tensor16 intermediate folds without the per-element non-finite tracking (PNCE_TUNE_T16_NF=0)
PNCE_TUNE_T16_NF=0 timeout 300 python -m pytest tests/test_gpu_tensor16.py tests/test_gpu_seam.py -x -q -m gpu 2>&1 | tail -2
for spec in "X=1" "PNCE_TUNE_T16_NF=0" "X=1" "PNCE_TUNE_T16_NF=0"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/t16_time.py 2048 2>&1 | tail -1)"
done
