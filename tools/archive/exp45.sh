#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_gpu_knobs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for sl in 1 2 1; do
  echo "== slots $sl"
  PNCE_TUNE_SCR_SLOTS=$sl timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1
  PNCE_TUNE_SCR_SLOTS=$sl timeout -s KILL 300 python tools/cfg4_time.py 256 fused,scored
done
