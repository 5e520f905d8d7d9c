#!/bin/bash
for cfg in "pol1 PNCE_TUNE_SCR_POL=1" "pol0 PNCE_TUNE_SCR_POL=0" "noreuse PNCE_TUNE_A_REUSE=0"; do
  set -- $cfg; n=$1; shift
  echo "=== $n"
  env "$@" timeout -s KILL 300 python tools/cfg4_time.py 512
  env "$@" timeout -s KILL 300 python tools/prof_scored.py | tail -1
done
timeout -s KILL 300 python -m pytest tests -m gpu -q -x -k "cfg4 or tensor16 or scored" 2>&1 | tail -2
