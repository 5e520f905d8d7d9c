#!/bin/bash
# raw chunks through LDGSTS (PNCE_TUNE_RAW_LSU=1) vs TMA: cfg4' (TMA ring forced), tensor16, bench legs
for spec in "X=1" "PNCE_TUNE_RAW_LSU=1" "PNCE_TUNE_WIDE_LDG=0" "PNCE_TUNE_WIDE_LDG=0 PNCE_TUNE_RAW_LSU=1"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/prof_cfg4.py 256 2>&1 | tail -1)  $(env $spec timeout -s KILL 300 python tools/t16_time.py 2048 2>&1 | tail -1)"
done
bash tools/ab.sh tools/ab_specs_36.txt
