#!/bin/bash
# cfg3 scored kernel cycle accounting (PNCE_DIAG_PROF build): default (4 converter + 8 epilogue
# warps) and the 8-converter split
mkdir -p gpurun_out
for spec in "X=1" "PNCE_TUNE_SCORED_EPI=4"; do
  env $spec PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/sc_$spec.bin timeout -s KILL 300 python tools/prof_scored.py > gpurun_out/sc_$spec.log 2>&1
  echo "== $spec: $(tail -1 gpurun_out/sc_$spec.log)"
  python tools/prof_view.py gpurun_out/sc_$spec.bin
done
for spec in "X=1"; do
  env $spec PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/pl_$spec.bin timeout -s KILL 300 python tools/prof_cfg4.py 256 > /dev/null 2>&1
done
