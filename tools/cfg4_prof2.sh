#!/bin/bash
# cfg4' cycle accounting: LDG converters (FUSED_MODE=1) vs the TMA raw ring
mkdir -p gpurun_out
for spec in "fused PNCE_TUNE_FUSED_MODE=1" "fused PNCE_TUNE_A_REUSE=0"; do
  set -- $spec
  env $2 PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/c4_$1_$2.bin timeout -s KILL 300 python tools/prof_cfg4.py 256 $1 > gpurun_out/c4_$1_$2.log 2>&1
  echo "== $spec: $(tail -1 gpurun_out/c4_$1_$2.log)"
  python tools/prof_view.py gpurun_out/c4_$1_$2.bin
done
