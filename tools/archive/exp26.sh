#!/bin/bash
mkdir -p gpurun_out
L=tools/bin/libpnce_diag_prof.so
for cfg in "s2_g512 PNCE_TUNE_TRUTH_SLOTS=2 PNCE_TUNE_SCORED_G=512" "s3_g256 PNCE_TUNE_TRUTH_SLOTS=3" "s0_g512 PNCE_TUNE_TRUTH_SLOTS=0 PNCE_TUNE_SCORED_G=512"; do
  set -- $cfg; n=$1; shift
  echo "=== $n"
  env "$@" PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_$n.bin timeout -s KILL 200 python tools/prof_scored.py
  python tools/prof_view.py gpurun_out/prof_$n.bin
done
