#!/bin/bash
# Bounds-checked build (tools/build_diag_checks.sh) over every mode: the sanitize workload per
# knob variant, the GPU test suite, and 500 random stress geometries.  Logs: gpurun_out/checks_*.txt
mkdir -p gpurun_out
export PNCE_LIB=tools/bin/libpnce_diag_checks.so
for v in "default PNCE_X=0" "ldg PNCE_TUNE_FUSED_MODE=1" "scored256 PNCE_TUNE_SCORED_G=256 PNCE_TUNE_TRUTH_SLOTS=3" \
         "scored_t0 PNCE_TUNE_TRUTH_SLOTS=0" "packedldg PNCE_TUNE_PACKED_MODE=3" "t16e4 PNCE_TUNE_T16_EPI=4" \
         "nosplit PNCE_TUNE_SPLIT_DRAIN=0" "noreuse PNCE_TUNE_A_REUSE=0" "nonarrow PNCE_TUNE_NARROW=0 PNCE_TUNE_MID=0" \
         "reuse2 PNCE_TUNE_A_REUSE=2" "wideldg0 PNCE_TUNE_WIDE_LDG=0"; do
  set -- $v; name=$1; shift
  env "$@" timeout -s KILL 600 python tools/sanitize_run.py > gpurun_out/checks_$name.txt 2>&1; echo "$name rc=$? $(grep -c PNCE_CHECK gpurun_out/checks_$name.txt) $(tail -1 gpurun_out/checks_$name.txt)"
done
[ -n "$SKIP_TESTS" ] || timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/checks_tests.txt 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/checks_tests.txt)"
[ -n "$SKIP_TESTS" ] || timeout -s KILL 1500 python tools/stress.py 7 500 > gpurun_out/checks_stress.txt 2>&1; echo "stress rc=$? $(tail -2 gpurun_out/checks_stress.txt | tr '\n' ' ')"
