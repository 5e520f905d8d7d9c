#!/bin/bash
# compute-sanitizer over every kernel mode (tools/sanitize_run.py); logs in gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool env...
  name=$1; tool=$2; shift 2
  env "$@" timeout -s KILL 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_${name}_${tool}.txt 2>&1
  echo "$name $tool rc=$? $(grep -E 'ERROR SUMMARY|sanitize workload ok' gpurun_out/sanitize_${name}_${tool}.txt | tr '\n' ' ')"
}
run default memcheck PNCE_X=0
run default racecheck PNCE_X=0
run default synccheck PNCE_X=0
run ldg memcheck PNCE_TUNE_FUSED_MODE=1
run scored256 memcheck PNCE_TUNE_SCORED_G=256 PNCE_TUNE_TRUTH_SLOTS=3
run packedldg memcheck PNCE_TUNE_PACKED_MODE=3
run t16e4 memcheck PNCE_TUNE_T16_EPI=4
run nosplit memcheck PNCE_TUNE_SPLIT_DRAIN=0
