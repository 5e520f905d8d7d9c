#!/bin/bash
# cfg4' fused: timing under the reuse knobs, then DRAM bytes / L2 hit rate of the fused launch (ncu).
mkdir -p gpurun_out
for envs in "X=1" "PNCE_TUNE_A_REUSE=0" "PNCE_TUNE_SCR_POL=0" "PNCE_TUNE_SCR_SLOTS=2"; do
  echo "$envs: $(env $envs timeout -s KILL 300 python tools/prof_cfg4.py 256 2>&1 | tail -1)"
done
for envs in "X=1" "PNCE_TUNE_A_REUSE=0"; do
  env $envs timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:k_correlate -s 3 -c 1 python tools/prof_cfg4.py 64 > gpurun_out/cfg4_ncu_$envs.txt 2>&1
  echo "== $envs"; grep -E "dram__|lts__|gpu__time" gpurun_out/cfg4_ncu_$envs.txt
done
