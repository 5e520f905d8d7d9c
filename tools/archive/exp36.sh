#!/bin/bash
for r in 1 0; do
PNCE_TUNE_A_REUSE=$r timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_correlate -c 3 python tools/cfg4_time.py 128 fused 2>&1 | grep -E "k_correlate|dram__|duration|hit_rate" | head -8
done
