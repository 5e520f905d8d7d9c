#!/bin/bash
# tensor16 cfg3 cycle accounting (PNCE_DIAG_PROF builds; the last launch's counters)
mkdir -p gpurun_out
for lib in prof prof_nostore; do
  PNCE_LIB=tools/bin/libpnce_diag_$lib.so PNCE_PROF_FILE=gpurun_out/t16_$lib.bin timeout -s KILL 300 python tools/t16_time.py 2048 > gpurun_out/t16_$lib.log 2>&1
  echo "== $lib: $(tail -1 gpurun_out/t16_$lib.log)"
  python tools/prof_view.py gpurun_out/t16_$lib.bin
done
