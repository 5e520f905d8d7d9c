#!/bin/bash
mkdir -p gpurun_out
for lib in prof prof_nostore; do
  PNCE_LIB=tools/bin/libpnce_diag_$lib.so PNCE_PROF_FILE=gpurun_out/$lib.c4.bin timeout -s KILL 300 python tools/prof_cfg4.py 256 > gpurun_out/$lib.c4.log 2>&1; echo "$lib=$? $(tail -1 gpurun_out/$lib.c4.log)"
  python tools/prof_view.py gpurun_out/$lib.c4.bin
done
