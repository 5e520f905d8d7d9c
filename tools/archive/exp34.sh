#!/bin/bash
L=tools/bin/libpnce_diag_prof.so
for leg in fused packed; do
PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_c4_$leg.bin timeout -s KILL 300 python tools/cfg4_time.py 256 $leg
python tools/prof_view.py gpurun_out/prof_c4_$leg.bin
done
