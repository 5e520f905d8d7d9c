#!/bin/bash
L=tools/bin/libpnce_diag_prof.so
PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_sc.bin timeout -s KILL 200 python tools/prof_scored.py
python tools/prof_view.py gpurun_out/prof_sc.bin
