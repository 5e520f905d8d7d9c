#!/bin/bash
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; }
run base X=1
run no_truth_pf PNCE_LIB=tools/bin/libpnce_diag_notpf.so
run base2 X=1
run no_truth_pf2 PNCE_LIB=tools/bin/libpnce_diag_notpf.so
run no_truth_pf_s4 PNCE_LIB=tools/bin/libpnce_diag_notpf.so PNCE_TUNE_TRUTH_SLOTS=4
