#!/bin/bash
mkdir -p gpurun_out
PNCE_TUNE_EPI8=1 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t_epi8.log 2>&1; echo tests_epi8=$?; tail -2 gpurun_out/t_epi8.log
A="--frames 4096 --gemm-frames 1024 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%%' % (d['us_per_frame'],100*d['roofline']['frac']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run base X=1
run epi8 PNCE_TUNE_EPI8=1
run base2 X=1
run epi8_2 PNCE_TUNE_EPI8=1
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu --no-quality --file-frames 0"
PNCE_TUNE_EPI8=1 PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/prof_e8.bin timeout -s KILL 200 python bench.py $T > /dev/null 2>&1; echo prof=$?
