#!/bin/bash
timeout -s KILL 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in "reuse X=1" "noreuse PNCE_TUNE_A_REUSE=0"; do
  set -- $cfg; n=$1; shift
  echo "=== $n"
  env "$@" timeout -s KILL 300 python tools/cfg4_time.py 512
  env "$@" timeout -s KILL 300 python tools/prof_scored.py | tail -1
done
L=tools/bin/libpnce_diag_prof.so
PNCE_LIB=$L PNCE_PROF_FILE=gpurun_out/prof_c4_fused.bin timeout -s KILL 300 python tools/cfg4_time.py 256 fused
python tools/prof_view.py gpurun_out/prof_c4_fused.bin 2>/dev/null
