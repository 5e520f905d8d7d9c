#!/bin/bash
# One GPU round: smoke, gpu tests, bench, optional ncu capture of k_correlate.
#   tools/gpu_round.sh [ncu]
mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 600 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -3 gpurun_out/gpu_tests.log
timeout -s KILL 400 python bench.py --cpu-seconds ${CPU_SECONDS:-3} > gpurun_out/bench.log 2>&1; echo "bench=$?"; tail -c 3000 gpurun_out/bench.log
if [ "$1" == "ncu" ]; then
  ARGS="--frames 512 --gemm-frames 512 --steps 1 --warmup 3 --no-e2e --no-cpu"
  timeout -s KILL 200 python bench.py $ARGS > gpurun_out/plain_ncu.log 2>&1 && \
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_correlate -s 3 -c 2 \
      -o gpurun_out/prof python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1; echo "ncu=$?"
fi
