#!/bin/bash
# Full GPU round: smoke, tests, default bench (10k frames), reference arm, ncu launch list + full capture.
mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -2 gpurun_out/gpu_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?"; tail -c 3500 gpurun_out/bench.log
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref=$?"; tail -c 1500 gpurun_out/bench_ref.log
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
A="--frames 1024 --gemm-frames 1024 --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 200 python bench.py $A > gpurun_out/plain_ncu.log 2>&1 && \
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
B="--frames 512 --gemm-frames 512 --scored-frames 512 --steps 1 --warmup 3 --no-e2e --no-cpu --file-frames 0"
timeout -s KILL 200 python bench.py $B > gpurun_out/plain_ncu2.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_correlate -s 3 -c 6 -o gpurun_out/prof_full python bench.py $B > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
