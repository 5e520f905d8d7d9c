#!/bin/bash
# Final round-2 measurement: smoke, GPU tests, bench (all legs), reference arm, ncu launch list,
# ncu DRAM traffic at 4096 frame-sets, ncu full capture of the fused + scored + packed kernels.
mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -1 gpurun_out/gpu_tests.log
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref=$?"
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
A="--frames 10000 --steps 2 --warmup 3 --no-e2e --no-cpu --latency-reps 5 --antenna-reps 5 --file-frames 0"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
T="--frames 4096 --gemm-frames 4096 --scored-frames 4096 --steps 1 --warmup 3 --no-e2e --no-cpu --file-frames 0 --latency-reps 0 --cfg4-frames 0 --antenna-reps 0"
timeout -s KILL 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum -k regex:k_correlate --clock-control none --csv --log-file gpurun_out/traffic.csv python bench.py $T > gpurun_out/ncu_traffic.log 2>&1; echo "ncu_traffic=$?"
B="--frames 1024 --gemm-frames 1024 --scored-frames 1024 --steps 1 --warmup 3 --no-e2e --no-cpu --file-frames 0 --latency-reps 0 --cfg4-frames 0 --antenna-reps 0"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_correlate -s 3 -c 4 -o gpurun_out/prof_full python bench.py $B > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
