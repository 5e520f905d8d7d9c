#!/bin/bash
# GPU tests only (optionally a file/pattern), no bench.
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest ${1:-tests} -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -30 gpurun_out/gpu_tests.log
