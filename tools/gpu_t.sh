#!/bin/bash
# GPU tests only (optionally a -k filter): tools/gpu_t.sh [pytest args...]
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -25 gpurun_out/gpu_tests.log
