#!/bin/bash
# GPU tests (default: the whole -m gpu suite; else the given files / pytest args)
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest -m gpu -q -x ${@:-tests} > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -25 gpurun_out/gpu_tests.log
