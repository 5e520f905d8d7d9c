#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_gpu_low_latency.py tests/test_gpu_parity.py tests/test_gpu_knobs.py -q -x 2>&1 | tail -2
timeout -s KILL 200 python tools/lat_split.py 1
timeout -s KILL 200 python tools/lat_split.py 8
