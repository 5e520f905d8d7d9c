#!/bin/bash
timeout -s KILL 300 python tools/cfg4_time.py 512
PNCE_TUNE_SPLIT_DRAIN=0 timeout -s KILL 300 python tools/cfg4_time.py 512
