#!/bin/bash
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout -s KILL 200 python tools/prof_scored.py 2>&1 | tail -1; done
