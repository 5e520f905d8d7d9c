#!/bin/bash
mkdir -p gpurun_out
A="--frames 4096 --gemm-frames 1024 --steps 5 --no-e2e --no-cpu --no-quality --file-frames 0"
run() { echo "== $1"; shift; env "$@" timeout -s KILL 200 python bench.py $A 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('fused us/frame %.3f  hbm %.1f%% | gemm %.3f' % (d['us_per_frame'],100*d['roofline']['frac'], d['gemm_leg']['us_per_frame']))
    elif 'Error' in l or 'error' in l: print(l.strip()[:200])
"; }
run base X=1
run hint PNCE_TUNE_STORE_HINT=1
run persist PNCE_TUNE_CIRC_PERSIST=1
run both PNCE_TUNE_STORE_HINT=1 PNCE_TUNE_CIRC_PERSIST=1
run base2 X=1
echo "== torchrun nproc 1"
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --frames 2048 --no-cpu > gpurun_out/torchrun1.log 2>&1; echo torchrun=$?; grep '^{' gpurun_out/torchrun1.log | cut -c1-300
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/torchrun1_ref.log 2>&1; echo torchrun_ref=$?; grep '^{' gpurun_out/torchrun1_ref.log | cut -c1-200
