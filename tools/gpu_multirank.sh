bash tools/gpu_t.sh tests/test_gpu_multirank.py
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --frames 2000 --no-cpu --cfg4-frames 0 --file-frames 0 > gpurun_out/bench_2rank.log 2>&1; echo bench2=$?; tail -c 1500 gpurun_out/bench_2rank.log
