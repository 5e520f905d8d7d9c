mkdir -p gpurun_out
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests=$?"; tail -3 gpurun_out/gpu_tests.log
timeout -s KILL 600 python bench.py --no-cpu > gpurun_out/bench_base.log 2>&1; echo "bench=$?"; tail -c 3500 gpurun_out/bench_base.log
