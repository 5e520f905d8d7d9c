mkdir -p gpurun_out
timeout -s KILL 120 tools/bin/store_probe > gpurun_out/store_probe.txt 2>&1; echo probe=$?
T="--frames 4096 --steps 1 --warmup 3 --no-gemm-leg --no-e2e --no-cpu"
PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace_v5.bin timeout -s KILL 200 python bench.py $T > gpurun_out/trace_v5.log 2>&1; echo trace=$?
PNCE_LIB=tools/bin/libpnce_diag_trace_pipe.so PNCE_TRACE_FILE=gpurun_out/trace_v5_pipe.bin timeout -s KILL 200 python bench.py $T > /dev/null 2>&1; echo trace2=$?
