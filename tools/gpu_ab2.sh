bash tools/ab.sh tools/ab_specs_2.txt
COMMON="--steps 1 --warmup 3 --no-e2e --no-cpu --latency-reps 0 --cfg4-frames 0 --antenna-reps 0 --file-frames 0 --frames 4096 --no-gemm-leg --no-quality"
PNCE_TUNE_FUSED_MODE=1 PNCE_LIB=tools/bin/libpnce_diag_prof.so PNCE_PROF_FILE=gpurun_out/prof.fm1.bin timeout -s KILL 200 python bench.py $COMMON > gpurun_out/prof.fm1.log 2>&1; echo "fm1=$?"
python tools/prof_view.py gpurun_out/prof.fm1.bin
