for LF in 0 2048 1024 5000; do
  python bench.py --frames 10000 --launch-frames $LF --no-e2e --no-cpu --latency-reps 0 --antenna-reps 0 --file-frames 0 --steps 10 --no-quality --no-gemm-leg --cfg4-frames 0 > gpurun_out/lf_$LF.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/lf_$LF.json').read().strip().splitlines()[-1]);print($LF, round(d['us_per_frame'],4), round(d['roofline']['frac'],3), d['gpu_launches'], d['clocks']['power_w'])"
done
nvidia-smi -q -d CLOCK | head -40
