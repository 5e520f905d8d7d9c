for F in 2048 4096 6000 8000 10000 12000; do
  python bench.py --frames $F --no-e2e --no-cpu --latency-reps 0 --antenna-reps 0 --file-frames 0 --steps 10 --no-quality --no-gemm-leg --cfg4-frames 0 > gpurun_out/fs_$F.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/fs_$F.json').read().strip().splitlines()[-1]);print($F, round(d['us_per_frame'],4), round(d['roofline']['frac'],3), d['clocks'])"
done
