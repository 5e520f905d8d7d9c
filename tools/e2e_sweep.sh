mkdir -p gpurun_out
for c in ${CHUNKS:-2 4 8 16 32 64}; do
 timeout -s KILL 300 python bench.py --frames 1024 --steps 4 --no-quality --no-gemm-leg --no-cpu --file-frames 0 --e2e-chunk $c 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('chunk $c e2e us/frame %.2f'%d['e2e']['us_per_frame'])
"
done
