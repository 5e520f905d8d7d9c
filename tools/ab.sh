#!/bin/bash
# A/B of tuning knobs within ONE gpurun call (boxes differ by ~7 %): each line
# "NAME ENV=.. ENV=.." runs the bench legs with those variables; prints the key numbers.
#   tools/ab.sh spec_file [bench args]
mkdir -p gpurun_out
SPEC=$1; shift
ARGS=${@:-"--no-e2e --no-cpu --cfg4-frames 0 --latency-reps 0 --antenna-reps 0 --file-frames 0 --steps 10"}
while read -r name envs; do
  [ -z "$name" ] && continue
  for rep in 1 2; do
    env $envs timeout -s KILL 300 python bench.py $ARGS > gpurun_out/ab_${name}_$rep.json 2>gpurun_out/ab_${name}_$rep.err
    python - "$name" "gpurun_out/ab_${name}_$rep.json" <<'PY'
import json, sys
name, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
except Exception as e:
    print(name, "FAILED", e); sys.exit(0)
g = d.get("gemm_leg") or {}
q = d.get("estimate_quality") or {}
t = d.get("tensor16_leg") or {}
c4 = d.get("cfg4_leg") or {}
print(f"{name:24s} fused {d['us_per_frame']:.4f} us ({d['roofline']['frac']:.3f})  gemm {g.get('us_per_frame', 0):.4f} ({g.get('frac_of_bf16_peak', 0):.3f})"
      f"  scored {q.get('scored_us_per_frame', 0):.3f}  t16 {t.get('us_per_frame', 0):.3f}"
      + (f"  c4f {c4['fused']['us_per_frame']:.2f} c4g {c4['gemm']['us_per_frame']:.2f}" if c4 else "")
      + f"  [{(d.get('clocks') or {}).get('sm_mhz')} MHz {(d.get('clocks') or {}).get('power_w')} W]", flush=True)
PY
  done
done < "$SPEC"
