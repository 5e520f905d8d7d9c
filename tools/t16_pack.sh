#!/bin/bash
# tensor16 binary16 folds: .pack::16b partial loads (PNCE_TUNE_T16_PACK=1) -- bit-identical? faster?
python - <<'PY'
import os, subprocess, sys, numpy as np
code = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2206_05506_b200 as P
from paper_2206_05506_b200 import synth as S
dev = torch.device('cuda:0')
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
h = S.draw_channel(corr, 16, seed=3); iq = S.simulate_frames(corr, h, 10.0, seed=4)
t, st = corr.process_tensor16(iq, chunk_len=256, accumulator='binary16', truth=h)
np.save(sys.argv[1], t.cpu().numpy())
"""
outs = []
for v in ("0", "1"):
    env = dict(os.environ, PNCE_TUNE_T16_PACK=v)
    subprocess.run([sys.executable, "-c", code, f"/tmp/t16_{v}.npy"], env=env, check=True)
    outs.append(np.load(f"/tmp/t16_{v}.npy"))
print("bit-identical:", np.array_equal(outs[0], outs[1]), "max diff", float(np.abs(outs[0] - outs[1]).max()))
PY
for spec in "X=1" "PNCE_TUNE_T16_PACK=1" "X=1" "PNCE_TUNE_T16_PACK=1"; do
  echo "$spec: $(env $spec timeout -s KILL 300 python tools/t16_time.py 2048 2>&1 | tail -1)"
done
