#!/bin/bash
# 5-9 cfg3 frame-sets per plain launch: the 256-column "mid" tiling (PNCE_TUNE_MID=1 TMA ring,
# 2 LDG converters) against the single 512-column group (0); taps compared bit for bit.
mkdir -p gpurun_out
N=1,4,5,6,8,9,10,16
for m in 0 1 2; do PNCE_TUNE_MID=$m timeout -s KILL 120 python tools/narrow_g_trial.py mid$m $N >> gpurun_out/mid.txt 2>&1; echo "mid$m rc=$?" >> gpurun_out/mid.txt; done
python - >> gpurun_out/mid.txt 2>&1 <<'PY'
import torch, os
ref = torch.load("gpurun_out/narrow_mid0.pt")
for t in ("mid1", "mid2"):
    p = f"gpurun_out/narrow_{t}.pt"
    if os.path.exists(p):
        d = torch.load(p); print(t, "bit-identical to mid0:", all(torch.equal(d[n], ref[n]) for n in ref))
PY
rm -f gpurun_out/narrow_*.pt
cat gpurun_out/mid.txt
