#!/bin/bash
# Few-frame-set (narrow tiling) launches: LDG converter mode (PNCE_TUNE_FUSED_MODE=1, no raw
# smem ring) x A/B stage depth, taps compared bit for bit with the default (TMA raw ring).
mkdir -p gpurun_out
timeout -s KILL 120 python tools/narrow_g_trial.py base >> gpurun_out/mode.txt 2>&1
for ab in 3 5 8; do PNCE_TUNE_FUSED_MODE=1 PNCE_TUNE_AB_STAGES=$ab timeout -s KILL 120 python tools/narrow_g_trial.py ldg$ab >> gpurun_out/mode.txt 2>&1; echo "ldg$ab rc=$?" >> gpurun_out/mode.txt; done
python - >> gpurun_out/mode.txt 2>&1 <<'PY'
import torch, os
ref = torch.load("gpurun_out/narrow_base.pt")
for t in ("ldg3", "ldg5", "ldg8"):
    p = f"gpurun_out/narrow_{t}.pt"
    if os.path.exists(p):
        d = torch.load(p); print(t, "bit-identical to base:", all(torch.equal(d[n], ref[n]) for n in ref))
PY
rm -f gpurun_out/narrow_*.pt
cat gpurun_out/mode.txt
