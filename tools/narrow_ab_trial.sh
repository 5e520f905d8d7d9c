#!/bin/bash
# Few-frame-set (narrow tiling) launches: A/B stage depth sweep (PNCE_TUNE_AB_STAGES), taps
# compared bit for bit with the default; plus the trace of one launch at the best depth.
mkdir -p gpurun_out
for ab in 3 4 5 6 7; do PNCE_TUNE_AB_STAGES=$ab timeout -s KILL 120 python tools/narrow_g_trial.py ab$ab >> gpurun_out/ab.txt 2>&1; echo "ab$ab rc=$?" >> gpurun_out/ab.txt; done
python - >> gpurun_out/ab.txt 2>&1 <<'PY'
import torch, os
ref = torch.load("gpurun_out/narrow_ab3.pt")
for t in ("ab4", "ab5", "ab6", "ab7"):
    p = f"gpurun_out/narrow_{t}.pt"
    if os.path.exists(p):
        d = torch.load(p); print(t, "bit-identical to ab3:", all(torch.equal(d[n], ref[n]) for n in ref))
PY
PNCE_TUNE_AB_STAGES=6 PNCE_LIB=tools/bin/libpnce_diag_trace.so PNCE_TRACE_FILE=gpurun_out/trace_lat_ab6.bin timeout -s KILL 120 python tools/narrow_g_trial.py t6 1 > /dev/null 2>&1
rm -f gpurun_out/narrow_*.pt
cat gpurun_out/ab.txt
