mkdir -p gpurun_out
for g in 128 64 96 192; do PNCE_TUNE_NARROW_G=$g timeout -s KILL 120 python tools/narrow_g_trial.py g$g >> gpurun_out/ng.txt 2>&1; echo "g$g rc=$?" >> gpurun_out/ng.txt; done
PNCE_TUNE_NARROW=0 timeout -s KILL 120 python tools/narrow_g_trial.py wide >> gpurun_out/ng.txt 2>&1; echo "wide rc=$?" >> gpurun_out/ng.txt
python - >> gpurun_out/ng.txt 2>&1 <<'PY'
import torch, os
ref = torch.load("gpurun_out/narrow_wide.pt")
for t in ("g128", "g64", "g96", "g192"):
    p = f"gpurun_out/narrow_{t}.pt"
    if os.path.exists(p):
        d = torch.load(p); print(t, "bit-identical to wide:", all(torch.equal(d[n], ref[n]) for n in ref))
PY
cat gpurun_out/ng.txt
rm -f gpurun_out/narrow_*.pt
