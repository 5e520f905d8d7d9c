"""Cycle accounting of the scored kernel (run with PNCE_LIB=tools/bin/libpnce_diag_prof.so
PNCE_PROF_FILE=...): cfg3, 2048 frame-sets, taps + sums + per-link MSE."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
F = 2048
h = S.draw_channel(corr, F, seed=1)
iq = S.simulate_frames(corr, h, 10.0, seed=2)
for _ in range(2):
    taps, st, lk = corr.process_scored(iq, h)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
corr.process_scored(iq, h, out=taps)
e1.record()
torch.cuda.synchronize()
print(f"scored {e0.elapsed_time(e1) * 1e3 / F:.3f} us/frame-set")
