"""A few single frame-set launches (cfg1, cfg3) for an ncu launch list (kernel-only duration)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
for (n, m, l, nb) in ((4, 127, 16, 1), (64, 1023, 64, 8)):
    cfg = P.PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n, device=dev)
    h = S.draw_channel(corr, 1, seed=1)
    iq = S.simulate_frames(corr, h, 10.0, seed=2)
    taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64, device=dev)
    for i in range(5):
        corr.process(iq, out=taps)
    torch.cuda.synchronize()
