"""Time the device synthesiser (untimed input of the bench; the sweeps' inner loop)."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
for (n_t, n_r, m, l, nb, F) in [(64, 64, 1023, 64, 8, 2048), (32, 256, 4095, 256, 8, 8), (16, 16, 255, 32, 4, 4096)]:
    deg = (m + 1).bit_length() - 1
    spec = P.LfsrSpec(12, (12, 6, 4, 1), 1) if deg == 12 else P.default_spec(deg)
    cfg = P.PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(spec, cfg, n_r, device=dev)
    h = S.draw_channel(corr, F, seed=1)
    iq = S.simulate_frames(corr, h, 10.0, seed=2)       # warm-up (plan cache, cuBLAS)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = S.draw_channel(corr, F, seed=3)
    S.simulate_frames(corr, h, 10.0, seed=4, out=iq)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    taps, _ = corr.process(iq)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    corr.process(iq, out=taps)
    torch.cuda.synchronize()
    de = time.perf_counter() - t1
    print(f"n_t={n_t} n_r={n_r} M={m} L={l} N_b={nb}: synth {dt / F * 1e6:9.1f} us/frame-set, "
          f"estimate {de / F * 1e6:8.2f} us/frame-set (F={F})")
