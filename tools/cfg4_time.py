"""BASELINE configs[3] (cfg4': 128x128 MIMO, PN 2047, L=C=127, N_b=16 -> R=2032, 4 lag-row
groups) on one GPU: fused, packed-GEMM and scored legs, tensor fraction of the bf16 peak."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

PEAK = 1645.7e12
dev = torch.device("cuda:0")
F = int(sys.argv[1]) if len(sys.argv) > 1 else 512
LEGS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fused", "packed", "scored"]
cfg = P.PilotConfig(m=2047, c=127, n_t=128, n_batch=16, l=127, f_s=10e6)
corr = P.Correlator(P.default_spec(11), cfg, 128, device=dev)
h = S.draw_channel(corr, F, seed=1)
iq = S.simulate_frames(corr, h, 10.0, seed=2)
flop = 4.0 * cfg.n_t * cfg.l * cfg.m * 128


def timed(fn, reps=5):
    fn()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps / F


taps, _ = corr.process(iq)
if "fused" in LEGS:
  t = timed(lambda: corr.process(iq, out=taps))
  print(f"cfg4' fused   {t:8.3f} us/frame-set  {flop / (t * 1e-6) / PEAK * 100:5.1f} % of bf16 peak")
if "packed" in LEGS:
  packed = corr.pack(iq)
  t = timed(lambda: corr.correlate(packed, F, out=taps))
  print(f"cfg4' packed  {t:8.3f} us/frame-set  {flop / (t * 1e-6) / PEAK * 100:5.1f} % of bf16 peak")
if "scored" in LEGS:
  t = timed(lambda: corr.process_scored(iq, h, out=taps))
  print(f"cfg4' scored  {t:8.3f} us/frame-set  {flop / (t * 1e-6) / PEAK * 100:5.1f} % of bf16 peak")
