"""Single frame-set latency of the fused kernel vs the split-K low-latency mode (cfg3)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
F = int(sys.argv[1]) if len(sys.argv) > 1 else 1
h = S.draw_channel(corr, F, seed=1)
iq = S.simulate_frames(corr, h, 10.0, seed=2)
out = torch.empty(corr.taps_shape(F), dtype=torch.complex64, device=dev)


def lat(fn, reps=60):
    ts = []
    for i in range(reps + 5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts), min(ts)


print(f"F={F}  fused          median %.1f us  min %.1f us" % lat(lambda: corr.process(iq, out=out)))
for ks in (2, 4, 8, 16):
    print(f"F={F}  split k={ks:2d}     median %.1f us  min %.1f us" % lat(lambda: corr.process_low_latency(iq, ks, out=out)))
