"""Why does the fused kernel's per-frame time grow with the frame-sets resident per step
(1.18 us at 2k, 1.25 us at 10k)?  Same kernel, same per-launch work:
  a) 10k frame-sets in one buffer, one launch;  b) a 2k buffer alone;
  c) a 2k buffer next to an untouched 40 GB allocation;  d) 10k frame-sets as 5 buffers of 2k,
  5 launches per step;  e) 10k in one buffer, 5 launches over 2k sub-ranges."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)


def make(F, seed):
    iq = torch.empty(corr.iq_shape(F), dtype=torch.float32, device=dev)
    for s0 in range(0, F, 1000):
        e0 = min(F, s0 + 1000)
        h = S.draw_channel(corr, e0 - s0, seed=seed + s0)
        S.simulate_frames(corr, h, 10.0, seed=seed + 7 + s0, out=iq[s0:e0])
    return iq


def timeit(launch, frames, reps=6):
    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps / frames


which = sys.argv[1]
if which == "a":
    iq = make(10000, 1); taps = torch.empty(corr.taps_shape(10000), dtype=torch.complex64, device=dev)
    print("a 10k one buffer", round(timeit(lambda: corr.process(iq, out=taps), 10000), 4))
    print("e 10k one buffer, 5 launches", round(timeit(lambda: [corr.process(iq[i:i + 2000], out=taps[i:i + 2000])
                                                               for i in range(0, 10000, 2000)], 10000), 4))
elif which == "b":
    iq = make(2000, 1); taps = torch.empty(corr.taps_shape(2000), dtype=torch.complex64, device=dev)
    print("b 2k buffer", round(timeit(lambda: corr.process(iq, out=taps), 2000), 4))
    pad = torch.empty(40 * 2**30, dtype=torch.uint8, device=dev)
    print("c 2k buffer + 40 GB allocated", round(timeit(lambda: corr.process(iq, out=taps), 2000), 4))
    del pad
elif which == "d":
    iqs = [make(2000, 1 + i * 10000) for i in range(5)]
    tps = [torch.empty(corr.taps_shape(2000), dtype=torch.complex64, device=dev) for _ in range(5)]
    print("d 5 buffers x 2k, 5 launches", round(timeit(lambda: [corr.process(a, out=b) for a, b in zip(iqs, tps)], 10000), 4))
