"""tensor16 (binary16, chunk 256) on cfg3 frame-sets resident in HBM, as bench.py's tensor16 leg:
us per frame-set (median of 5 launches).  Knobs come from the environment."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
F = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
acc = sys.argv[2] if len(sys.argv) > 2 else "binary16"
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
h = S.draw_channel(corr, F, seed=1)
iq = S.simulate_frames(corr, h, 10.0, seed=2)
taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64, device=dev)
st = torch.zeros((F, 4), dtype=torch.float64, device=dev)
ts = []
for i in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    corr.process_tensor16(iq, chunk_len=256, accumulator=acc, out=taps, stats=st)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1) * 1e3 / F)
ts.sort()
print(f"tensor16 {acc} {ts[len(ts) // 2]:.3f} us/frame-set")
