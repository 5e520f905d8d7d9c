"""Single frame-set launch latency (CUDA events around one launch, median of 200) for cfg1..cfg3:
separates the fixed launch + prologue cost from the K chain."""
import statistics
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
for name, (n, m, l, nb) in {"cfg1": (4, 127, 16, 1), "cfg2": (16, 255, 32, 4), "cfg3_nr8": (64, 1023, 64, 8),
                            "cfg3": (64, 1023, 64, 8)}.items():
    n_r = 8 if name == "cfg3_nr8" else n
    cfg = P.PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n_r, device=dev)
    h = S.draw_channel(corr, 1, seed=1)
    iq = S.simulate_frames(corr, h, 10.0, seed=2)
    taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64, device=dev)
    ts = []
    for i in range(220):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        corr.process(iq, out=taps)
        b.record()
        b.synchronize()
        if i >= 20:
            ts.append(a.elapsed_time(b) * 1e3)
    # empty-event baseline (event pair with nothing between)
    es = []
    for i in range(100):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        b.record()
        b.synchronize()
        es.append(a.elapsed_time(b) * 1e3)
    print(f"{name:9s} M={m:5d} K-blocks={-(-m // 64):3d}  median {statistics.median(ts):6.1f} us  min {min(ts):6.1f} us"
          f"  (empty event pair {statistics.median(es):.1f} us)", flush=True)
