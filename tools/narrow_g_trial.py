"""Few-frame-set plain launch: latency and taps under the current PNCE_TUNE_* environment.

Run once per knob setting (knobs are read once per process); writes the taps of 1..4
frame-sets to gpurun_out/narrow_<tag>.pt so the settings can be compared bit for bit.
    PNCE_TUNE_NARROW_G=64 python tools/narrow_g_trial.py g64 [1,2,4]
"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import _lib  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

tag = sys.argv[1]
dev = torch.device("cuda", 0)
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
L = _lib.lib()
NS = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (1, 2, 4)
iq = torch.empty(corr.iq_shape(max(NS)), dtype=torch.float32, device=dev)
h = S.draw_channel(corr, max(NS), seed=11)
S.simulate_frames(corr, h, 10.0, seed=12, out=iq)
s = torch.cuda.current_stream(dev)
out = {}
for n in NS:
    taps = torch.empty(corr.taps_shape(n), dtype=torch.complex64, device=dev)
    ts = []
    for i in range(55):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        _lib.check(L.pnce_process_frames(corr._plan, ctypes.c_void_p(iq.data_ptr()), ctypes.c_void_p(taps.data_ptr()),
                                         None, None, None, 0, n, ctypes.c_void_p(s.cuda_stream)))
        b.record(s)
        b.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    out[n] = taps.cpu()
    print(f"{tag:8s} frame-sets={n}  median {statistics.median(ts):6.1f} us  min {min(ts):6.1f} us")
torch.save(out, f"gpurun_out/narrow_{tag}.pt")
