"""Single frame-set launches under the trace build: PNCE_LIB=tools/bin/libpnce_diag_trace.so,
PNCE_TRACE_FILE=<path> (the last launch's timeline is kept)."""
import os
import shutil
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
out = os.environ["PNCE_TRACE_FILE"]
for name, (n, m, l, nb) in {"cfg1": (4, 127, 16, 1), "cfg3": (64, 1023, 64, 8)}.items():
    cfg = P.PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n, device=dev)
    h = S.draw_channel(corr, 1, seed=1)
    iq = S.simulate_frames(corr, h, 10.0, seed=2)
    taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64, device=dev)
    for i in range(4):
        corr.process(iq, out=taps)
    torch.cuda.synchronize()
    shutil.copy(out, out + "." + name)
    print(name, "traced")
