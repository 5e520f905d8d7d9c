"""Small workload that exercises every kernel mode of libpnce_b200.so, for compute-sanitizer
(memcheck / racecheck / synccheck): plain (narrow, mid, wide tilings), scored (per-frame sums +
per-link MSE + saturation finish), packed GEMM, tensor16 (binary16 / binary32), the LDG
converter mode, compact bodies, the operator seam, and the synthesiser.  cfg1 / cfg2 sizes so
the sanitizer finishes in minutes.  Run through tools/gpu_sanitize.sh (one mode per process
for the knob-selected variants)."""

import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402
from paper_2206_05506_b200.backend import BackendConfig  # noqa: E402


def run(dev):
    for (n, m, l, nb, F) in ((4, 127, 16, 1, 3), (16, 255, 32, 4, 2), (16, 1023, 64, 8, 9), (16, 2047, 127, 16, 2)):
        cfg = P.PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
        corr = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n, device=dev)
        h = S.draw_channel(corr, F, seed=1)
        iq = S.simulate_frames(corr, h, 10.0, seed=2)
        iq[0, 0, 0, l + 3, 0] = float("inf")                 # one saturated batch
        for f in (1, F):                                      # few-tile (narrow/mid) and wide launches
            corr.process(iq[:f])
            corr.process_scored(iq[:f], h[:f])
            corr.process_tensor16(iq[:f], chunk_len=64, accumulator="binary16", truth=h[:f])
            corr.process_tensor16(iq[:f], chunk_len=None, accumulator="binary32")
            packed = corr.pack(iq[:f])
            corr.correlate(packed, f, truth=h[:f])
        seq = P.sequence_for_length(m, dev)
        P.process_frames(seq, cfg, P.build_batch_plan(cfg), iq[0], backend=BackendConfig(kind="tensor16", chunk_len=64),
                         rows_per_batch=corr, truth=h[0])
        hi = torch.empty(corr.iq_shape(F), dtype=torch.float32).pin_memory()
        hi.copy_(iq.cpu())
        ht = torch.empty(corr.taps_shape(F), dtype=torch.complex64).pin_memory()
        corr.process_host(hi, ht, chunk=2)
        S.simulate_frames(corr, h, math.inf)
        if n >= 4:  # the fused antenna gather: half the receivers into two full-CSI buffers
            part = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n // 2, device=dev)
            bufs = [torch.zeros(corr.taps_shape(F), dtype=torch.complex64, device=dev) for _ in range(2)]
            part.process_gather(iq[:, :, n // 2:].contiguous(), bufs[0], n // 2, peers=bufs[1:])
    rows = np.sign(np.random.default_rng(0).standard_normal((40, 255)))
    y = np.random.default_rng(1).standard_normal((255, 3)) + 1j
    P.correlate_rows(rows, y)
    P.correlate_rows(rows, y, backend=BackendConfig(kind="tensor16", chunk_len=128))
    torch.cuda.synchronize(dev)
    print("sanitize workload ok", os.environ.get("PNCE_TUNE_FUSED_MODE", "default"))


if __name__ == "__main__":
    run(torch.device("cuda:0"))
