"""PCIe probe for the e2e leg: pinned host -> HBM copy rates for the cfg3 IQ payload as
one contiguous copy (whole rows incl. CP) and as the pitched body-only copy
(pnce_copy_bodies_h2d), alone and with the taps D2H running concurrently.

    python tools/pcie_probe.py [--frames 64]
"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05506_b200 import PilotConfig, _lib, default_spec  # noqa: E402
from paper_2206_05506_b200.estimator import Correlator  # noqa: E402


def timed(fn, streams, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for s in streams:
        s.wait_stream(cur)
    for _ in range(reps):
        fn()
    for s in streams:
        cur.wait_stream(s)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    a = ap.parse_args()
    cfg = PilotConfig(m=1023, c=64, l=64, n_t=64, n_batch=8, f_s=10e6)
    corr = Correlator(default_spec(10), cfg, 64, "fp16", device="cuda:0")
    F = a.frames
    h_iq = torch.empty(corr.iq_shape(F), dtype=torch.float32).pin_memory()
    h_iq.fill_(0.5)
    h_taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64).pin_memory()
    d_iq = torch.empty(corr.iq_shape(F), dtype=torch.float32, device="cuda")
    stride = cfg.m + 1
    d_body = torch.empty((F, cfg.n_batches, 64, stride, 2), dtype=torch.float32, device="cuda")
    d_taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64, device="cuda")
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    L = _lib.lib()
    full_b = h_iq.numel() * 4
    body_b = F * cfg.n_batches * 64 * cfg.m * 8
    taps_b = h_taps.numel() * 8

    def h2d_full():
        with torch.cuda.stream(s_in):
            d_iq.copy_(h_iq, non_blocking=True)

    def h2d_body():
        _lib.check(L.pnce_copy_bodies_h2d(corr._plan, ctypes.c_void_p(h_iq.data_ptr()),
                                          ctypes.c_void_p(d_body.data_ptr()), stride, F,
                                          ctypes.c_void_p(s_in.cuda_stream)))

    def d2h():
        with torch.cuda.stream(s_out):
            h_taps.copy_(d_taps, non_blocking=True)

    t = timed(h2d_full, [s_in])
    print(f"H2D contiguous   {full_b / 1e6:8.1f} MB  {t * 1e6:9.1f} us  {full_b / t / 1e9:6.1f} GB/s")
    t = timed(h2d_body, [s_in])
    print(f"H2D pitched body {body_b / 1e6:8.1f} MB  {t * 1e6:9.1f} us  {body_b / t / 1e9:6.1f} GB/s")
    t = timed(d2h, [s_out])
    print(f"D2H taps         {taps_b / 1e6:8.1f} MB  {t * 1e6:9.1f} us  {taps_b / t / 1e9:6.1f} GB/s")
    t = timed(lambda: (h2d_full(), d2h()), [s_in, s_out])
    print(f"H2D contiguous + D2H concurrently: {t * 1e6:9.1f} us  -> {full_b / t / 1e9:6.1f} GB/s in, "
          f"{taps_b / t / 1e9:6.1f} GB/s out; {t / F * 1e6:6.1f} us per frame-set")
    t = timed(lambda: (h2d_body(), d2h()), [s_in, s_out])
    print(f"H2D pitched   + D2H concurrently: {t * 1e6:9.1f} us  -> {body_b / t / 1e9:6.1f} GB/s in, "
          f"{taps_b / t / 1e9:6.1f} GB/s out; {t / F * 1e6:6.1f} us per frame-set")
    # split the pitched copy into per-frame-set pieces (many smaller DMAs)
    def h2d_body_split(parts=8):
        n = F // parts
        for i in range(parts):
            _lib.check(L.pnce_copy_bodies_h2d(corr._plan, ctypes.c_void_p(h_iq[i * n].data_ptr()),
                                              ctypes.c_void_p(d_body[i * n].data_ptr()), stride, n,
                                              ctypes.c_void_p(s_in.cuda_stream)))
    t = timed(h2d_body_split, [s_in])
    print(f"H2D pitched, 8 pieces: {body_b / t / 1e9:6.1f} GB/s")


if __name__ == "__main__":
    main()
