"""IQ-file ingest sweep: reader threads x piece size x staging chunk for
iqfile.estimate_file on a cfg3 reference-format file in the page cache; host wall clock.

    python tools/ingest_sweep.py [--frames 256]
"""
import argparse
import itertools
import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_05506_b200 import PilotConfig, default_spec  # noqa: E402
from paper_2206_05506_b200 import iqfile as IQ  # noqa: E402
from paper_2206_05506_b200.estimator import Correlator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=256)
    a = ap.parse_args()
    cfg = PilotConfig(m=1023, c=64, l=64, n_t=64, n_batch=8, f_s=10e6)
    corr = Correlator(default_spec(10), cfg, 64, "fp16", device="cuda:0")
    F = a.frames
    iq = torch.randn(corr.iq_shape(F), dtype=torch.float32, device="cuda")
    hdr = IQ.IqFileHeader(n_t=64, n_r=64, p=64 + 1023, l=64, m=1023, c=64, n_batch=8,
                          frame_count=F * cfg.n_batches, seed=1)
    print(f"host cpus {os.cpu_count()}")
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "frames.iq")
        IQ.write_iq_tensor(path, hdr, iq)
        size = os.path.getsize(path)
        taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64).pin_memory()
        for threads, piece_mb, chunk in itertools.product((16,), (2, 4, 8), (8, 16, 32)):
            IQ._READ_THREADS = threads
            IQ._PIECE = piece_mb << 20
            IQ._POOL = None
            IQ.estimate_file(path, corr, chunk_sets=chunk, taps_host=taps)
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                IQ.estimate_file(path, corr, chunk_sets=chunk, taps_host=taps)
                ts.append(time.perf_counter() - t0)
            t = min(ts)
            print(f"threads {threads:2d} piece {piece_mb:2d} MB chunk {chunk:3d}: {t / F * 1e6:7.1f} us/frame-set "
                  f"{size / t / 1e9:6.1f} GB/s")


if __name__ == "__main__":
    main()
