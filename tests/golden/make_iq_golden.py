"""Golden IQ files written by the REAL reference (`pnce.iqfile`), for the IQ ingest (f2).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_iq_golden.py

Writes tests/golden/ref_frames.iq (reference `write_iq_bytes` of simulated frames:
4x4 MIMO, M=127, C=L=16, N_b=2 -> 2 batches per frame-set, 3 frame-sets) and
tests/golden/ref_frames.npz (the reference's own `read_iq_bytes` of it, the truth taps
per frame-set and the reference64 `process_frames` estimates).  Nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from pnce.channel import ChannelSpec, SnrSpec, simulate_frame  # noqa: E402
from pnce.experiments import process_frames  # noqa: E402
from pnce.halfprec import REFERENCE64  # noqa: E402
from pnce.iqfile import IqFileHeader, read_iq_bytes, write_iq_bytes  # noqa: E402
from pnce.pilots import PilotConfig, build_batch_plan  # noqa: E402
from pnce.pn import default_spec, generate_mseq  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    n_t = n_r = 4
    m, l, nb, sets = 127, 16, 2, 3
    cfg = PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
    seq = generate_mseq(default_spec(7))
    plan = build_batch_plan(cfg)
    frames, truths, ests = [], [], []
    for k in range(sets):
        chan = ChannelSpec(l=l, l_nz=l, n_t=n_t, n_r=n_r, seed=100 + k)
        truth, fr = simulate_frame(cfg, chan, SnrSpec(10.0, noise_seed=200 + k), seq)
        frames += fr
        truths.append(truth.taps)
        ests.append(process_frames(seq, cfg, plan, fr, REFERENCE64).taps)
    header = IqFileHeader(n_t=n_t, n_r=n_r, p=cfg.p, l=l, m=m, c=l, n_batch=nb,
                          frame_count=len(frames), seed=100)
    raw = write_iq_bytes(header, frames)
    with open(os.path.join(HERE, "ref_frames.iq"), "wb") as fh:
        fh.write(raw)
    _, back = read_iq_bytes(raw)
    np.savez_compressed(os.path.join(HERE, "ref_frames.npz"),
                        samples=np.stack([f.samples for f in back]),      # (frames, n_r, P+L-1) c128
                        truth=np.stack(truths), est_ref64=np.stack(ests),
                        geometry=np.array([n_t, n_r, m, l, l, nb, len(frames)]))
    print("wrote", len(raw), "bytes,", len(frames), "frames")


if __name__ == "__main__":
    main()
