"""Golden tensor16 estimates from the REAL reference (`pnce.halfprec` through
`process_frames`), for the binary16/binary32 chunked-accumulation mode.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_t16_golden.py

cfg2 geometry (16x16, M=255, L=C=32, N_b=4), two seeded frame-sets at 10 dB.  Cases:
  b32  : tensor16, chunk_len 256, binary32 partials
  b16  : tensor16, chunk_len 64, binary16 partials (no saturation at unit amplitude)
  sat  : tensor16, chunk_len 256, binary16, the received batches scaled by (3000, 1000,
         3000, 500) so that batches 0 and 2 overflow binary16 (peak partial ~81000 > 65504)
         and 1, 3 do not (~27000, ~13500); the reference counts and zeroes 0 and 2
Writes tests/golden/t16.npz (f32 IQ payloads, truth, reference taps, saturations).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from pnce.channel import ChannelSpec, ReceivedFrame, SnrSpec, simulate_frame  # noqa: E402
from pnce.experiments import _derive_seeds, process_frames  # noqa: E402
from pnce.halfprec import BackendConfig  # noqa: E402
from pnce.pilots import PilotConfig, build_batch_plan  # noqa: E402
from pnce.pn import default_spec, generate_mseq  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def to_f32(frames, scales):
    """Frames as the IQ file stores them (float32 I/Q), batch b scaled by scales[b] first."""
    out = []
    for f, sc in zip(frames, scales):
        s = f.samples * sc
        s = s.real.astype(np.float32).astype(np.float64) + 1j * s.imag.astype(np.float32).astype(np.float64)
        out.append(ReceivedFrame(samples=s, batch_index=f.batch_index))
    return out


def main():
    n, m, l, nb = 16, 255, 32, 4
    cfg = PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
    seq = generate_mseq(default_spec(8))
    plan = build_batch_plan(cfg)
    cases = {"b32": (256, "binary32", (1.0,) * 4), "b16": (64, "binary16", (1.0,) * 4),
             "sat": (256, "binary16", (3000.0, 1000.0, 3000.0, 500.0))}
    out = {}
    for name, (chunk, acc, scale) in cases.items():
        iqs, truths, taps, sats = [], [], [], []
        for it in range(2):
            cs, ns = _derive_seeds(0, m, nb, l, 2, it)
            truth, frames = simulate_frame(cfg, ChannelSpec(l=l, l_nz=l, n_t=n, n_r=n, seed=cs), SnrSpec(10.0, ns), seq)
            frames = to_f32(frames, scale)
            est = process_frames(seq, cfg, plan, frames, BackendConfig(kind="tensor16", chunk_len=chunk, accumulator=acc))
            iqs.append(np.stack([np.stack([f.samples.real, f.samples.imag], -1) for f in frames]).astype(np.float32))
            truths.append(truth.taps * np.repeat(np.asarray(scale), nb)[None, :, None])
            taps.append(est.taps)
            sats.append(est.saturations)
        out[f"{name}_iq"] = np.stack(iqs)
        out[f"{name}_truth"] = np.stack(truths)
        out[f"{name}_taps"] = np.stack(taps)
        out[f"{name}_sat"] = np.array(sats)
        out[f"{name}_cfg"] = np.array([chunk, 1 if acc == "binary16" else 0])
        print(name, "saturations", sats)
    np.savez_compressed(os.path.join(HERE, "t16.npz"), **out)


if __name__ == "__main__":
    main()
