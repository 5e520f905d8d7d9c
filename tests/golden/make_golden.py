"""Generate golden vectors by running the REAL reference package (`pnce`).

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (read-only) and writes
tests/golden/golden.npz.  The fixtures pin the CPU oracle (oracle/pnce_oracle.py)
and, transitively, the CUDA path.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from pnce.channel import ChannelSpec, SnrSpec, simulate_frame  # noqa: E402
from pnce.experiments import _derive_seeds, process_frames  # noqa: E402
from pnce.halfprec import BackendConfig, REFERENCE64  # noqa: E402
from pnce.iqfile import _HEADER, IqFileHeader, read_iq_bytes, write_iq_bytes  # noqa: E402
from pnce.metrics import mae  # noqa: E402
from pnce.pilots import PilotConfig, build_batch_plan  # noqa: E402
from pnce.pn import LfsrSpec, default_spec, generate_mseq  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# name: (n_t=n_r, m, l=c, n_batch)
CONFIGS = {
    "cfg1": (4, 127, 16, 1),
    "cfg2": (16, 255, 32, 4),
    "cfg3": (64, 1023, 64, 8),
    "cfg4p": (128, 2047, 127, 16),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def seq_for(m: int):
    degree = (m + 1).bit_length() - 1
    return generate_mseq(default_spec(degree))


def to_iq(frames) -> np.ndarray:
    """Round-trip through the reference's own IQ file writer/reader (iqfile.py)."""
    n_r, s = frames[0].samples.shape
    hdr = IqFileHeader(n_t=1, n_r=n_r, p=1, l=s, m=1, c=0, n_batch=1,
                       frame_count=len(frames), seed=0)
    raw = write_iq_bytes(hdr, frames)
    _, back = read_iq_bytes(raw)
    iq = np.frombuffer(raw, dtype="<f4", offset=_HEADER.size).reshape(len(frames), n_r, s, 2)
    return iq.copy(), back


def main() -> None:
    g: dict[str, np.ndarray] = {}

    # --- a1 KATs: chips for every built-in degree plus the explicit degree-12 spec
    for degree in range(2, 12):
        chips = generate_mseq(default_spec(degree)).chips
        g[f"chips_d{degree}"] = np.packbits(chips < 0)
    chips12 = generate_mseq(LfsrSpec(degree=12, taps=(12, 6, 4, 1), state=1)).chips
    g["chips_d12"] = np.packbits(chips12 < 0)
    # non-default start state
    g["chips_d10_state77"] = np.packbits(generate_mseq(default_spec(10, state=77)).chips < 0)

    # --- per-config frame sets: 10 dB, master seed 0, seed key (m, n_b, l_nz, 0, it)
    for name, (n, m, l, nb) in CONFIGS.items():
        cfg = PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
        plan = build_batch_plan(cfg)
        g[f"{name}_shifts"] = np.array([[a.shift for a in b] + [-1] * (nb - len(b)) for b in plan.batches])
        seq = seq_for(m)
        n_sets = {"cfg1": 6, "cfg2": 2, "cfg3": 1, "cfg4p": 1}[name]
        for it in range(n_sets):
            cs, ns = _derive_seeds(0, m, nb, l, 0, it)
            truth, frames = simulate_frame(cfg, ChannelSpec(l=l, l_nz=l, n_t=n, n_r=n, seed=cs),
                                           SnrSpec(10.0, noise_seed=ns), seq)
            iq, frames32 = to_iq(frames)
            est_raw = process_frames(seq, cfg, plan, frames, REFERENCE64).taps
            est32 = process_frames(seq, cfg, plan, frames32, REFERENCE64).taps
            key = f"{name}_it{it}"
            g[f"{key}_seeds"] = np.array([cs, ns], dtype=np.uint64)
            g[f"{key}_iq_sha"] = np.array(sha(iq))
            g[f"{key}_truth_sha"] = np.array(sha(truth.taps))
            g[f"{key}_mae_raw"] = np.array(mae(truth, est_raw))
            g[f"{key}_mae32"] = np.array(mae(truth, est32))
            g[f"{key}_mse32"] = np.array(float(np.mean(np.abs(est32 - truth.taps) ** 2)))
            if name in ("cfg1", "cfg2"):
                g[f"{key}_iq"] = iq
                g[f"{key}_truth"] = truth.taps
                g[f"{key}_est32"] = est32
                chunk = 128 if m == 127 else 256
                t16 = process_frames(seq, cfg, plan, frames32,
                                     BackendConfig(kind="tensor16", chunk_len=chunk)).taps
                g[f"{key}_est_t16"] = t16
            else:
                rng = np.random.default_rng(5)
                idx = rng.integers(0, est32.size, size=4096)
                g[f"{key}_sample_idx"] = idx
                g[f"{key}_sample_est32"] = est32.reshape(-1)[idx]
                g[f"{key}_sample_truth"] = truth.taps.reshape(-1)[idx]

    # --- MAE/MSE-vs-SNR anchor curve: cfg2, master seed 0, grid index = seed key
    n, m, l, nb = CONFIGS["cfg2"]
    cfg = PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
    plan = build_batch_plan(cfg)
    seq = seq_for(m)
    grid = (-10.0, 0.0, 10.0, 20.0, 30.0)
    iters = 8
    curve_mae = np.zeros((len(grid), iters))
    curve_mse = np.zeros((len(grid), iters))
    for si, snr in enumerate(grid):
        for it in range(iters):
            cs, ns = _derive_seeds(0, m, nb, l, si, it)
            truth, frames = simulate_frame(cfg, ChannelSpec(l=l, l_nz=l, n_t=n, n_r=n, seed=cs),
                                           SnrSpec(snr, noise_seed=ns), seq)
            _, frames32 = to_iq(frames)
            est = process_frames(seq, cfg, plan, frames32, REFERENCE64).taps
            curve_mae[si, it] = mae(truth, est)
            curve_mse[si, it] = float(np.mean(np.abs(est - truth.taps) ** 2))
    g["curve_snr"] = np.array(grid)
    g["curve_mae32"] = curve_mae
    g["curve_mse32"] = curve_mse

    # --- noiseless cfg3 (per-lag bound of Eq. 4 / acceptance criterion 3 style)
    n, m, l, nb = CONFIGS["cfg3"]
    cfg = PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
    cs, _ = _derive_seeds(0, m, nb, l, 99, 0)
    truth, frames = simulate_frame(cfg, ChannelSpec(l=l, l_nz=l, n_t=n, n_r=n, seed=cs),
                                   SnrSpec(math.inf), seq_for(m))
    iq, frames32 = to_iq(frames)
    est32 = process_frames(seq_for(m), cfg, build_batch_plan(cfg), frames32, REFERENCE64).taps
    g["cfg3_noiseless_seed"] = np.array(cs, dtype=np.uint64)
    g["cfg3_noiseless_iq_sha"] = np.array(sha(iq))
    g["cfg3_noiseless_mae32"] = np.array(mae(truth, est32))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {os.path.getsize(OUT) / 1e6:.2f} MB, {len(g)} arrays")


if __name__ == "__main__":
    main()
