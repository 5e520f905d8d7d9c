"""BASELINE configs[4] coverage: corners of the parameter sweep (PN 127..4095 x CIR 8..256
x N_b 1..32) at 256 receive antennas, each against the oracle (per-link tolerance 1e-2)
on frames from the device synthesiser.  Only feasible points exist (L <= M, N_b <=
floor(M/L), shift spacing >= L; pilots.py:39-42, 134-142)."""

import math

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from paper_2206_05506_b200 import synth as S
from oracle import pnce_oracle as O

pytestmark = pytest.mark.gpu

POINTS = [
    # (m, l, n_batch, n_t)
    (4095, 256, 8, 32),     # longest PN, longest CIR: R = 2048 lag rows, K = 4096
    (4095, 8, 32, 32),      # longest PN, 32 multiplexed Tx of 8 taps
    (2047, 128, 8, 32),
    (511, 16, 16, 32),
    (127, 8, 8, 16),        # shortest PN, multiplexed
    (127, 64, 1, 8),        # shortest PN, one Tx per slot
]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


@pytest.mark.parametrize("m,l,nb,n_t", POINTS)
def test_sweep_corner(dev, m, l, nb, n_t):
    n_r = 256
    cfg = P.PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
    ocfg = O.Config(m=m, c=l, n_t=n_t, n_batch=nb, l=l, n_r=n_r)
    deg = (m + 1).bit_length() - 1
    # degree 12 has no built-in polynomial in the reference (pn.py:25-36): explicit taps
    spec = P.LfsrSpec(degree=12, taps=(12, 6, 4, 1), state=1) if deg == 12 else P.default_spec(deg)
    corr = P.Correlator(spec, cfg, n_r, device=dev)
    h = S.draw_channel(corr, 1, seed=m + l + nb)
    iq = S.simulate_frames(corr, h, 20.0, seed=7)
    taps, stats, link = corr.process_scored(iq, h)
    ref = O.process_frames(O.sequence_for_length(m), ocfg, O.iq_to_frames(iq[0].cpu().numpy()))[0]
    got = taps[0].cpu().numpy().astype(np.complex128)
    err = np.abs(got - ref) / np.abs(ref).max(axis=-1, keepdims=True)
    assert err.max() <= 1e-2
    mse_ref = float(np.mean(np.abs(ref - h[0].cpu().numpy()) ** 2))
    mse_gpu = stats[0, 1].item() / h[0].numel()
    assert abs(10 * math.log10(mse_gpu / mse_ref)) <= 0.1


def _grid():
    pts = []
    for m in (127, 255, 511, 1023, 2047, 4095):
        for l in (8, 16, 32, 64, 128, 256):
            for nb in (1, 2, 4, 8, 16, 32):
                if l <= m and nb <= m // l and m // nb >= l:
                    pts.append((m, l, nb))
    return pts


def test_sweep_grid_every_point(dev):
    """Every feasible point of the configs[4] grid (135 of 216), each against the oracle: same
    (M, L, N_b) geometry -- lag-row tiling, circulant, demux -- at 4 receive antennas and
    2 N_b + 1 transmitters (three batches, the last one a single-transmitter row prefix),
    one frame-set at 20 dB, per-link tolerance 1e-2."""
    pts = _grid()
    assert len(pts) == 135
    worst = 0.0
    for m, l, nb in pts:
        n_r, n_t = 4, 2 * nb + 1
        cfg = P.PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
        ocfg = O.Config(m=m, c=l, n_t=n_t, n_batch=nb, l=l, n_r=n_r)
        deg = (m + 1).bit_length() - 1
        spec = P.LfsrSpec(degree=12, taps=(12, 6, 4, 1), state=1) if deg == 12 else P.default_spec(deg)
        corr = P.Correlator(spec, cfg, n_r, device=dev)
        h = S.draw_channel(corr, 1, seed=m * 7 + l * 3 + nb)
        iq = S.simulate_frames(corr, h, 20.0, seed=11)
        taps, _ = corr.process(iq)
        ref = O.process_frames(O.sequence_for_length(m), ocfg, O.iq_to_frames(iq[0].cpu().numpy()))[0]
        got = taps[0].cpu().numpy().astype(np.complex128)
        err = float((np.abs(got - ref) / np.abs(ref).max(axis=-1, keepdims=True)).max())
        assert err <= 1e-2, (m, l, nb, err)
        worst = max(worst, err)
        del corr, h, iq, taps
    print(f"135 grid points, worst per-link error {worst:.2e}")
