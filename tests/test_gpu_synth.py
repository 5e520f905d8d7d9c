"""Device input synthesis against the CPU oracle's restatement of
channel.py: noiseless frames are deterministic given the CIRs (compared sample by sample),
the channel law and the noise calibration are checked statistically (Philox streams)."""

import math
import os

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from paper_2206_05506_b200 import synth as S
from oracle import pnce_oracle as O

pytestmark = pytest.mark.gpu

LAYOUTS = {
    # name: (n_t, n_r, m, l, c, n_batch)
    "cfg2": (16, 16, 255, 32, 32, 4),
    "odd": (5, 3, 255, 20, 20, 5),
    "cfg3": (64, 8, 1023, 64, 64, 8),
    "c_gt_l": (4, 2, 127, 8, 16, 2),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def make(name, dev):
    n_t, n_r, m, l, c, nb = LAYOUTS[name]
    cfg = P.PilotConfig(m=m, c=c, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
    ocfg = O.Config(m=m, c=c, n_t=n_t, n_batch=nb, l=l, n_r=n_r)
    corr = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n_r, device=dev)
    return cfg, ocfg, corr


def oracle_frames(chips, ocfg, h):
    """channel.py:186-214 noiseless, with the given CIRs (F, n_r, n_t, L)."""
    out = []
    for hf in h:
        sets = []
        for batch in O.build_batch_plan(ocfg):
            pilots = [O.build_pilot(chips, s, ocfg.c) for _, s in batch]
            sets.append(O.apply_channel(pilots, hf, [t for t, _ in batch]))
        out.append(np.stack(sets))
    return np.stack(out)                                   # (F, n_batches, n_r, P+L-1) complex


@pytest.mark.parametrize("name", list(LAYOUTS))
def test_noiseless_frames_match_oracle(dev, name):
    cfg, ocfg, corr = make(name, dev)
    h = S.draw_channel(corr, 3, seed=7)
    iq = S.simulate_frames(corr, h, math.inf).cpu().numpy()
    got = iq[..., 0] + 1j * iq[..., 1]
    ref = oracle_frames(O.sequence_for_length(ocfg.m), ocfg, h.cpu().numpy().astype(np.complex128))
    assert got.shape == ref.shape
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 2e-6 * scale * math.sqrt(ocfg.n_batch * ocfg.l)


@pytest.mark.parametrize("l_nz", [None, 5])
def test_channel_law(dev, l_nz):
    cfg, ocfg, corr = make("cfg2", dev)
    h = S.draw_channel(corr, 64, l_nz=l_nz, seed=11).cpu().numpy()
    lnz = cfg.l if l_nz is None else l_nz
    amax = math.sqrt(1.0 / (cfg.n_t * math.sqrt(lnz)))
    a = np.abs(h)
    nz = a > 0
    assert (nz.sum(axis=-1) == lnz).all()                  # exactly L_nz distinct taps per link
    assert a.max() <= amax * (1 + 1e-6) and a[nz].min() > 0
    assert abs(a[nz].mean() / amax - 0.5) < 0.01           # uniform on (0, A_max]
    ph = np.angle(h[nz])
    assert abs(np.exp(1j * ph).mean()) < 0.02             # uniform phase
    if l_nz is not None:                                   # positions spread over all lags
        counts = nz.reshape(-1, cfg.l).sum(axis=0)
        assert counts.min() > 0.5 * counts.mean()
    # different seeds, different draws; same seed, same draw
    h2 = S.draw_channel(corr, 2, l_nz=l_nz, seed=11).cpu().numpy()
    assert np.array_equal(h2, h[:2])
    assert not np.array_equal(S.draw_channel(corr, 2, l_nz=l_nz, seed=12).cpu().numpy(), h[:2])


@pytest.mark.parametrize("snr_db", [0.0, 10.0, 30.0])
def test_noise_calibration(dev, snr_db):
    """sigma^2 = noise_reference_power / 10^(SNR/10) (channel.py:145-183), on every sample."""
    cfg, ocfg, corr = make("cfg2", dev)
    h = S.draw_channel(corr, 32, seed=3)
    clean = S.simulate_frames(corr, h, math.inf)
    noisy = S.simulate_frames(corr, h, snr_db, seed=5)
    n = (noisy - clean).double()
    npow = (n[..., 0] ** 2 + n[..., 1] ** 2).mean(dim=(2, 3))         # (F, n_batches)
    c = clean.double()
    body = c[..., cfg.c:cfg.c + cfg.m, :]
    ref = (body[..., 0] ** 2 + body[..., 1] ** 2).mean(dim=(2, 3)) / (cfg.n_batch * cfg.l)
    ratio = (npow / ref).mean().item() * 10 ** (snr_db / 10)
    assert abs(ratio - 1.0) < 0.02
    # I and Q independent, zero mean
    assert abs(n.mean().item()) < 0.01 * math.sqrt(npow.mean().item())


def test_estimation_on_device_frames(dev):
    """Noiseless device frames through the estimator == the oracle path on oracle frames
    with the same CIRs (within the north-star tolerance); noisy MSE sits on the oracle's
    cfg2 MSE-vs-SNR anchor (statistical, 0.5 dB)."""
    cfg, ocfg, corr = make("cfg2", dev)
    chips = O.sequence_for_length(ocfg.m)
    h = S.draw_channel(corr, 4, seed=21)
    taps, _ = corr.process(S.simulate_frames(corr, h, math.inf))
    ref = np.stack([O.process_frames(chips, ocfg, list(fs))[0]
                    for fs in oracle_frames(chips, ocfg, h.cpu().numpy().astype(np.complex128))])
    err = np.abs(taps.cpu().numpy() - ref) / np.abs(ref).max(axis=-1, keepdims=True)
    assert err.max() <= 1e-2
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    snrs, mse_ref = gold["curve_snr"], gold["curve_mse32"].mean(axis=1)   # reference64, 8 frame-sets each
    hh = S.draw_channel(corr, 256, seed=99)
    for snr, want in zip(snrs, mse_ref):
        _, stats, _ = corr.process_scored(S.simulate_frames(corr, hh, float(snr), seed=int(snr) + 1000), hh)
        mse = stats[:, 1].sum().item() / hh.numel()
        assert abs(10 * math.log10(mse / want)) < 0.5, (snr, mse, want)
