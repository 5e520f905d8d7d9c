"""The reference's tensor16 backend on real tensor cores against the
real reference's own estimates (tests/golden/t16.npz, written by make_t16_golden.py)."""

import os

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from paper_2206_05506_b200.errors import InvalidConfigError

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "t16.npz"))


@pytest.fixture(scope="module")
def corr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = P.PilotConfig(m=255, c=32, n_t=16, n_batch=4, l=32, f_s=10e6)
    return P.Correlator(P.default_spec(8), cfg, 16, device=torch.device("cuda:0"))


def link_err(got, ref):
    scale = np.abs(ref).max(axis=-1, keepdims=True)
    scale[scale == 0] = 1.0
    return float((np.abs(got - ref) / scale).max())


def run(corr, case):
    chunk, acc16 = (int(x) for x in G[f"{case}_cfg"])
    iq = torch.from_numpy(G[f"{case}_iq"]).to(corr.device)
    truth = torch.from_numpy(G[f"{case}_truth"].astype(np.complex64)).to(corr.device)
    taps, stats = corr.process_tensor16(iq, chunk_len=chunk, accumulator="binary16" if acc16 else "binary32",
                                        truth=truth)
    return taps.cpu().numpy().astype(np.complex128), stats.cpu().numpy()


def test_binary32_chunks(corr):
    got, stats = run(corr, "b32")
    assert link_err(got, G["b32_taps"]) <= 1e-5      # same partials to fp32 rounding
    assert (stats[:, 3] == 0).all()


def test_binary16_chunks(corr):
    got, stats = run(corr, "b16")
    err = link_err(got, G["b16_taps"])
    assert err <= 1e-2, err                          # binary16 rounding points differ (MMA vs 4-tile)
    assert (stats[:, 3] == 0).all()


def test_binary16_saturation(corr):
    """Batches 0 and 2 (scaled x3000) overflow binary16 in both implementations: counted as
    n_r * n_tx saturations each and scored as zero taps; batches 1 and 3 estimate normally."""
    got, stats = run(corr, "sat")
    ref = G["sat_taps"]
    assert (stats[:, 3] == G["sat_sat"]).all()
    sat_tx = np.r_[0:4, 8:12]
    assert (got[:, :, sat_tx, :] == 0).all()
    ok_tx = np.r_[4:8, 12:16]
    assert link_err(got[:, :, ok_tx, :], ref[:, :, ok_tx, :]) <= 1e-2
    # scoring includes the zeroed batches, like mae(truth, est) on the reference's estimate
    truth = G["sat_truth"]
    want = np.abs(ref - truth).sum(axis=(1, 2, 3))
    assert np.allclose(stats[:, 0], want, rtol=1e-3)


def test_single_chunk_equals_default_path(corr):
    """chunk_len=None, binary32: one partial x 1/M == the default fused path."""
    iq = torch.from_numpy(G["b32_iq"]).to(corr.device)
    t16, _ = corr.process_tensor16(iq, chunk_len=None)
    plain, _ = corr.process(iq)
    assert torch.equal(t16, plain)


def test_chunk_validation(corr):
    iq = torch.from_numpy(G["b32_iq"]).to(corr.device)
    with pytest.raises(InvalidConfigError):
        corr.process_tensor16(iq, chunk_len=100)     # not whole 64-sample K-blocks
    with pytest.raises(InvalidConfigError):
        corr.process_tensor16(iq, chunk_len=512)     # exceeds the padded length (256)
    with pytest.raises(InvalidConfigError):
        corr.process_tensor16(iq, accumulator="binary8")
