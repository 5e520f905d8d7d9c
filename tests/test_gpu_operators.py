"""Operator-level seam (correlate_rows / estimate_sequential / estimate_batched,
pnce/estimator.py:50-140) on the tensor cores, following the reference's
tests/test_estimator.py (TestEstimateSequential / TestEstimateBatched) with the tensor16
precision bound where the reference64 tests demand 1e-12."""

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from oracle import pnce_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def seq511():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return P.generate_mseq(P.default_spec(9), torch.device("cuda:0"))


def chips(seq):
    return seq.numpy()


def test_own_body_gives_autocorrelation(seq511):
    est = P.estimate_sequential(chips(seq511).astype(complex), seq511, 4).cpu().numpy()
    np.testing.assert_allclose(est.real, [1, -1 / 511, -1 / 511, -1 / 511], atol=1e-7)
    np.testing.assert_allclose(est.imag, 0, atol=1e-12)


def test_delayed_body_peaks_at_delay(seq511):
    y = np.roll(chips(seq511), 2).astype(complex)
    est = P.estimate_sequential(y, seq511, 4).cpu().numpy()
    np.testing.assert_allclose(est.real, [-1 / 511, -1 / 511, 1, -1 / 511], atol=1e-7)


def test_zero_input_and_wrong_length(seq511):
    est = P.estimate_sequential(np.zeros(511, dtype=complex), seq511, 8).cpu().numpy()
    assert (est == 0).all()
    with pytest.raises(P.DimensionMismatchError):
        P.estimate_sequential(np.zeros(510, dtype=complex), seq511, 8)
    with pytest.raises(P.RowsOutOfRangeError):
        P.build_partial_circulant(seq511, 512)


def test_matches_fft_oracle(seq511):
    rng = np.random.default_rng(17)
    for _ in range(3):
        y = rng.standard_normal(511) + 1j * rng.standard_normal(511)
        est = P.estimate_sequential(y, seq511, 511).cpu().numpy()
        ora = O.oracle_circular_correlate(y, chips(seq511))
        assert np.abs(est - ora).max() <= 5e-3 * np.abs(ora).max()


def test_tensor16_bound_against_reference64(seq511):
    """test_estimator.py:123-134: < 5e-3 per lag on unit-power inputs."""
    rng = np.random.default_rng(31)
    rows = O.lag_rows(chips(seq511), np.arange(64))
    worst = 0.0
    for _ in range(10):
        y = rng.standard_normal(511) + 1j * rng.standard_normal(511)
        y /= np.sqrt(np.mean(np.abs(y) ** 2))
        e64 = O.correlate_rows(rows, y[:, None], "reference64", 511)[:, 0]
        e16 = P.estimate_sequential(y, seq511, 64).cpu().numpy()
        worst = max(worst, float(np.abs(e16 - e64).max()))
    assert worst < 5e-3


def test_columns_and_backends(seq511):
    """(M, cols) operands, fp16 and bf16, against reference64 (north-star 1e-2 per column)."""
    rng = np.random.default_rng(5)
    rows = O.lag_rows(chips(seq511), np.arange(100) * 3)
    y = rng.standard_normal((511, 7)) + 1j * rng.standard_normal((511, 7))
    ref = O.correlate_rows(rows, y, "reference64", 511)
    for backend in ("fp16", "bf16"):
        got = P.correlate_rows(rows, y, backend=backend).cpu().numpy()
        assert got.shape == (100, 7)
        assert (np.abs(got - ref).max(axis=0) <= 1e-2 * np.abs(ref).max(axis=0)).all()
    with pytest.raises(P.InvalidConfigError):
        P.correlate_rows(rows, y[:510])


def test_degenerate_batch_equals_sequential(seq511):
    rng = np.random.default_rng(37)
    y = rng.standard_normal(511) + 1j * rng.standard_normal(511)
    batched = P.estimate_batched(y, seq511, [P.BatchAssignment(0, 0)], 64)
    assert torch.equal(batched[0], P.estimate_sequential(y, seq511, 64))


def test_two_transmitters_demux(seq511):
    c = chips(seq511)
    y = (c + np.roll(np.roll(c, 255), 3)).astype(complex)      # Tx0 at delay 0, Tx1 (shift 255) at delay 3
    est = P.estimate_batched(y, seq511, [P.BatchAssignment(0, 0), P.BatchAssignment(1, 255)], 64)
    e0, e1 = est[0].cpu().numpy(), est[1].cpu().numpy()
    assert np.argmax(np.abs(e0)) == 0 and np.argmax(np.abs(e1)) == 3
    assert abs(e0[0].real - 1.0) <= 2 / 511 and abs(e1[3].real - 1.0) <= 2 / 511


def test_windows_match_full_correlation(seq511):
    rng = np.random.default_rng(41)
    y = rng.standard_normal(511) + 1j * rng.standard_normal(511)
    est = P.estimate_batched(y, seq511, [P.BatchAssignment(0, 0), P.BatchAssignment(1, 255)], 64)
    full = P.estimate_sequential(y, seq511, 511)
    assert torch.equal(est[0], full[:64])
    assert torch.equal(est[1], full[255:255 + 64])


def test_separation_violation_rejected(seq511):
    with pytest.raises(P.PlanMismatchError):
        P.estimate_batched(np.zeros(511, complex), seq511, [P.BatchAssignment(0, 0), P.BatchAssignment(1, 32)], 64)
    with pytest.raises(P.PlanMismatchError):
        P.estimate_batched(np.zeros(511, complex), seq511, [], 64)
