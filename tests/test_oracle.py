"""Pin the CPU oracle against golden vectors produced by the real reference.

These run on CPU (no GPU marker).  Golden vectors: tests/golden/make_golden.py.
"""

import hashlib
import math

import numpy as np
import pytest

from oracle import pnce_oracle as O

CONFIGS = {
    "cfg1": (4, 127, 16, 1),
    "cfg2": (16, 255, 32, 4),
    "cfg3": (64, 1023, 64, 8),
    "cfg4p": (128, 2047, 127, 16),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_of(name):
    n, m, l, nb = CONFIGS[name]
    return O.Config(m=m, c=l, n_t=n, n_batch=nb, l=l, n_r=n)


@pytest.mark.parametrize("degree", list(range(2, 13)))
def test_chips_match_reference(golden, degree):
    chips = O.generate_mseq(degree, O.taps_for_degree(degree), 1)
    assert np.array_equal(np.packbits(chips < 0), golden[f"chips_d{degree}"])
    assert chips.shape[0] == (1 << degree) - 1
    assert abs(int((chips > 0).sum()) - int((chips < 0).sum())) == 1


def test_chips_nondefault_state(golden):
    chips = O.generate_mseq(10, O.taps_for_degree(10), 77)
    assert np.array_equal(np.packbits(chips < 0), golden["chips_d10_state77"])


def test_degree2_kat():
    # test_pn.py:66-73
    assert np.array_equal(O.generate_mseq(2, (2, 1), 1), [1.0, -1.0, -1.0])


def test_non_primitive_rejected():
    # test_pn.py:61-64 (x^9 + x + 1 has period 73)
    with pytest.raises(O.OracleError):
        O.generate_mseq(9, (9, 1), 1)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_shifts_match_reference(golden, name):
    cfg = cfg_of(name)
    plan = O.build_batch_plan(cfg)
    nb = cfg.n_batch
    got = np.array([[s for _, s in b] + [-1] * (nb - len(b)) for b in plan])
    assert np.array_equal(got, golden[f"{name}_shifts"])


def test_shift_kats():
    # test_pilots.py:53-61
    c4 = O.Config(m=2047, c=128, n_t=16, n_batch=4, l=128, n_r=1)
    assert O.shift_for_transmitter(5, c4) == 511
    assert [s for _, s in O.build_batch_plan(c4)[0]] == [0, 511, 1022, 1533]
    assert O.shift_for_transmitter(3, O.Config(m=511, c=64, n_t=16, n_batch=2, l=64, n_r=1)) == 255


@pytest.mark.parametrize("name,it", [("cfg1", i) for i in range(6)] + [("cfg2", 0), ("cfg2", 1)])
def test_small_configs_bit_exact(golden, name, it):
    cfg = cfg_of(name)
    key = f"{name}_it{it}"
    cs, ns = (int(x) for x in golden[f"{key}_seeds"])
    chips = O.sequence_for_length(cfg.m)
    truth, frames = O.simulate_frame(chips, cfg, cfg.l, 10.0, cs, ns)
    iq = O.frames_to_iq(frames)
    assert sha(iq) == str(golden[f"{key}_iq_sha"])
    assert sha(truth) == str(golden[f"{key}_truth_sha"])
    assert np.array_equal(iq, golden[f"{key}_iq"])
    est, sat, _ = O.process_frames(chips, cfg, O.iq_to_frames(iq))
    assert sat == 0
    np.testing.assert_allclose(est, golden[f"{key}_est32"], rtol=0, atol=1e-13)
    assert O.mae(truth, est) == pytest.approx(float(golden[f"{key}_mae32"]), rel=1e-12)
    t16, _, _ = O.process_frames(chips, cfg, O.iq_to_frames(iq), backend="tensor16",
                                 chunk_len=128 if cfg.m == 127 else 256)
    np.testing.assert_allclose(t16, golden[f"{key}_est_t16"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["cfg3", "cfg4p"])
def test_large_configs_sampled(golden, name):
    cfg = cfg_of(name)
    key = f"{name}_it0"
    cs, ns = (int(x) for x in golden[f"{key}_seeds"])
    chips = O.sequence_for_length(cfg.m)
    truth, frames = O.simulate_frame(chips, cfg, cfg.l, 10.0, cs, ns)
    iq = O.frames_to_iq(frames)
    assert sha(iq) == str(golden[f"{key}_iq_sha"])
    assert sha(truth) == str(golden[f"{key}_truth_sha"])
    est, _, macs = O.process_frames(chips, cfg, O.iq_to_frames(iq))
    idx = golden[f"{key}_sample_idx"]
    np.testing.assert_allclose(est.reshape(-1)[idx], golden[f"{key}_sample_est32"], rtol=0, atol=1e-13)
    assert O.mae(truth, est) == pytest.approx(float(golden[f"{key}_mae32"]), rel=1e-12)
    assert O.mse(truth, est) == pytest.approx(float(golden[f"{key}_mse32"]), rel=1e-12)
    assert macs == cfg.n_r * cfg.n_t * cfg.l * cfg.m


def test_fft_oracle_agreement():
    # test_estimator.py:98-105 / acceptance criterion 2
    chips = O.sequence_for_length(511)
    rng = np.random.default_rng(17)
    y = rng.standard_normal(511) + 1j * rng.standard_normal(511)
    rows = O.lag_rows(chips, np.arange(511))
    est = O.correlate_rows(rows, y[:, None], "reference64", 511)[:, 0]
    ora = O.oracle_circular_correlate(y, chips)
    assert np.abs(est - ora).max() <= 1e-9 * np.abs(ora).max()


def test_own_body_autocorrelation():
    # test_estimator.py:78-81
    chips = O.sequence_for_length(511)
    est = O.correlate_rows(O.lag_rows(chips, np.arange(4)), chips.astype(complex)[:, None],
                           "reference64", 511)[:, 0]
    np.testing.assert_allclose(est.real, [1, -1 / 511, -1 / 511, -1 / 511], atol=1e-12)


def test_mae_kat():
    # test_metrics.py:27-30
    assert O.mae(np.array([[[1.0 + 0j, 0j]]]), np.array([[[1.0 + 0j, 0.5j]]])) == pytest.approx(0.25)


def test_snr_curve_anchor(golden):
    # cfg2 reference64 MAE/MSE-vs-SNR anchor, first two iterations per grid point
    cfg = cfg_of("cfg2")
    chips = O.sequence_for_length(cfg.m)
    for si, snr in enumerate(golden["curve_snr"]):
        for it in range(2):
            cs, ns = O.derive_seeds(0, cfg.m, cfg.n_batch, cfg.l, si, it)
            truth, frames = O.simulate_frame(chips, cfg, cfg.l, float(snr), cs, ns)
            est, _, _ = O.process_frames(chips, cfg, O.iq_to_frames(O.frames_to_iq(frames)))
            assert O.mae(truth, est) == pytest.approx(golden["curve_mae32"][si, it], rel=1e-12)
            assert O.mse(truth, est) == pytest.approx(golden["curve_mse32"][si, it], rel=1e-12)


def test_noiseless_cfg3(golden):
    cfg = cfg_of("cfg3")
    chips = O.sequence_for_length(cfg.m)
    cs = int(golden["cfg3_noiseless_seed"])
    truth, frames = O.simulate_frame(chips, cfg, cfg.l, math.inf, cs, 0)
    iq = O.frames_to_iq(frames)
    assert sha(iq) == str(golden["cfg3_noiseless_iq_sha"])
    est, _, _ = O.process_frames(chips, cfg, O.iq_to_frames(iq))
    assert O.mae(truth, est) == pytest.approx(float(golden["cfg3_noiseless_mae32"]), rel=1e-12)


# ------------------------------------------------------------------ tensor16 (f3)
def _t16():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "t16.npz"))


@pytest.mark.parametrize("case", ["b32", "b16", "sat"])
def test_oracle_tensor16_matches_reference(case):
    """halfprec.py binary32 / binary16 chunked accumulation, incl. saturation accounting,
    reproduced by the oracle on the reference's own inputs and estimates."""
    g = _t16()
    chunk, acc16 = (int(x) for x in g[f"{case}_cfg"])
    cfg = O.Config(m=255, c=32, n_t=16, n_batch=4, l=32, n_r=16)
    chips = O.sequence_for_length(255)
    for s in range(g[f"{case}_iq"].shape[0]):
        frames = O.iq_to_frames(g[f"{case}_iq"][s])
        taps, sats, _ = O.process_frames(chips, cfg, frames, backend="tensor16", chunk_len=chunk,
                                         accumulator="binary16" if acc16 else "binary32")
        assert sats == int(g[f"{case}_sat"][s])
        assert np.array_equal(taps, g[f"{case}_taps"][s])
