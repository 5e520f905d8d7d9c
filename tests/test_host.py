"""Host-side mirror of the reference interface (no GPU): configs, plans, errors."""

import pytest

import paper_2206_05506_b200 as P
from oracle import pnce_oracle as O


def test_pilot_config_validation():
    with pytest.raises(P.InvalidConfigError):
        P.PilotConfig(m=511, c=32, n_t=16, n_batch=1, l=64, f_s=1.0)    # C < L
    with pytest.raises(P.InvalidConfigError):
        P.PilotConfig(m=511, c=64, n_t=16, n_batch=16, l=64, f_s=1.0)   # floor(511/64)=7
    with pytest.raises(P.InvalidConfigError):
        P.PilotConfig(m=2047, c=128, n_t=128, n_batch=16, l=128, f_s=1.0)  # BASELINE cfg4 as stated
    assert P.PilotConfig(m=511, c=64, n_t=16, n_batch=1, l=64, f_s=10e6).p == 575


@pytest.mark.parametrize("m,c,l,n_t,nb", [(127, 16, 16, 4, 1), (255, 32, 32, 16, 4), (1023, 64, 64, 64, 8),
                                           (2047, 127, 127, 128, 16), (2047, 128, 128, 14, 4),
                                           (2047, 128, 128, 32, 15)])
def test_batch_plan_matches_oracle(m, c, l, n_t, nb):
    plan = P.build_batch_plan(P.PilotConfig(m=m, c=c, n_t=n_t, n_batch=nb, l=l, f_s=1.0))
    ref = O.build_batch_plan(O.Config(m=m, c=c, n_t=n_t, n_batch=nb, l=l, n_r=1))
    assert [[(a.transmitter, a.shift) for a in b] for b in plan.batches] == ref


def test_shift_and_propagation_kats():
    c4 = P.PilotConfig(m=2047, c=128, n_t=16, n_batch=4, l=128, f_s=10e6)
    assert P.shift_for_transmitter(5, c4) == 511
    with pytest.raises(P.InvalidConfigError):
        P.shift_for_transmitter(16, c4)
    t1 = P.propagation_time(P.PilotConfig(m=511, c=64, n_t=16, n_batch=1, l=64, f_s=10e6))
    t4 = P.propagation_time(P.PilotConfig(m=511, c=64, n_t=16, n_batch=4, l=64, f_s=10e6))
    assert t1 == pytest.approx(0.92e-3) and t4 == t1 / 4


def test_lfsr_spec_validation():
    with pytest.raises(P.ZeroStateError):
        P.LfsrSpec(degree=9, taps=(9, 5), state=0)
    with pytest.raises(P.InvalidSpecError):
        P.LfsrSpec(degree=9, taps=(5, 3), state=1)
    with pytest.raises(P.InvalidSpecError):
        P.default_spec(12)
    assert P.LfsrSpec(degree=10, taps=(10, 3)).tap_mask == (1 << 9) | (1 << 2)


def test_remove_cp_and_errors():
    import numpy as np
    assert list(P.remove_cp(np.arange(10.0), 3, 7)) == list(np.arange(3.0, 10.0))
    with pytest.raises(P.FrameTooShortError):
        P.remove_cp(np.zeros(9), 3, 7)
