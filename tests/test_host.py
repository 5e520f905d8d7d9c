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


# ---------------------------------------------------------------- pn / pilot helpers (CPU tensors)
def _cpu_seq(degree):
    import torch

    from oracle import pnce_oracle as O
    from paper_2206_05506_b200 import PnSequence, default_spec
    taps = O.taps_for_degree(degree)
    return PnSequence(chips=torch.from_numpy(O.generate_mseq(degree, taps, 1)).float(), spec=default_spec(degree))


def test_circular_autocorrelation_two_valued():
    """test_pn.py: m-sequences have R(0) = 1 and R(lag) = -1/M elsewhere."""
    import pytest

    import paper_2206_05506_b200 as P
    seq = _cpu_seq(9)
    assert P.circular_autocorrelation(seq, 0) == 1.0
    for lag in (1, 2, 100, 510):
        assert abs(P.circular_autocorrelation(seq, lag) + 1 / 511) < 1e-12
    with pytest.raises(P.LagOutOfRangeError):
        P.circular_autocorrelation(seq, 511)


def test_circular_shift_and_pilot():
    """pn.py:149-160 delay semantics and pilots.py:103-110 against the oracle's build_pilot."""
    import numpy as np
    import pytest

    import paper_2206_05506_b200 as P
    from oracle import pnce_oracle as O
    seq = _cpu_seq(8)
    s = P.circular_shift(seq, 5)
    assert s.chips[5].item() == seq.chips[0].item()
    assert np.array_equal(P.circular_shift(s, 7).chips.numpy(), P.circular_shift(seq, 12).chips.numpy())
    with pytest.raises(P.ShiftOutOfRangeError):
        P.circular_shift(seq, 255)
    pf = P.build_pilot(seq, 63, 32, transmitter=1)
    assert len(pf) == 32 + 255 and pf.transmitter == 1 and pf.shift == 63
    assert np.array_equal(pf.samples.double().numpy(), O.build_pilot(seq.chips.double().numpy(), 63, 32))
    with pytest.raises(P.InvalidConfigError):
        P.build_pilot(seq, 0, 0)
