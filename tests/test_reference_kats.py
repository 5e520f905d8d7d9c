"""The reference's own host-side unit tests, ported onto this package's mirror of its API
(CPU, no GPU): pkg/tests/test_pn.py (LfsrSpec validation, circular autocorrelation and
shift), pkg/tests/test_pilots.py (max_batch, PilotConfig, shifts, build_pilot, batch plans,
propagation time), pkg/tests/test_metrics.py (mae) and the host parts of
pkg/tests/test_estimator.py (remove_cp, partial circulant / lag-window rows, batch
separation).  The m-sequences come from the
oracle's LFSR restatement (the device LFSR is pinned bit-exact to it in
tests/test_gpu_parity.py), so these run without a GPU."""

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from oracle import pnce_oracle as O


def seq(degree: int, state: int = 1) -> P.PnSequence:
    chips = O.generate_mseq(degree, O.taps_for_degree(degree), state)
    return P.PnSequence(chips=torch.from_numpy(chips).float(), spec=P.default_spec(degree, state))


@pytest.fixture(scope="module")
def seq511():
    return seq(9)


def cfg(m=511, c=64, n_t=16, n_batch=1, l=64, f_s=10e6):
    return P.PilotConfig(m=m, c=c, n_t=n_t, n_batch=n_batch, l=l, f_s=f_s)


# ------------------------------------------------------------------ test_pn.py
class TestLfsrSpec:  # test_pn.py:23-46
    def test_zero_state_rejected(self):
        with pytest.raises(P.ZeroStateError):
            P.LfsrSpec(degree=9, taps=(9, 5), state=0)

    def test_taps_must_include_degree(self):
        with pytest.raises(P.InvalidSpecError):
            P.LfsrSpec(degree=9, taps=(5, 3), state=1)

    def test_taps_out_of_range(self):
        with pytest.raises(P.InvalidSpecError):
            P.LfsrSpec(degree=9, taps=(10, 9), state=1)

    def test_degree_too_small(self):
        with pytest.raises(P.InvalidSpecError):
            P.LfsrSpec(degree=1, taps=(1,), state=1)

    def test_state_too_wide(self):
        with pytest.raises(P.InvalidSpecError):
            P.LfsrSpec(degree=3, taps=(3, 2), state=8)

    def test_unknown_degree_has_no_default(self):
        with pytest.raises(P.InvalidSpecError):
            P.default_spec(23)


class TestMseqProperties:  # test_pn.py:49-104 (sequence values from the oracle LFSR)
    def test_table_i_lengths(self):
        for degree, m in [(9, 511), (10, 1023), (11, 2047)]:
            s = seq(degree)
            assert s.m == m
            assert set(np.unique(s.numpy())) == {-1.0, 1.0}

    def test_degree2_sequence_and_autocorrelation(self):
        s = seq(2)
        np.testing.assert_array_equal(s.numpy(), [1.0, -1.0, -1.0])
        r = [P.circular_autocorrelation(s, n) for n in range(3)]
        np.testing.assert_allclose(r, [1.0, -1 / 3, -1 / 3], atol=1e-15)

    @pytest.mark.parametrize("degree", [9, 10, 11])
    def test_balance(self, degree):
        c = seq(degree).numpy()
        assert abs(int((c > 0).sum()) - int((c < 0).sum())) == 1

    @pytest.mark.parametrize("degree", [2, 3, 5, 9])
    def test_period_rerun_reproduces_sequence_twice(self, degree):
        spec = P.default_spec(degree)
        s = seq(degree)
        k, mask, state, bits = spec.degree, (1 << spec.degree) - 1, spec.state, []
        for _ in range(2 * s.m):
            bits.append((state >> (k - 1)) & 1)
            fb = (state & spec.tap_mask).bit_count() & 1
            state = ((state << 1) | fb) & mask
        chips = 1.0 - 2.0 * np.array(bits)
        np.testing.assert_array_equal(chips[: s.m], s.numpy())
        np.testing.assert_array_equal(chips[s.m:], s.numpy())


class TestCircularAutocorrelation:  # test_pn.py:107-125
    @pytest.mark.parametrize("degree", [9, 10, 11])
    def test_two_valued_everywhere(self, degree):
        s = seq(degree)
        m = s.m
        assert P.circular_autocorrelation(s, 0) == 1.0
        spot = np.array([P.circular_autocorrelation(s, n) for n in (1, 17, m // 2, m - 1)])
        np.testing.assert_allclose(spot, -1.0 / m, atol=1e-12, rtol=0)

    def test_lag_out_of_range(self, seq511):
        with pytest.raises(P.LagOutOfRangeError):
            P.circular_autocorrelation(seq511, 511)
        with pytest.raises(P.LagOutOfRangeError):
            P.circular_autocorrelation(seq511, -1)

    def test_constant_sequence(self):
        assert P.circular_autocorrelation(P.PnSequence(chips=torch.ones(3)), 1) == 1.0


class TestCircularShift:  # test_pn.py:128-154
    def test_identity(self, seq511):
        np.testing.assert_array_equal(P.circular_shift(seq511, 0).numpy(), seq511.numpy())

    def test_shift_out_of_range(self, seq511):
        with pytest.raises(P.ShiftOutOfRangeError):
            P.circular_shift(seq511, 511)
        with pytest.raises(P.ShiftOutOfRangeError):
            P.circular_shift(seq511, -3)

    def test_composition_adds_mod_m(self, seq511):
        rng = np.random.default_rng(7)
        for _ in range(20):
            a, b = (int(x) for x in rng.integers(0, seq511.m, size=2))
            lhs = P.circular_shift(P.circular_shift(seq511, a), b)
            rhs = P.circular_shift(seq511, (a + b) % seq511.m)
            np.testing.assert_array_equal(lhs.numpy(), rhs.numpy())

    def test_delay_semantics(self):
        s = seq(3)
        shifted = P.circular_shift(s, 2).numpy()
        for i in range(s.m):
            assert shifted[i] == s.numpy()[(i - 2) % s.m]


# ------------------------------------------------------------------ test_pilots.py
class TestMaxBatch:  # test_pilots.py:28-37
    @pytest.mark.parametrize("m,c,expected", [(2047, 128, 15), (511, 64, 7), (511, 511, 1)])
    def test_values(self, m, c, expected):
        assert P.max_batch(m, c) == expected

    def test_invalid(self):
        with pytest.raises(P.InvalidConfigError):
            P.max_batch(511, 0)
        with pytest.raises(P.InvalidConfigError):
            P.max_batch(511, 512)


class TestPilotConfig:  # test_pilots.py:40-50
    def test_rejects_cp_shorter_than_cir(self):
        with pytest.raises(P.InvalidConfigError):
            cfg(c=32, l=64)

    def test_rejects_oversized_batch(self):
        with pytest.raises(P.InvalidConfigError):
            cfg(m=511, c=64, n_batch=16)

    def test_p_is_c_plus_m(self):
        assert cfg().p == 575


class TestShiftForTransmitter:  # test_pilots.py:53-66
    def test_eq8_with_floor(self):
        c4 = cfg(m=2047, c=128, n_batch=4)
        assert P.shift_for_transmitter(5, c4) == 511
        assert P.shift_for_transmitter(0, c4) == 0

    def test_m511_nbatch2(self):
        assert P.shift_for_transmitter(3, cfg(m=511, c=64, n_batch=2)) == 255

    def test_out_of_range_transmitter(self):
        with pytest.raises(P.InvalidConfigError):
            P.shift_for_transmitter(16, cfg())


class TestBuildPilot:  # test_pilots.py:69-92
    def test_cp_is_copy_of_tail(self):
        frame = P.build_pilot(seq(3), shift=0, c=3)
        assert len(frame) == 10
        np.testing.assert_array_equal(frame.samples[:3].numpy(), frame.samples[-3:].numpy())

    def test_body_is_shifted_sequence(self, seq511):
        frame = P.build_pilot(seq511, shift=255, c=64)
        assert frame.shift == 255
        np.testing.assert_array_equal(frame.samples[:64].numpy(), frame.samples[-64:].numpy())
        np.testing.assert_array_equal(frame.samples[64:].numpy(), P.circular_shift(seq511, 255).numpy())

    def test_shift_at_m_rejected(self, seq511):
        with pytest.raises(P.ShiftOutOfRangeError):
            P.build_pilot(seq511, shift=511, c=64)

    def test_cp_removal_recovers_body(self, seq511):
        for shift in (0, 17, 510):
            frame = P.build_pilot(seq511, shift=shift, c=64)
            np.testing.assert_array_equal(P.remove_cp(frame.samples.numpy(), 64, 511),
                                          P.circular_shift(seq511, shift).numpy())


class TestBuildBatchPlan:  # test_pilots.py:95-130
    def test_sequential_degenerate(self):
        plan = P.build_batch_plan(cfg(n_t=16, n_batch=1))
        assert plan.n_batches == 16
        assert all(len(b) == 1 and b[0].shift == 0 for b in plan.batches)

    def test_four_by_four(self):
        plan = P.build_batch_plan(cfg(m=2047, c=128, n_t=16, n_batch=4))
        assert plan.n_batches == 4
        for batch in plan.batches:
            assert sorted(a.shift for a in batch) == [0, 511, 1022, 1533]
            shifts = [a.shift for a in batch]
            for i in range(len(shifts)):
                for j in range(i + 1, len(shifts)):
                    assert P.cyclic_separation(shifts[i], shifts[j], 2047) >= 128

    def test_every_transmitter_exactly_once(self):
        plan = P.build_batch_plan(cfg(m=2047, c=128, n_t=14, n_batch=4))
        seen = [a.transmitter for batch in plan.batches for a in batch]
        assert sorted(seen) == list(range(14))
        assert len(plan.batches[-1]) == 2

    def test_overfull_batch_rejected(self):
        with pytest.raises(P.InvalidConfigError):
            P.build_batch_plan(cfg(m=511, c=64, n_t=16, n_batch=16))

    @pytest.mark.parametrize("m,c,l", [(511, 64, 64), (1023, 128, 100), (2047, 128, 128)])
    def test_separation_property(self, m, c, l):
        for n_batch in range(1, P.max_batch(m, c) + 1):
            plan = P.build_batch_plan(cfg(m=m, c=c, l=l, n_t=2 * n_batch, n_batch=n_batch))
            for batch in plan.batches:
                shifts = [a.shift for a in batch]
                for i in range(len(shifts)):
                    for j in range(i + 1, len(shifts)):
                        assert P.cyclic_separation(shifts[i], shifts[j], m) >= l


class TestPropagationTime:  # test_pilots.py:133-155
    def test_sequential_16tx(self):
        assert P.propagation_time(cfg(m=511, c=64, n_t=16, n_batch=1)) == pytest.approx(0.92e-3)

    def test_batched_reduction(self):
        t1 = P.propagation_time(cfg(m=511, c=64, n_t=16, n_batch=1))
        assert P.propagation_time(cfg(m=511, c=64, n_t=16, n_batch=4)) == t1 / 4

    def test_unit_case(self):
        assert P.propagation_time(P.PilotConfig(m=511, c=64, n_t=1, n_batch=1, l=64, f_s=575.0)) == 1.0

    @pytest.mark.parametrize("n_batch", [1, 2, 4])
    def test_reduction_is_exact_for_every_config(self, n_batch):
        base = cfg(m=2047, c=128, n_t=16, n_batch=1)
        assert P.propagation_time(cfg(m=2047, c=128, n_t=16, n_batch=n_batch)) == P.propagation_time(base) / n_batch


# ------------------------------------------------------------------ test_metrics.py
class TestMae:  # test_metrics.py:16-34
    def test_identity_is_zero(self):
        rng = np.random.default_rng(1)
        taps = torch.from_numpy(rng.standard_normal((2, 3, 8)) + 1j * rng.standard_normal((2, 3, 8)))
        assert P.mae(taps, taps) == 0.0

    def test_constant_offset(self):
        truth = torch.zeros((1, 1, 4), dtype=torch.complex128)
        est = torch.full((1, 1, 4), 0.3 - 0.4j, dtype=torch.complex128)
        assert P.mae(truth, est) == pytest.approx(0.5)

    def test_hand_sum(self):
        truth = torch.tensor([[[1.0 + 0j, 0.0 + 0j]]])
        est = torch.tensor([[[1.0 + 0j, 0.5j]]])
        assert P.mae(truth, est) == pytest.approx(0.25)

    def test_dimension_mismatch(self):
        with pytest.raises(P.DimensionMismatchError):
            P.mae(torch.zeros((1, 1, 4)), torch.zeros((1, 1, 5)))

    def test_mse_hand_sum(self):  # (north-star MSE, same conventions)
        truth = torch.tensor([[[1.0 + 0j, 0.0 + 0j]]])
        est = torch.tensor([[[1.0 + 0j, 0.5j]]])
        assert P.mse(truth, est) == pytest.approx(0.125)


# ------------------------------------------------------------------ test_estimator.py (host parts)
class TestRemoveCp:  # test_estimator.py:34-47
    def test_slicing(self):
        np.testing.assert_array_equal(P.remove_cp(np.arange(10.0), 3, 7), np.arange(3.0, 10.0))

    def test_identity_channel_recovers_body(self, seq511):
        frame = P.build_pilot(seq511, 0, 64)
        np.testing.assert_array_equal(P.remove_cp(frame.samples.numpy(), 64, 511), seq511.numpy())

    def test_too_short(self):
        with pytest.raises(P.FrameTooShortError):
            P.remove_cp(np.zeros(9), 3, 7)


class TestPartialCirculant:  # test_estimator.py:50-74 (the lag-window rows K1 builds on the device)
    def test_full_circulant_times_self(self):
        s7 = seq(3)
        s = P.build_partial_circulant(s7, 7).double()
        corr = (s @ s7.chips.double() / 7).numpy()
        np.testing.assert_allclose(corr, [1] + [-1 / 7] * 6, atol=1e-15)

    def test_single_row_is_sequence(self, seq511):
        np.testing.assert_array_equal(P.build_partial_circulant(seq511, 1)[0].numpy(), seq511.numpy())

    def test_shape_and_entries(self, seq511):
        s = P.build_partial_circulant(seq511, 64)
        assert tuple(s.shape) == (64, 511)
        assert set(np.unique(s.numpy())) == {-1.0, 1.0}

    def test_rows_are_shifted_base_row(self, seq511):
        s = P.build_partial_circulant(seq511, 5).numpy()
        for i in range(5):
            np.testing.assert_array_equal(s[i], np.roll(s[0], i))

    def test_rows_out_of_range(self, seq511):
        with pytest.raises(P.RowsOutOfRangeError):
            P.build_partial_circulant(seq511, 0)
        with pytest.raises(P.RowsOutOfRangeError):
            P.build_partial_circulant(seq511, 512)

    def test_batched_rows_are_windows_of_the_full_circulant(self, seq511):
        # estimator.py:114-117: the stacked lag windows equal rows [s, s+L) of the circulant
        full = P.build_partial_circulant(seq511, 511).numpy()
        batch = [P.BatchAssignment(0, 0), P.BatchAssignment(1, 255)]
        rows = P.batched_lag_rows(seq511, batch, 64).numpy()
        np.testing.assert_array_equal(rows[:64], full[:64])
        np.testing.assert_array_equal(rows[64:], full[255:255 + 64])

    def test_separation_violation_rejected(self):
        with pytest.raises(P.PlanMismatchError):
            P.validate_batch_separation([P.BatchAssignment(0, 0), P.BatchAssignment(1, 32)], 511, 64)
