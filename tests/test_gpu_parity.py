"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (north star): per-tap error normalised per link,
    |h_gpu - h_ref64| <= 1e-2 * max_l |h_ref64[r, t, :]|,
with fp16/bf16 operands and fp32 accumulation; MSE-vs-SNR within 0.1 dB.
Integer work (LFSR chips, plan/demux indices, packing) is bit-exact.
"""

import math

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from oracle import pnce_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-2
CONFIGS = {
    "cfg1": (4, 127, 16, 1),
    "cfg2": (16, 255, 32, 4),
    "cfg3": (64, 1023, 64, 8),
    "cfg4p": (128, 2047, 127, 16),
}


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def make_cfg(n_t, m, l, nb, n_r=None, c=None):
    c = l if c is None else c
    return (P.PilotConfig(m=m, c=c, n_t=n_t, n_batch=nb, l=l, f_s=10e6),
            O.Config(m=m, c=c, n_t=n_t, n_batch=nb, l=l, n_r=n_r or n_t))


def sim_sets(ocfg, n_sets, snr=10.0, master=0, si=0, l_nz=None):
    chips = O.sequence_for_length(ocfg.m)
    iqs, truths = [], []
    for it in range(n_sets):
        cs, ns = O.derive_seeds(master, ocfg.m, ocfg.n_batch, ocfg.l, si, it)
        truth, frames = O.simulate_frame(chips, ocfg, l_nz or ocfg.l, snr, cs, ns)
        iqs.append(O.frames_to_iq(frames))
        truths.append(truth)
    return chips, np.stack(iqs), np.stack(truths)


def link_err(got, ref):
    scale = np.abs(ref).max(axis=-1, keepdims=True)
    return float((np.abs(got - ref) / np.maximum(scale, 1e-30)).max())


def oracle_est(chips, ocfg, iq):
    return np.stack([O.process_frames(chips, ocfg, O.iq_to_frames(iq[f]))[0] for f in range(iq.shape[0])])


# ------------------------------------------------------------------ a1: LFSR
@pytest.mark.parametrize("degree", list(range(2, 13)))
def test_device_lfsr_bit_exact(dev, degree):
    taps = O.taps_for_degree(degree)
    spec = P.LfsrSpec(degree=degree, taps=taps, state=1)
    seq = P.generate_mseq(spec, dev)
    assert np.array_equal(seq.numpy(), O.generate_mseq(degree, taps, 1))


def test_device_lfsr_state_and_rejection(dev):
    seq = P.generate_mseq(P.default_spec(10, state=77), dev)
    assert np.array_equal(seq.numpy(), O.generate_mseq(10, (10, 3), 77))
    with pytest.raises(P.NotMaximalLengthError):
        P.generate_mseq(P.LfsrSpec(degree=9, taps=(9, 1), state=1), dev)
    with pytest.raises(P.ZeroStateError):
        P.LfsrSpec(degree=9, taps=(9, 5), state=0)


# ------------------------------------------------------------------ a4: pack
@pytest.mark.parametrize("dtype,n_r,n_sets", [("fp16", 16, 2), ("bf16", 16, 2), ("fp16", 3, 1)])
def test_pack_bit_exact(dev, dtype, n_r, n_sets):
    cfg, ocfg = make_cfg(16, 255, 32, 4, n_r=n_r)
    chips, iq, _ = sim_sets(ocfg, n_sets)
    corr = P.Correlator(P.default_spec(8), cfg, n_r, dtype=dtype, device=dev)
    packed = corr.pack(torch.from_numpy(iq).to(dev)).cpu()
    body = iq[..., cfg.c:cfg.c + cfg.m, :]                     # (F, nb, n_r, M, 2)
    links = np.moveaxis(body, -1, -2).reshape(-1, 2, cfg.m)    # (link, part, M)
    pad = -len(links) % 8
    links = np.concatenate([links, np.zeros((pad, 2, cfg.m), links.dtype)])
    # 16-row blocks of 8 links: the 8 Re rows, then the 8 Im rows
    rows = links.reshape(-1, 8, 2, cfg.m).transpose(0, 2, 1, 3).reshape(-1, cfg.m)
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    want = torch.from_numpy(np.ascontiguousarray(rows)).to(tdt)
    assert packed.shape[0] == len(rows)
    assert torch.equal(packed[:, :cfg.m], want)
    assert torch.count_nonzero(packed[:, cfg.m:]) == 0


# ------------------------------------------------------------------ a5-a8: full path
@pytest.mark.parametrize("name,n_sets", [("cfg1", 6), ("cfg2", 2), ("cfg3", 2), ("cfg4p", 1)])
@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_process_frames_parity(dev, name, n_sets, dtype):
    n, m, l, nb = CONFIGS[name]
    cfg, ocfg = make_cfg(n, m, l, nb)
    chips, iq, truth = sim_sets(ocfg, n_sets)
    ref = oracle_est(chips, ocfg, iq)
    seq = P.sequence_for_length(m, dev)
    corr = P.correlator_rows_for_plan(seq, P.build_batch_plan(cfg), cfg, n, dtype=dtype)
    taps, stats = corr.process(torch.from_numpy(iq).to(dev),
                               truth=torch.from_numpy(truth.astype(np.complex64)).to(dev))
    got = taps.cpu().numpy().astype(np.complex128)
    err = link_err(got, ref)
    assert err <= TOL, f"{name}/{dtype}: per-link normalised error {err:.3e}"
    # fused scoring vs oracle metrics, per frame-set
    st = stats.cpu().numpy()
    for f in range(n_sets):
        n_taps = truth[f].size
        mse_gpu = st[f, 1] / n_taps
        mse_ref = O.mse(truth[f], ref[f])
        assert abs(10 * math.log10(mse_gpu / mse_ref)) <= 0.1
        assert st[f, 0] / n_taps == pytest.approx(O.mae(truth[f], ref[f]), rel=0.05)
        # the fused sums score exactly what was written to taps
        assert st[f, 1] / n_taps == pytest.approx(O.mse(truth[f], got[f]), rel=1e-4)
        assert st[f, 2] == 0


def test_reference_seam_host_frames(dev):
    """process_frames with the reference's host-side list-of-frames input."""
    cfg, ocfg = make_cfg(16, 255, 32, 4)
    chips = O.sequence_for_length(255)
    cs, ns = O.derive_seeds(0, 255, 4, 32, 0, 0)
    truth, frames = O.simulate_frame(chips, ocfg, 32, 10.0, cs, ns)
    seq = P.sequence_for_length(255, dev)
    counters = P.WorkCounters()
    est = P.process_frames(seq, cfg, P.build_batch_plan(cfg), frames, counters=counters)
    ref = O.process_frames(chips, ocfg, O.iq_to_frames(O.frames_to_iq(frames)))[0]
    assert est.taps.shape == (16, 16, 32)
    assert link_err(est.taps.cpu().numpy(), ref) <= TOL
    assert counters.macs == 16 * 16 * 32 * 255                   # test_acceptance.py:265
    assert counters.samples_moved == 16 * (255 + 32) * 4          # test_acceptance.py:264


def test_partial_last_batch(dev):
    """cfg4'' (L=C=128, N_b=15 at M=2047, n_t=32): last batch has 2 Tx -> row prefix of A."""
    cfg, ocfg = make_cfg(32, 2047, 128, 15, n_r=8)
    chips, iq, truth = sim_sets(ocfg, 1)
    ref = oracle_est(chips, ocfg, iq)
    corr = P.Correlator(P.default_spec(11), cfg, 8, device=dev)
    taps, _ = corr.process(torch.from_numpy(iq).to(dev))
    assert link_err(taps.cpu().numpy(), ref) <= TOL


def test_frames_are_independent(dev):
    """F frame-sets in one call == F single calls, bit for bit (shard concatenation)."""
    cfg, ocfg = make_cfg(16, 255, 32, 4)
    _, iq, _ = sim_sets(ocfg, 5)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    x = torch.from_numpy(iq).to(dev)
    whole, _ = corr.process(x)
    parts = torch.cat([corr.process(x[i:i + 1])[0] for i in range(5)])
    assert torch.equal(whole, parts)


def test_own_body_autocorrelation(dev):
    """test_estimator.py:78-88: own body -> [1, -1/M, ...]; delayed body peaks at the delay."""
    m, l = 511, 8
    cfg = P.PilotConfig(m=m, c=8, n_t=1, n_batch=1, l=l, f_s=1.0)
    chips = O.sequence_for_length(m)
    s = cfg.samples_per_receiver
    iq = np.zeros((1, 1, 2, s, 2), dtype=np.float32)
    iq[0, 0, 0, 8:8 + m, 0] = chips
    iq[0, 0, 1, 8:8 + m, 0] = np.roll(chips, 2)
    corr = P.Correlator(P.default_spec(9), cfg, 2, device=dev)
    taps = corr.process(torch.from_numpy(iq).to(dev))[0].cpu().numpy()[0]
    want0 = np.full(l, -1 / m); want0[0] = 1
    want1 = np.full(l, -1 / m); want1[2] = 1
    np.testing.assert_allclose(taps[0, 0].real, want0, atol=1e-6)
    np.testing.assert_allclose(taps[1, 0].real, want1, atol=1e-6)
    np.testing.assert_allclose(taps[..., :].imag, 0, atol=1e-7)


def test_zero_input_and_empty(dev):
    cfg, _ = make_cfg(16, 255, 32, 4)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    z = torch.zeros(corr.iq_shape(3), dtype=torch.float32, device=dev)
    taps, _ = corr.process(z)
    assert torch.count_nonzero(taps) == 0
    e, _ = corr.process(torch.zeros(corr.iq_shape(0), dtype=torch.float32, device=dev))
    assert e.shape[0] == 0


def test_errors_map_to_reference_classes(dev):
    cfg, _ = make_cfg(16, 255, 32, 4)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    with pytest.raises(P.FrameTooShortError):
        corr.process(torch.zeros((1, 4, 16, 200, 2), device=dev))
    with pytest.raises(P.DimensionMismatchError):
        corr.process(torch.zeros((1, 3, 16, 318, 2), device=dev))
    with pytest.raises(P.DimensionMismatchError):
        P.Correlator(P.default_spec(9), cfg, 16, device=dev)
    with pytest.raises(P.InvalidConfigError):
        P.PilotConfig(m=511, c=64, n_t=16, n_batch=16, l=64, f_s=1.0)


def test_nonfinite_counted_not_raised(dev):
    """experiments.py:201-205 counts saturation instead of aborting: inf input -> the batch
    (4 receivers x 1 transmitter) is zeroed and counted as n_r * n_tx = 4 saturations."""
    cfg, ocfg = make_cfg(4, 127, 16, 1)
    _, iq, truth = sim_sets(ocfg, 1)
    iq[0, 0, 0, 20, 0] = np.inf
    corr = P.Correlator(P.default_spec(7), cfg, 4, device=dev)
    taps, stats = corr.process(torch.from_numpy(iq).to(dev),
                               truth=torch.from_numpy(truth.astype(np.complex64)).to(dev))
    assert stats[0, 3].item() == 4 and stats[0, 2].item() == 0
    assert (taps[0, :, 0] == 0).all() and torch.isfinite(torch.view_as_real(taps)).all()


def test_snr_curve_within_01db(dev, golden):
    """MSE-vs-SNR identical to the reference64 anchor curve within 0.1 dB (cfg2, seed 0)."""
    n, m, l, nb = CONFIGS["cfg2"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    seq = P.sequence_for_length(m, dev)
    corr = P.Correlator(seq.spec, cfg, n, device=dev)
    iters = golden["curve_mse32"].shape[1]
    for si, snr in enumerate(golden["curve_snr"]):
        _, iq, truth = sim_sets(ocfg, iters, snr=float(snr), si=si)
        _, stats = corr.process(torch.from_numpy(iq).to(dev),
                                truth=torch.from_numpy(truth.astype(np.complex64)).to(dev))
        mse_gpu = float(stats[:, 1].sum().item()) / truth.size
        mse_ref = float(golden["curve_mse32"][si].mean())
        assert abs(10 * math.log10(mse_gpu / mse_ref)) <= 0.1, (snr, mse_gpu, mse_ref)
        mae_gpu = float(stats[:, 0].sum().item()) / truth.size
        assert mae_gpu == pytest.approx(float(golden["curve_mae32"][si].mean()), rel=0.02)


def test_noiseless_bound_at_scale(dev):
    """Size-independent property at cfg3 with 256 frame-sets: noiseless per-lag error is
    bounded by the batched sidelobe bound sum_{batch}|h| / M (test_acceptance.py:106-137)
    plus fp16 quantisation slack; spot frames match the oracle."""
    n, m, l, nb = CONFIGS["cfg3"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    chips, iq, truth = sim_sets(ocfg, 4, snr=math.inf)
    reps = 64
    x = torch.from_numpy(iq).to(dev).repeat(reps, 1, 1, 1, 1)
    corr = P.Correlator(P.default_spec(10), cfg, n, device=dev)
    taps, _ = corr.process(x)
    taps = taps.view(reps, 4, n, n, l)
    assert torch.equal(taps[0], taps[-1])                          # deterministic across copies
    h = torch.from_numpy(truth).to(dev)
    err = (taps[0].to(torch.complex128) - h).abs()
    hb = h.abs().sum(-1).view(4, n, n // nb, nb).sum(-1)           # per (f, r, batch)
    bound = hb.repeat_interleave(nb, dim=-1).unsqueeze(-1) / m
    slack = 2e-3 * h.abs().amax(-1, keepdim=True)
    assert bool((err <= bound + slack).all())
    ref = oracle_est(chips, ocfg, iq[:1])
    assert link_err(taps[0, :1].cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("mode", ["1", "2"])
def test_fused_variants_agree(dev, mode, monkeypatch):
    """Both fused K3 variants (LDG converters / TMA-staged converters) match the oracle and
    each other bit for bit (same quantisation, same MMA order)."""
    n, m, l, nb = CONFIGS["cfg3"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    chips, iq, _ = sim_sets(ocfg, 2)
    corr = P.Correlator(P.default_spec(10), cfg, n, device=dev)
    x = torch.from_numpy(iq).to(dev)
    monkeypatch.setenv("PNCE_TUNE_FUSED_MODE", mode)
    taps, _ = corr.process(x)
    monkeypatch.delenv("PNCE_TUNE_FUSED_MODE")
    ref_gpu, _ = corr.process(x)
    assert torch.equal(taps, ref_gpu)
    assert link_err(taps.cpu().numpy(), oracle_est(chips, ocfg, iq)) <= TOL


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_packed_variants_agree(dev, monkeypatch, name):
    """Packed operand through TMA (mode 0, 512-column group) == through LDG (mode 3,
    256-column double-buffered groups), bit for bit, and within tolerance of the oracle."""
    n, m, l, nb = CONFIGS[name]
    cfg, ocfg = make_cfg(n, m, l, nb)
    chips, iq, _ = sim_sets(ocfg, 2)
    deg = (m + 1).bit_length() - 1
    corr = P.Correlator(P.default_spec(deg), cfg, n, device=dev)
    packed = corr.pack(torch.from_numpy(iq).to(dev))
    via_tma, _ = corr.correlate(packed, 2)
    monkeypatch.setenv("PNCE_TUNE_PACKED_MODE", "3")
    via_ldg, _ = corr.correlate(packed, 2)
    monkeypatch.delenv("PNCE_TUNE_PACKED_MODE")
    assert torch.equal(via_tma, via_ldg)
    assert link_err(via_ldg.cpu().numpy(), oracle_est(chips, ocfg, iq)) <= TOL


LINK_CASES = [("cfg2", None), ("cfg3", None), ("cfg4p", None), ("odd_l", (5, 3, 255, 20, 20, 5)),
              ("l127", (16, 2, 1023, 127, 127, 8))]


@pytest.mark.parametrize("name,layout", LINK_CASES)
def test_link_mse_fused(dev, name, layout):
    """Per-link MSE from the fused epilogue (north star (4)) == mean_l |h_est - h|^2 of the
    written taps; frame sums agree with the per-link values; quad (L % 8 == 0) and per-lane
    (odd L) reductions both covered."""
    if layout is None:
        n, m, l, nb = CONFIGS[name]
        cfg, ocfg = make_cfg(n, m, l, nb)
        n_r = n
    else:
        n, n_r, m, l, c, nb = layout
        cfg, ocfg = make_cfg(n, m, l, nb, n_r=n_r, c=c)
    chips, iq, truth = sim_sets(ocfg, 2)
    deg = (m + 1).bit_length() - 1
    corr = P.Correlator(P.default_spec(deg), cfg, n_r, device=dev)
    h = torch.from_numpy(truth.astype(np.complex64)).to(dev)
    taps, stats, link = corr.process_scored(torch.from_numpy(iq).to(dev), h)
    e2 = (taps - h).abs().double() ** 2
    want = e2.mean(dim=-1)
    got = link.double()
    assert torch.allclose(got, want, rtol=1e-4, atol=1e-12)
    # frame sums: sum|e|^2 over the frame == L * sum of the per-link means
    assert torch.allclose(stats[:, 1], e2.sum(dim=(1, 2, 3)), rtol=1e-4)
    assert torch.allclose(stats[:, 1], got.sum(dim=(1, 2)) * cfg.l, rtol=1e-4)


@pytest.mark.parametrize("mode", ["1", "2"])
def test_scored_modes_agree(dev, monkeypatch, mode):
    """Scored drains of both converter modes (TMA-staged: 8 epilogue warps; LDG: 4) give
    the same taps bit for bit and the same sums to rounding."""
    n, m, l, nb = CONFIGS["cfg3"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    _, iq, truth = sim_sets(ocfg, 2)
    corr = P.Correlator(P.default_spec(10), cfg, n, device=dev)
    x = torch.from_numpy(iq).to(dev)
    h = torch.from_numpy(truth.astype(np.complex64)).to(dev)
    plain, _ = corr.process(x)
    monkeypatch.setenv("PNCE_TUNE_FUSED_MODE", mode)
    taps, stats, link = corr.process_scored(x, h)
    monkeypatch.delenv("PNCE_TUNE_FUSED_MODE")
    assert torch.equal(taps, plain)
    e2 = (taps - h).abs().double() ** 2
    assert torch.allclose(link.double(), e2.mean(dim=-1), rtol=1e-4, atol=1e-12)
    assert torch.allclose(stats[:, 0], (taps - h).abs().double().sum(dim=(1, 2, 3)), rtol=1e-4)


def test_link_mse_front_end(dev):
    """process_frames(truth=...) returns CirEstimate.link_mse; MSE curve helpers agree."""
    n, m, l, nb = CONFIGS["cfg2"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    chips, iq, truth = sim_sets(ocfg, 1)
    seq = P.sequence_for_length(m, dev)
    est = P.process_frames(seq, cfg, P.build_batch_plan(cfg), torch.from_numpy(iq[0]).to(dev), truth=truth[0])
    assert est.link_mse is not None and tuple(est.link_mse.shape) == (n, n)
    assert abs(float(est.link_mse.double().mean()) - est.mse()) <= 1e-4 * est.mse()


def test_odd_row_stride(dev):
    """C + L odd -> odd samples per row (8-byte aligned rows): exercises the LDG path."""
    cfg, ocfg = make_cfg(16, 255, 32, 4, c=33)
    assert cfg.samples_per_receiver % 2 == 1
    chips, iq, _ = sim_sets(ocfg, 3)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    taps, _ = corr.process(torch.from_numpy(iq).to(dev))
    assert link_err(taps.cpu().numpy(), oracle_est(chips, ocfg, iq)) <= TOL


def test_packed_path_matches_fused(dev):
    """K2 (pack) + K3 on the packed operand == the fused kernel, bit for bit."""
    n, m, l, nb = CONFIGS["cfg4p"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    _, iq, _ = sim_sets(ocfg, 1)
    corr = P.Correlator(P.default_spec(11), cfg, n, device=dev)
    x = torch.from_numpy(iq).to(dev)
    fused, _ = corr.process(x)
    packed, _ = corr.correlate(corr.pack(x), 1)
    assert torch.equal(fused, packed)


# Lag-layout coverage of the resident Hankel-table circulant: window pairs (odd/even N_b,
# L not a multiple of 8), chunked long windows (L > 128), a single window, and the
# contiguous-lag case (delta == L).
LAYOUTS = [
    # (n_t, n_r, m, l, c, n_batch)
    (5, 3, 255, 20, 20, 5),      # pair mode, odd N_b, L % 8 != 0
    (6, 4, 511, 64, 64, 3),      # pair mode, odd N_b
    (4, 2, 1023, 200, 200, 2),   # chunk mode, separate windows, L > 128
    (3, 2, 511, 128, 128, 1),    # single window
    (4, 2, 127, 8, 8, 4),        # pair mode, tiny windows
    (16, 2, 1023, 127, 127, 8),  # contiguous lags (delta == L)
    (8, 2, 2047, 256, 256, 7),   # chunk mode, several long windows
]


@pytest.mark.parametrize("n_t,n_r,m,l,c,nb", LAYOUTS)
def test_lag_layouts(dev, n_t, n_r, m, l, c, nb):
    cfg, ocfg = make_cfg(n_t, m, l, nb, n_r=n_r, c=c)
    chips, iq, _ = sim_sets(ocfg, 2)
    deg = (m + 1).bit_length() - 1
    corr = P.Correlator(P.default_spec(deg), cfg, n_r, device=dev)
    x = torch.from_numpy(iq).to(dev)
    taps, _ = corr.process(x)
    ref = oracle_est(chips, ocfg, iq)
    assert link_err(taps.cpu().numpy(), ref) <= TOL
    packed, _ = corr.correlate(corr.pack(x), 2)
    assert torch.equal(taps, packed)


def test_unaligned_buffers(dev):
    """8-byte (not 16-byte) aligned IQ and taps buffers: the LDG converter path and the
    scalar-store epilogue path give the same estimates bit for bit."""
    n, m, l, nb = CONFIGS["cfg2"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    _, iq, truth = sim_sets(ocfg, 2)
    corr = P.Correlator(P.default_spec(8), cfg, n, device=dev)
    x = torch.from_numpy(iq).to(dev)
    want, _ = corr.process(x)
    xb = torch.empty(x.numel() + 2, dtype=torch.float32, device=dev)
    xu = xb[2:].view(x.shape)                                   # 8-byte offset
    xu.copy_(x)
    assert xu.data_ptr() % 16 == 8
    tb = torch.empty(want.numel() + 1, dtype=torch.complex64, device=dev)
    tu = tb[1:].view(want.shape)                                # 8-byte offset
    assert tu.data_ptr() % 16 == 8
    got, _ = corr.process(xu, out=tu)
    assert torch.equal(got, want)
    h = torch.from_numpy(truth.astype(np.complex64)).to(dev)
    got2, st2, l2 = corr.process_scored(xu, h, out=tu)
    _, st, lk = corr.process_scored(x, h)
    assert torch.equal(got2, want)
    assert torch.allclose(st2, st, rtol=1e-6) and torch.allclose(l2, lk, rtol=1e-6)


@pytest.mark.parametrize("chunk", [2, 8])
@pytest.mark.parametrize("bodies_only", [True, False])
def test_process_host(dev, bodies_only, chunk):
    """Pinned host IQ -> (pitched body-only DMA | full rows) -> kernel -> pinned host taps,
    chunked and double-buffered (chunk 2) or one in-order stage (chunk 8 >= 5 frame-sets):
    equal to the resident-input path bit for bit."""
    n, m, l, nb = CONFIGS["cfg2"]
    cfg, ocfg = make_cfg(n, m, l, nb)
    _, iq, _ = sim_sets(ocfg, 5)
    corr = P.Correlator(P.default_spec(8), cfg, n, device=dev)
    want, _ = corr.process(torch.from_numpy(iq).to(dev))
    host = torch.from_numpy(iq).pin_memory()
    out = torch.empty(corr.taps_shape(5), dtype=torch.complex64).pin_memory()
    corr.process_host(host, out, chunk=chunk, bodies_only=bodies_only)
    torch.cuda.synchronize()
    assert torch.equal(out, want.cpu())
    if chunk == 8:  # the single-stage path after a double-buffered call on the same correlator
        out2 = torch.zeros_like(out).pin_memory()
        corr.process_host(host, out2, chunk=2, bodies_only=bodies_only)
        corr.process_host(host[:1], out2[:1], chunk=8, bodies_only=bodies_only)
        torch.cuda.synchronize()
        assert torch.equal(out2, want.cpu())
