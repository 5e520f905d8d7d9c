"""The reference seam on the device: process_frames / correlate_rows with the
reference's BackendConfig (halfprec.py:29-55), saturation accounting in the reference's unit
(experiments.py:201-205), device/stream checks and the no-allocation-per-launch contract."""

import numpy as np
import pytest
import torch

import paper_2206_05506_b200 as P
from oracle import pnce_oracle as O
from paper_2206_05506_b200.backend import BackendConfig

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def cfg2_sets(n_sets, snr=10.0):
    cfg = P.PilotConfig(m=255, c=32, n_t=16, n_batch=4, l=32, f_s=10e6)
    ocfg = O.Config(m=255, c=32, n_t=16, n_batch=4, l=32, n_r=16)
    chips = O.sequence_for_length(255)
    iqs, truths = [], []
    for it in range(n_sets):
        cs, ns = O.derive_seeds(0, 255, 4, 32, 0, it)
        truth, frames = O.simulate_frame(chips, ocfg, 32, snr, cs, ns)
        iqs.append(O.frames_to_iq(frames))
        truths.append(truth)
    return cfg, ocfg, chips, np.stack(iqs), np.stack(truths)


def link_err(got, ref):
    scale = np.abs(ref).max(axis=-1, keepdims=True)
    scale[scale == 0] = 1.0
    return float((np.abs(got - ref) / scale).max())


def test_backendconfig_routes(dev):
    """reference64/32 -> the fused fp16 path (bit-identical to Correlator.process); tensor16 ->
    the tensor16 mode with the config's chunk_len / accumulator (bit-identical to
    Correlator.process_tensor16, and within 1e-2 of the oracle's tensor16 emulation)."""
    cfg, ocfg, chips, iq, truth = cfg2_sets(1)
    seq = P.sequence_for_length(255, dev)
    plan = P.build_batch_plan(cfg)
    corr = P.correlator_rows_for_plan(seq, plan, cfg, 16)
    x = torch.from_numpy(iq).to(dev)
    plain, _ = corr.process(x)
    for kind in ("reference64", "reference32"):
        est = P.process_frames(seq, cfg, plan, x[0], backend=BackendConfig(kind=kind), rows_per_batch=corr)
        assert est.backend == kind and est.saturations == 0
        assert torch.equal(est.taps, plain[0])
    for chunk, acc in ((128, "binary16"), (64, "binary32"), (None, "binary32")):
        bc = BackendConfig(kind="tensor16", chunk_len=chunk, accumulator=acc)
        est = P.process_frames(seq, cfg, plan, x[0], backend=bc, rows_per_batch=corr)
        want, _ = corr.process_tensor16(x, chunk_len=chunk, accumulator=acc)
        assert est.backend == "tensor16"
        assert torch.equal(est.taps, want[0])
        ref, sats, _ = O.process_frames(chips, ocfg, O.iq_to_frames(iq[0]), backend="tensor16",
                                        chunk_len=chunk, accumulator=acc)
        assert sats == est.saturations == 0
        assert link_err(est.taps.cpu().numpy().astype(np.complex128), ref) <= 1e-2
    # the reference's own class is duck-typed on kind / chunk_len / accumulator
    class RefLike:
        kind, tile, chunk_len, accumulator = "tensor16", 4, 128, "binary16"
    est = P.process_frames(seq, cfg, plan, x[0], backend=RefLike(), rows_per_batch=corr)
    want, _ = corr.process_tensor16(x, chunk_len=128, accumulator="binary16")
    assert torch.equal(est.taps, want[0])


def test_backendconfig_validation(dev):
    with pytest.raises(P.InvalidConfigError):
        BackendConfig(kind="reference128")
    with pytest.raises(P.InvalidConfigError):
        BackendConfig(kind="tensor16", chunk_len=6)
    with pytest.raises(P.InvalidConfigError):
        BackendConfig(accumulator="binary8")
    cfg, _, _, iq, _ = cfg2_sets(1)
    seq = P.sequence_for_length(255, dev)
    with pytest.raises(P.InvalidConfigError):    # multiple of 4, not of the 64-sample K-block
        P.process_frames(seq, cfg, P.build_batch_plan(cfg), torch.from_numpy(iq[0]).to(dev),
                         backend=BackendConfig(kind="tensor16", chunk_len=100))


def test_saturation_in_reference_unit(dev):
    """An input beyond the fp16 range saturates its (frame-set, batch): the batch's taps are
    zero, n_r * n_tx saturations are counted, the error sums and per-link MSE score those
    taps as zeros -- what the reference's process_frames does for a saturated batch
    (experiments.py:201-205; oracle tensor16 with the same input gives the same count)."""
    cfg, ocfg, chips, iq, truth = cfg2_sets(2)
    iq[1, 2, 5, 100, 0] = np.inf                  # frame-set 1, batch 2 (transmitters 8-11)
    iq[0, 0, 3, 60, 1] = 1e6                      # frame-set 0, batch 0: fp16 overflow -> inf
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    x = torch.from_numpy(iq).to(dev)
    h = torch.from_numpy(truth.astype(np.complex64)).to(dev)
    taps, stats, link = corr.process_scored(x, h)
    t, st, lk = taps.cpu().numpy(), stats.cpu().numpy(), link.cpu().numpy()
    assert st[1, 3] == 16 * 4 and st[0, 3] == 16 * 4
    assert (t[1, :, 8:12] == 0).all() and (t[0, :, 0:4] == 0).all()
    assert np.isfinite(t).all() and (st[:, 2] == 0).all()
    _, sats, _ = O.process_frames(chips, ocfg, O.iq_to_frames(iq[1]), backend="tensor16")
    assert sats == st[1, 3]
    # rescored sums == scoring the returned taps
    want = np.abs(t.astype(np.complex128) - truth).sum(axis=(1, 2, 3))
    assert np.allclose(st[:, 0], want, rtol=1e-5)
    assert np.allclose(lk[1, :, 8:12], (np.abs(truth[1, :, 8:12]) ** 2).mean(-1), rtol=1e-5)
    # untouched batches keep the fused result
    clean, _ = corr.process(torch.from_numpy(cfg2_sets(2)[3]).to(dev))
    assert np.array_equal(t[1, :, :8], clean.cpu().numpy()[1, :, :8])
    # process_frames reports the count on the CirEstimate
    seq = P.sequence_for_length(255, dev)
    est = P.process_frames(seq, cfg, P.build_batch_plan(cfg), x[1], rows_per_batch=corr, truth=h[1])
    assert est.saturations == 64 and np.isfinite(est.mse())


def test_correlate_rows_tensor16(dev):
    """Operator seam with BackendConfig(kind="tensor16") against the oracle's emulation."""
    chips = O.sequence_for_length(511)
    rows = O.lag_rows(chips, np.arange(64))
    rng = np.random.default_rng(3)
    y = rng.standard_normal((511, 8)) + 1j * rng.standard_normal((511, 8))
    got = P.correlate_rows(rows, y, backend=BackendConfig(kind="tensor16", chunk_len=128,
                                                          accumulator="binary16")).cpu().numpy()
    ref = O.correlate_rows(rows, y, "tensor16", 511, 128, "binary16")
    assert link_err(got.T.astype(np.complex128), ref.T) <= 1e-2
    with pytest.raises(P.SaturationDetectedError):
        P.correlate_rows(rows, y * 1e4, backend=BackendConfig(kind="tensor16", chunk_len=128,
                                                              accumulator="binary16"))


def test_foreign_device_tensors_rejected(dev):
    cfg, _, _, iq, truth = cfg2_sets(1)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    x = torch.from_numpy(iq).to(dev)
    with pytest.raises(P.DimensionMismatchError):
        corr.process(x, truth=torch.from_numpy(truth.astype(np.complex64)))     # host truth
    with pytest.raises(P.DimensionMismatchError):
        corr.process(x, out=torch.empty(corr.taps_shape(1), dtype=torch.complex64))
    if torch.cuda.device_count() > 1:
        other = torch.device("cuda:1")
        with pytest.raises(P.DimensionMismatchError):
            corr.process(x.to(other))
        # plans on two devices in one process (per-device kernel attributes)
        corr1 = P.Correlator(P.default_spec(8), cfg, 16, device=other)
        a, _ = corr.process(x)
        b, _ = corr1.process(x.to(other))
        assert torch.equal(a.cpu(), b.cpu())


def test_no_allocation_after_first_launch(dev):
    """Launch resources (A-stage scratch, saturation flags, tensor maps) belong to the plan and
    stream: after the first launch of each mode, repeated launches allocate nothing."""
    cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
    corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
    from paper_2206_05506_b200 import synth as S
    h = S.draw_channel(corr, 8, seed=1)
    iq = S.simulate_frames(corr, h, 10.0, seed=2)
    taps = torch.empty(corr.taps_shape(8), dtype=torch.complex64, device=dev)
    stats = torch.zeros((8, 4), dtype=torch.float64, device=dev)
    link = torch.zeros((8, 64, 64), dtype=torch.float32, device=dev)

    def all_modes():
        corr.process(iq, out=taps)
        corr.process_scored(iq, h, out=taps, stats=stats, link_mse=link)   # two groups: A-stage reuse
        corr.process_tensor16(iq, chunk_len=256, accumulator="binary16", out=taps, stats=stats)

    all_modes()
    torch.cuda.synchronize(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]
    for _ in range(20):
        all_modes()
    torch.cuda.synchronize(dev)
    assert torch.cuda.mem_get_info(dev)[0] == free0


def test_streams_share_a_plan(dev):
    """Reentrancy: the same plan launched on two streams at once gives identical taps."""
    cfg, _, _, iq, _ = cfg2_sets(3)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    x = torch.from_numpy(iq).to(dev).repeat(64, 1, 1, 1, 1)            # 192 frame-sets
    ref, _ = corr.process(x)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    outs = []
    torch.cuda.synchronize(dev)
    for s in (s1, s2):
        with torch.cuda.stream(s):
            st = torch.zeros((x.shape[0], 4), dtype=torch.float64, device=dev)
            outs.append(corr.process(x, stats=st)[0])
    torch.cuda.synchronize(dev)
    for o in outs:
        assert torch.equal(o, ref)


def test_graph_capture_replays_the_fused_launch(dev):
    """Correlator.capture: a CUDA graph of the fused launch gives the same taps on replay,
    also after the input buffer is refilled in place."""
    cfg, _, _, iq, _ = cfg2_sets(2)
    corr = P.Correlator(P.default_spec(8), cfg, 16, device=dev)
    x = torch.from_numpy(iq[:1]).to(dev).contiguous()
    graph, out = corr.capture(x)
    want0, _ = corr.process(x)
    graph.replay()
    torch.cuda.synchronize(dev)
    assert torch.equal(out, want0)
    x.copy_(torch.from_numpy(iq[1:2]))
    graph.replay()
    torch.cuda.synchronize(dev)
    want1, _ = corr.process(x)
    assert torch.equal(out, want1) and not torch.equal(want0, want1)


def test_gather_launch_writes_every_buffer(dev):
    """pnce_process_frames_gather in one process: a correlator for receivers [16, 40) of a
    64-receiver cfg3 writes its slice into the local CSI and into two more "peer" buffers
    (plain device pointers), rows r0.. of the full layout, bit-identical to the full
    correlator's rows; nothing else is touched.  Bad slices are rejected."""
    cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
    from paper_2206_05506_b200 import synth as S
    full = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
    h = S.draw_channel(full, 3, seed=5)
    iq = S.simulate_frames(full, h, 10.0, seed=6)
    ref, _ = full.process(iq)
    r0, r1 = 16, 40
    part = P.Correlator(P.default_spec(10), cfg, r1 - r0, device=dev)
    bufs = [torch.full((3, 64, 64, 64), 7 + 7j, dtype=torch.complex64, device=dev) for _ in range(3)]
    part.process_gather(iq[:, :, r0:r1].contiguous(), bufs[0], r0, peers=bufs[1:])
    torch.cuda.synchronize(dev)
    for b in bufs:
        assert torch.equal(b[:, r0:r1], ref[:, r0:r1])
        assert bool((b[:, :r0] == 7 + 7j).all()) and bool((b[:, r1:] == 7 + 7j).all())
    with pytest.raises(P.DimensionMismatchError):
        part.process_gather(iq[:, :, r0:r1].contiguous(), bufs[0], 48, peers=bufs[1:])   # rows 48..72 > 64
    with pytest.raises(P.InvalidConfigError):
        part.process_gather(iq[:, :, r0:r1].contiguous(), bufs[0], r0, peers=[bufs[1]] * 8)
