"""INTEGRATION.md's reference-side binding (integration/pnce_gpu.py) executed on the
reference's OWN objects: the unmodified `pnce` package installed into baseline/_ref by
tools/install_ref.sh (git-ignored; it travels to the GPU box with the repo snapshot).
The binding's process_frames_gpu must be a drop-in for pnce.experiments.process_frames:
same arguments, same CirEstimate, estimates within the north-star tolerance of the
reference's reference64 and of its tensor16 emulation, MAE within 0.1 dB."""

import math
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def pnce_mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "pnce")):
        pytest.skip("baseline/_ref not installed (tools/install_ref.sh)")
    sys.path.insert(0, REF)
    os.environ["PNCE_B200_LIB"] = os.path.join(ROOT, "paper_2206_05506_b200", "lib", "libpnce_b200.so")
    import pnce.channel as ch
    import pnce.experiments as ex
    import pnce.halfprec as hp
    import pnce.metrics as me
    import pnce.pilots as pi
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import pnce_gpu
    return ch, ex, hp, me, pi, pnce_gpu


def link_err(got, ref):
    scale = np.abs(ref).max(axis=-1, keepdims=True)
    scale[scale == 0] = 1.0
    return float((np.abs(got - ref) / scale).max())


@pytest.mark.parametrize("geom", [(4, 4, 127, 16, 1), (16, 16, 255, 32, 4), (64, 64, 1023, 64, 8)])
def test_binding_on_reference_objects(pnce_mods, geom):
    ch, ex, hp, me, pi, G = pnce_mods
    n_t, n_r, m, l, nb = geom
    cfg = pi.PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
    seq = ex.sequence_for_length(m)
    plan = pi.build_batch_plan(cfg)
    gp = G.GpuPlan(seq, cfg, n_r)
    for it in range(3):
        cs, ns = ex._derive_seeds(0, m, nb, l, 0, it)
        truth, frames = ch.simulate_frame(cfg, ch.ChannelSpec(l=l, l_nz=l, n_t=n_t, n_r=n_r, seed=cs),
                                          ch.SnrSpec(snr_db=10.0, noise_seed=ns), seq)
        ref_c, gpu_c = ex.WorkCounters(), ex.WorkCounters()
        ref = ex.process_frames(seq, cfg, plan, frames, hp.REFERENCE64, ref_c)
        got = G.process_frames_gpu(seq, cfg, plan, frames, hp.REFERENCE64, gpu_c, rows_per_batch=gp)
        assert type(got) is type(ref) and got.taps.shape == ref.taps.shape and got.taps.dtype == ref.taps.dtype
        assert (got.backend, got.norm, got.saturations) == (ref.backend, ref.norm, ref.saturations)
        assert (gpu_c.samples_moved, gpu_c.macs) == (ref_c.samples_moved, ref_c.macs)
        assert link_err(got.taps, ref.taps) <= 1e-2
        assert abs(10 * math.log10(me.mae(truth, got) / me.mae(truth, ref))) <= 0.1


def test_binding_tensor16_on_reference_objects(pnce_mods):
    """BackendConfig(kind="tensor16") through the binding vs the reference's own emulation,
    including its saturation count on an overflowing batch."""
    ch, ex, hp, me, pi, G = pnce_mods
    cfg = pi.PilotConfig(m=255, c=32, n_t=16, n_batch=4, l=32, f_s=10e6)
    seq = ex.sequence_for_length(255)
    plan = pi.build_batch_plan(cfg)
    cs, ns = ex._derive_seeds(0, 255, 4, 32, 0, 0)
    truth, frames = ch.simulate_frame(cfg, ch.ChannelSpec(l=32, l_nz=32, n_t=16, n_r=16, seed=cs),
                                      ch.SnrSpec(snr_db=10.0, noise_seed=ns), seq)
    for bc in (hp.BackendConfig(kind="tensor16", chunk_len=128, accumulator="binary32"),
               hp.BackendConfig(kind="tensor16", chunk_len=64, accumulator="binary16")):
        ref = ex.process_frames(seq, cfg, plan, frames, bc)
        got = G.process_frames_gpu(seq, cfg, plan, frames, bc)
        assert got.saturations == ref.saturations == 0
        assert link_err(got.taps, ref.taps) <= 1e-2
    # batch 1 scaled past the binary16 accumulator range: saturated in both, counted n_r * n_tx
    loud = [ch.ReceivedFrame(samples=f.samples * (3000.0 if i == 1 else 1.0), batch_index=f.batch_index)
            for i, f in enumerate(frames)]
    bc = hp.BackendConfig(kind="tensor16", chunk_len=256, accumulator="binary16")
    ref = ex.process_frames(seq, cfg, plan, loud, bc)
    got = G.process_frames_gpu(seq, cfg, plan, loud, bc)
    assert ref.saturations == got.saturations == 16 * 4
    assert (got.taps[:, 4:8] == 0).all() and (ref.taps[:, 4:8] == 0).all()
    assert link_err(np.delete(got.taps, np.s_[4:8], 1), np.delete(ref.taps, np.s_[4:8], 1)) <= 1e-2
