"""IQ file format + ingest against files written by the real reference.

Mirrors the reference's tests/test_iqfile.py (round trips, header validation, error
classes) and pins the byte layout on tests/golden/ref_frames.iq (reference writer).
"""

import os
import struct

import numpy as np
import pytest
import torch

from paper_2206_05506_b200 import iqfile as IQ
from paper_2206_05506_b200.errors import (BadMagicError, DimensionMismatchError, InvalidConfigError,
                                          TruncatedFileError, VersionMismatchError)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RAW = open(os.path.join(GOLD, "ref_frames.iq"), "rb").read()
NPZ = np.load(os.path.join(GOLD, "ref_frames.npz"))


def make_frames(n_r=2, p=10, l=3, count=2, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        s = rng.standard_normal((n_r, p + l - 1)) + 1j * rng.standard_normal((n_r, p + l - 1))
        out.append(s.real.astype(np.float32).astype(np.float64) + 1j * s.imag.astype(np.float32).astype(np.float64))
    return out


def make_header(n_r=2, p=10, l=3, count=2):
    return IQ.IqFileHeader(n_t=4, n_r=n_r, p=p, l=l, m=7, c=3, n_batch=1, frame_count=count, seed=5)


def test_reference_file_parses():
    header, frames = IQ.read_iq_bytes(RAW)
    n_t, n_r, m, l, c, nb, count = NPZ["geometry"]
    assert (header.n_t, header.n_r, header.m, header.l, header.c, header.n_batch, header.frame_count) == \
        (n_t, n_r, m, l, c, nb, count)
    assert header.p == c + m and header.seed == 100
    np.testing.assert_array_equal(np.stack(frames), NPZ["samples"])


def test_reference_bytes_reproduced():
    """Our writer emits the reference writer's bytes exactly."""
    header, frames = IQ.read_iq_bytes(RAW)
    assert IQ.write_iq_bytes(header, frames) == RAW


def test_values_round_trip(tmp_path):
    header, frames = make_header(), make_frames()
    path = tmp_path / "frames.iq"
    IQ.write_iq(path, header, frames)
    got_header, got = IQ.read_iq(path)
    assert got_header == header
    for a, b in zip(frames, got):
        np.testing.assert_array_equal(a, b)


def test_bytes_round_trip_is_bit_exact():
    raw = IQ.write_iq_bytes(make_header(), make_frames(seed=3))
    assert IQ.write_iq_bytes(*IQ.read_iq_bytes(raw)) == raw


def test_p_must_equal_c_plus_m():
    with pytest.raises(InvalidConfigError):
        IQ.IqFileHeader(n_t=1, n_r=1, p=9, l=3, m=7, c=3, n_batch=1, frame_count=0, seed=0)


def test_bad_magic():
    raw = IQ.write_iq_bytes(make_header(count=0), [])
    with pytest.raises(BadMagicError):
        IQ.read_iq_bytes(b"XXXX" + raw[4:])


def test_version_mismatch():
    raw = bytearray(IQ.write_iq_bytes(make_header(count=0), []))
    struct.pack_into("<H", raw, 4, 9)
    with pytest.raises(VersionMismatchError):
        IQ.read_iq_bytes(bytes(raw))


def test_truncated_header():
    with pytest.raises(TruncatedFileError):
        IQ.read_iq_bytes(b"PNCE\x01")


def test_truncated_payload_reports_offset():
    raw = IQ.write_iq_bytes(make_header(), make_frames())
    with pytest.raises(TruncatedFileError) as err:
        IQ.read_iq_bytes(raw[:-5])
    assert "byte" in str(err.value)


def test_write_validation():
    with pytest.raises(InvalidConfigError):
        IQ.write_iq_bytes(make_header(count=3), make_frames(count=2))
    with pytest.raises(InvalidConfigError):
        IQ.write_iq_bytes(make_header(), make_frames(n_r=3))


class _FakeCorr:
    """Geometry-only stand-in for Correlator (load_iq needs no device)."""

    def __init__(self, n_t, n_r, m, l, nb):
        from paper_2206_05506_b200 import PilotConfig
        self.cfg = PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
        self.n_r = n_r

    def iq_shape(self, n):
        return (n, self.cfg.n_batches, self.n_r, self.cfg.samples_per_receiver, 2)


def test_load_iq_payload_in_place(tmp_path):
    path = tmp_path / "ref.iq"
    path.write_bytes(RAW)
    n_t, n_r, m, l, c, nb, count = (int(v) for v in NPZ["geometry"])
    corr = _FakeCorr(n_t, n_r, m, l, nb)
    host = IQ.load_iq(path, corr, pin=False)
    assert tuple(host.shape) == corr.iq_shape(count // corr.cfg.n_batches)
    s = NPZ["samples"].reshape(host.shape[:-1])
    assert np.array_equal(host[..., 0].numpy(), s.real.astype(np.float32))
    assert np.array_equal(host[..., 1].numpy(), s.imag.astype(np.float32))
    with pytest.raises(DimensionMismatchError):
        IQ.load_iq(path, _FakeCorr(n_t, n_r, m, l, 1), pin=False)     # other batching
    (tmp_path / "cut.iq").write_bytes(RAW[:-8])
    with pytest.raises(TruncatedFileError):
        IQ.load_iq(tmp_path / "cut.iq", corr, pin=False)


@pytest.mark.gpu
def test_estimate_file_matches_device_path(tmp_path):
    """IQ file -> pinned chunks -> HBM -> taps == the resident-input path, bit for bit, and
    within the north-star tolerance of the reference's own reference64 estimates."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2206_05506_b200 as P
    dev = torch.device("cuda:0")
    path = tmp_path / "ref.iq"
    path.write_bytes(RAW)
    n_t, n_r, m, l, c, nb, count = (int(v) for v in NPZ["geometry"])
    cfg = P.PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(P.default_spec(7), cfg, n_r, device=dev)
    taps_file = IQ.estimate_file(path, corr, chunk_sets=2)               # 3 sets: chunks 2 + 1
    iq = IQ.load_iq(path, corr).to(dev)
    taps_dev, _ = corr.process(iq)
    assert torch.equal(taps_file, taps_dev.cpu())
    ref = NPZ["est_ref64"]
    err = np.abs(taps_file.numpy() - ref) / np.abs(ref).max(axis=-1, keepdims=True)
    assert err.max() <= 1e-2
