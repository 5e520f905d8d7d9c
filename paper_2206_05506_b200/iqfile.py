"""IQ frame files, host format and device ingest.

The byte layout is the reference's versioned format (pnce/iqfile.py:1-16):

    magic "PNCE" | version u16 | n_t, n_r, p, l, m, c, n_batch, frame_count u32 | seed u64
    payload: frame_count frames x n_r receivers x (p + l - 1) samples x (I, Q) float32

The host functions mirror the reference API (`IqFileHeader`, `write_iq_bytes`,
`read_iq_bytes`, `write_iq`, `read_iq`, same validation and error classes).  The
payload is exactly the device IQ layout of `Correlator` ((F, n_batches, n_r,
samples, 2) float32 with one frame-set = n_batches consecutive frames), so the device
ingest reads it straight into pinned host memory (`readinto`, no parsing or
widening) and streams it through `Correlator.process_host` in chunks: disk -> pinned
-> HBM copies overlap the kernel of the previous chunk.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from .errors import (BadMagicError, DimensionMismatchError, InvalidConfigError, TruncatedFileError,
                     VersionMismatchError)

MAGIC = b"PNCE"
VERSION = 1
_HEADER = struct.Struct("<4sH8IQ")   # 46 bytes
HEADER_BYTES = _HEADER.size


@dataclass(frozen=True)
class IqFileHeader:
    """iqfile.py:34-72: frame geometry + provenance seed."""

    n_t: int
    n_r: int
    p: int
    l: int
    m: int
    c: int
    n_batch: int
    frame_count: int
    seed: int
    version: int = VERSION

    def __post_init__(self):
        if self.p != self.c + self.m:
            raise InvalidConfigError(f"P={self.p} must equal C+M={self.c + self.m}")
        if self.version != VERSION:
            raise VersionMismatchError(f"unsupported version {self.version}")

    @property
    def samples_per_receiver(self) -> int:
        return self.p + self.l - 1

    @property
    def frame_bytes(self) -> int:
        return self.n_r * self.samples_per_receiver * 8

    def pack(self) -> bytes:
        return _HEADER.pack(MAGIC, self.version, self.n_t, self.n_r, self.p, self.l, self.m, self.c,
                            self.n_batch, self.frame_count, self.seed)


def _frame_samples(frame) -> np.ndarray:
    return np.asarray(getattr(frame, "samples", frame))


def write_iq_bytes(header: IqFileHeader, frames: Sequence) -> bytes:
    """iqfile.py:75-91.  ``frames``: (n_r, p + l - 1) complex arrays or objects with .samples."""
    if len(frames) != header.frame_count:
        raise InvalidConfigError(f"header declares {header.frame_count} frames, got {len(frames)}")
    shape = (header.n_r, header.samples_per_receiver)
    out = bytearray(header.pack())
    for frame in frames:
        s = _frame_samples(frame)
        if s.shape != shape:
            raise InvalidConfigError(f"frame shape {s.shape} != {shape}")
        iq = np.empty(shape + (2,), dtype="<f4")
        iq[..., 0] = s.real.astype(np.float32)
        iq[..., 1] = s.imag.astype(np.float32)
        out += iq.tobytes()
    return bytes(out)


def parse_header(raw) -> IqFileHeader:
    """Header validation of iqfile.py:94-107."""
    if len(raw) < HEADER_BYTES:
        raise TruncatedFileError(f"file ends at byte {len(raw)}, header needs {HEADER_BYTES} bytes")
    magic, version, n_t, n_r, p, l, m, c, n_batch, frame_count, seed = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise BadMagicError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise VersionMismatchError(f"unsupported version {version}")
    return IqFileHeader(n_t=n_t, n_r=n_r, p=p, l=l, m=m, c=c, n_batch=n_batch,
                        frame_count=frame_count, seed=seed)


def read_iq_bytes(raw: bytes) -> tuple[IqFileHeader, list[np.ndarray]]:
    """iqfile.py:94-122: frames widened to complex128 (byte-exact round trips)."""
    header = parse_header(raw)
    fb = header.frame_bytes
    frames = []
    for bi in range(header.frame_count):
        off = HEADER_BYTES + bi * fb
        end = off + fb
        if len(raw) < end:
            raise TruncatedFileError(f"file ends at byte {len(raw)}, frame {bi} needs bytes [{off}, {end})")
        iq = np.frombuffer(raw, dtype="<f4", count=fb // 4, offset=off).reshape(
            header.n_r, header.samples_per_receiver, 2)
        frames.append(iq[..., 0].astype(np.float64) + 1j * iq[..., 1].astype(np.float64))
    return header, frames


def write_iq(path, header: IqFileHeader, frames: Sequence) -> None:
    with open(path, "wb") as fh:
        fh.write(write_iq_bytes(header, frames))


def read_iq(path) -> tuple[IqFileHeader, list[np.ndarray]]:
    with open(path, "rb") as fh:
        return read_iq_bytes(fh.read())


# ---------------------------------------------------------------- device ingest
def read_header(path) -> IqFileHeader:
    with open(path, "rb") as fh:
        return parse_header(fh.read(HEADER_BYTES))


def _check_geometry(header: IqFileHeader, corr) -> int:
    cfg = corr.cfg
    if (header.n_t, header.n_r, header.m, header.c, header.l, header.n_batch) != \
            (cfg.n_t, corr.n_r, cfg.m, cfg.c, cfg.l, cfg.n_batch):
        raise DimensionMismatchError(f"file geometry {header} does not match the correlator")
    if header.frame_count % cfg.n_batches:
        raise DimensionMismatchError(
            f"{header.frame_count} frames is not a whole number of {cfg.n_batches}-batch frame-sets")
    return header.frame_count // cfg.n_batches


_POOL = None
_READ_THREADS = max(1, min(16, (os.cpu_count() or 1)))
_PIECE = 8 << 20          # upper bound; a read is split so every reader thread gets a piece
_MIN_PIECE = 1 << 20


def _pread_into(fd: int, view: memoryview, offset: int) -> None:
    done = 0
    while done < len(view):
        n = os.preadv(fd, [view[done:]], offset + done)
        if n <= 0:
            raise TruncatedFileError(f"file ends at byte {offset + done}, payload needs byte {offset + len(view)}")
        done += n


def _parallel_read(fd: int, view: memoryview, offset: int) -> None:
    """Page-cache/NVMe -> pinned memory with several threads (a single memcpy-bound reader
    tops out near 6-7 GB/s; preadv releases the GIL)."""
    global _POOL
    piece = min(_PIECE, max(_MIN_PIECE, -(-len(view) // _READ_THREADS)))
    piece = -(-piece // 4096) * 4096
    pieces = [(s, min(len(view), s + piece)) for s in range(0, len(view), piece)]
    if len(pieces) <= 1 or _READ_THREADS == 1:
        _pread_into(fd, view, offset)
        return
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=_READ_THREADS, thread_name_prefix="pnce-iq")
    futs = [_POOL.submit(_pread_into, fd, view[a:b], offset + a) for a, b in pieces]
    for f in futs:
        f.result()


def load_iq(path, corr, pin: bool = True) -> torch.Tensor:
    """Whole payload -> pinned host float32 (F, n_batches, n_r, samples, 2), read in place."""
    with open(path, "rb") as fh:
        header = parse_header(fh.read(HEADER_BYTES))
        n_sets = _check_geometry(header, corr)
        host = torch.empty(corr.iq_shape(n_sets), dtype=torch.float32, pin_memory=pin)
        _parallel_read(fh.fileno(), memoryview(host.numpy()).cast("B"), HEADER_BYTES)
    return host


def estimate_file(path, corr, chunk_sets: int = 16, taps_host: torch.Tensor | None = None) -> torch.Tensor:
    """IQ file -> CSI taps in pinned host memory: the file is read in chunks of
    ``chunk_sets`` frame-sets into two pinned staging buffers while the previous chunk
    is copied to HBM, correlated and copied back (`Correlator.process_host`).  Returns
    complex64 (F, n_r, n_t, L) on the host (synchronised)."""
    header = read_header(path)
    n_sets = _check_geometry(header, corr)
    if taps_host is None:
        taps_host = torch.empty(corr.taps_shape(n_sets), dtype=torch.complex64, pin_memory=True)
    elif tuple(taps_host.shape) != corr.taps_shape(n_sets) or taps_host.dtype != torch.complex64:
        raise DimensionMismatchError("taps_host must be complex64 (F, n_r, n_t, L)")
    chunk_sets = max(1, min(chunk_sets, n_sets)) if n_sets else 1
    stage = [torch.empty(corr.iq_shape(chunk_sets), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    done = [None, None]
    set_bytes = corr.cfg.n_batches * header.frame_bytes
    stream = torch.cuda.current_stream(corr.device)
    with open(path, "rb", buffering=0) as fh:
        fd = fh.fileno()
        for i, s in enumerate(range(0, n_sets, chunk_sets)):
            n = min(chunk_sets, n_sets - s)
            b = i & 1
            if done[b] is not None:
                done[b].synchronize()        # the H2D copy that read this staging buffer finished
            view = memoryview(stage[b][:n].numpy()).cast("B")
            _parallel_read(fd, view, HEADER_BYTES + s * set_bytes)
            corr.process_host(stage[b][:n], taps_host[s:s + n], chunk=n)
            done[b] = torch.cuda.Event()
            done[b].record(stream)
    torch.cuda.synchronize(corr.device)
    return taps_host


def write_iq_tensor(path, header: IqFileHeader, iq: torch.Tensor) -> None:
    """Device/host float32 IQ (F, n_batches, n_r, samples, 2) -> IQ file (frames in order)."""
    arr = iq.detach().to("cpu").contiguous().numpy().astype("<f4", copy=False)
    n_frames = arr.shape[0] * arr.shape[1]
    if n_frames != header.frame_count or arr.shape[2:] != (header.n_r, header.samples_per_receiver, 2):
        raise InvalidConfigError(f"tensor {arr.shape} does not match header {header}")
    with open(path, "wb") as fh:
        fh.write(header.pack())
        fh.write(arr.tobytes())
