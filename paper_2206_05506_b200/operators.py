"""Operator-level seam: `correlate_rows` and its callers
`estimate_sequential` / `estimate_batched` (pnce/estimator.py:50-140) on the tensor cores.

The rows are arbitrary (caller-built lag windows at any shifts), so each call builds a
rows plan (`pnce_plan_create_rows`: fp16/bf16 K-major operand of the given rows, 1/norm_len
scale) and correlates the received columns as compact body rows (`pnce_process_bodies`).
`RowsCorrelator` keeps the plan for repeated use with the same rows.  The single device
path computes with fp16 (default) or bf16 operands and fp32 accumulation -- the
reference's tensor16 quantiser; the reference's ``BackendConfig`` is accepted (backend.py):
reference64/32 run that path, tensor16 runs the chunked tensor16 mode and raises
SaturationDetectedError like halfprec.py:118-124.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .backend import resolve as resolve_backend
from .errors import (DimensionMismatchError, InvalidConfigError, PlanMismatchError, RowsOutOfRangeError,
                     SaturationDetectedError)
from .estimator import DTYPES, _stream_ptr
from .pilots import BatchAssignment, cyclic_separation
from .pn import PnSequence


class RowsCorrelator:
    """Device plan over caller rows (R x M, +-1) for `cols` received columns."""

    def __init__(self, rows, cols: int, norm_len: int | None = None, dtype: str = "fp16",
                 device: torch.device | str | None = None):
        if dtype not in DTYPES:
            raise InvalidConfigError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        r = torch.as_tensor(np.asarray(rows, dtype=np.float32) if not isinstance(rows, torch.Tensor) else rows)
        r = r.to(device=self.device, dtype=torch.float32).contiguous()
        if r.dim() != 2:
            raise DimensionMismatchError(f"rows must be 2-D (R, M), got {tuple(r.shape)}")
        self.n_rows, self.m = int(r.shape[0]), int(r.shape[1])
        if not 1 <= self.n_rows <= self.m:
            raise RowsOutOfRangeError(f"rows {self.n_rows} outside [1, {self.m}]")
        self.cols = int(cols)
        self.norm_len = int(norm_len if norm_len is not None else self.m)
        self.stride = self.m + (self.m & 1)
        cfg = _lib.CfgStruct(m=self.m, c=0, n_t=1, n_r=self.cols, n_batch=1, l=self.n_rows, degree=0, tap_mask=0,
                             state=0, dtype=DTYPES[dtype])
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_plan_create_rows(ctypes.byref(cfg), ctypes.c_void_p(r.data_ptr()),
                                                        self.n_rows, self.norm_len, ctypes.byref(handle),
                                                        _stream_ptr(self.device)))
        self._plan = handle

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None and plan.value:
            try:
                _lib.lib().pnce_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    def __call__(self, y, tensor16: tuple | None = None) -> torch.Tensor:
        """y: (M,) or (M, cols) complex -> (R,) or (R, cols) complex64 on the device.
        ``tensor16``: (chunk_len | None, accumulator) runs the tensor16 mode."""
        yt = y if isinstance(y, torch.Tensor) else torch.from_numpy(np.asarray(y, dtype=np.complex128))
        squeeze = yt.dim() == 1
        y2 = yt[:, None] if squeeze else yt
        if y2.shape[0] != self.m:
            raise InvalidConfigError(f"operand lengths differ: rows have {self.m} columns, y has {y2.shape[0]}")
        if y2.shape[1] != self.cols:
            raise DimensionMismatchError(f"y has {y2.shape[1]} columns, correlator built for {self.cols}")
        # compact body rows: [1 frame][1 batch][cols][stride][2] float32
        body = torch.zeros((self.cols, self.stride, 2), dtype=torch.float32, device=self.device)
        yc = y2.to(device=self.device, dtype=torch.complex64).transpose(0, 1)
        body[:, :self.m] = torch.view_as_real(yc.contiguous())
        taps = torch.empty((1, self.cols, 1, self.n_rows), dtype=torch.complex64, device=self.device)
        with torch.cuda.device(self.device):
            if tensor16 is not None:
                chunk_len, acc = tensor16
                stats = torch.zeros((1, 4), dtype=torch.float64, device=self.device)
                _lib.check(_lib.lib().pnce_process_bodies_tensor16(
                    self._plan, ctypes.c_void_p(body.data_ptr()), self.stride, ctypes.c_void_p(taps.data_ptr()),
                    None, ctypes.c_void_p(stats.data_ptr()), 0 if chunk_len is None else int(chunk_len),
                    1 if acc == "binary16" else 0, 1, _stream_ptr(self.device)))
                if float(stats[0, 3].item()) > 0:
                    raise SaturationDetectedError(f"non-finite {acc} partial or running total")
            else:
                _lib.check(_lib.lib().pnce_process_bodies(self._plan, ctypes.c_void_p(body.data_ptr()), self.stride,
                                                          ctypes.c_void_p(taps.data_ptr()), None, None, None, 1,
                                                          _stream_ptr(self.device)))
        out = taps[0, :, 0, :].transpose(0, 1)                       # (R, cols)
        return out[:, 0] if squeeze else out


def correlate_rows(rows, y, backend=None, norm_len: int | None = None) -> torch.Tensor:
    """estimator.py:68-86: (1/norm_len) rows @ y for complex y ((M,) or (M, cols)).
    ``backend``: the reference's BackendConfig (backend.py mapping) or "fp16" (default) / "bf16"."""
    mode = resolve_backend(backend)
    yt = y if isinstance(y, torch.Tensor) else np.asarray(y)
    cols = 1 if yt.ndim == 1 else int(yt.shape[1])
    corr = RowsCorrelator(rows, cols, norm_len, dtype=mode.dtype)
    return corr(y, (mode.chunk_len, mode.accumulator) if mode.tensor16 else None)


def _lag_rows(seq: PnSequence, lags) -> torch.Tensor:
    m = seq.m
    idx = (torch.arange(m, device=seq.chips.device)[None, :] - torch.as_tensor(lags, device=seq.chips.device)[:, None]) % m
    return seq.chips[idx]


def build_partial_circulant(seq: PnSequence, rows: int) -> torch.Tensor:
    """estimator.py:50-59: the first ``rows`` lag rows of the PN circulant (device, +-1)."""
    if not 1 <= rows <= seq.m:
        raise RowsOutOfRangeError(f"rows {rows} outside [1, {seq.m}]")
    return _lag_rows(seq, torch.arange(rows))


def batched_lag_rows(seq: PnSequence, batch: Sequence[BatchAssignment], l: int) -> torch.Tensor:
    """estimator.py:114-117: stacked lag windows [shift, shift + L) of every transmitter."""
    lags = torch.cat([(a.shift + torch.arange(l)) % seq.m for a in batch])
    return _lag_rows(seq, lags)


def validate_batch_separation(batch: Sequence[BatchAssignment], m: int, l: int) -> None:
    """estimator.py:103-111."""
    shifts = [a.shift for a in batch]
    for i in range(len(shifts)):
        for j in range(i + 1, len(shifts)):
            sep = cyclic_separation(shifts[i], shifts[j], m)
            if sep < l:
                raise PlanMismatchError(f"shifts {shifts[i]} and {shifts[j]} separated by {sep} < L={l}")


def estimate_sequential(y, seq: PnSequence, l: int, backend: str | None = None) -> torch.Tensor:
    """estimator.py:89-100: correlation estimate of the first L CIR lags of one body."""
    yt = y if isinstance(y, torch.Tensor) else np.asarray(y)
    if yt.shape[-1 if yt.ndim == 1 else 0] != seq.m:
        raise DimensionMismatchError(f"received body has {yt.shape[0]} samples, expected M={seq.m}")
    return correlate_rows(build_partial_circulant(seq, l), y, backend, norm_len=seq.m)


def estimate_batched(y, seq: PnSequence, batch: Sequence[BatchAssignment], l: int,
                     backend: str | None = None) -> dict[int, torch.Tensor]:
    """estimator.py:120-140: de-multiplexed CIR estimates for every transmitter of a batch."""
    yt = y if isinstance(y, torch.Tensor) else np.asarray(y)
    if yt.shape[0] != seq.m:
        raise DimensionMismatchError(f"received body has {yt.shape[0]} samples, expected M={seq.m}")
    if not batch:
        raise PlanMismatchError("empty batch")
    validate_batch_separation(batch, seq.m, l)
    flat = correlate_rows(batched_lag_rows(seq, batch, l), y, backend, norm_len=seq.m)
    return {a.transmitter: flat[i * l:(i + 1) * l] for i, a in enumerate(batch)}
