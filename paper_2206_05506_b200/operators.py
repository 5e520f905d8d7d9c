"""Operator-level seam: `correlate_rows` and its callers
`estimate_sequential` / `estimate_batched` (pnce/estimator.py:50-140) on the tensor cores.

The rows are arbitrary (caller-built lag windows at any shifts), so each call builds a
rows plan (`pnce_plan_create_rows`: fp16/bf16 K-major operand of the given rows, 1/norm_len
scale) and correlates the received columns as compact body rows (`pnce_process_bodies`).
`RowsCorrelator` keeps the plan for repeated use with the same rows.  The single device
path computes with fp16 (default) or bf16 operands and fp32 accumulation -- the
reference's tensor16 quantiser; there is no reference64/32 branch.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatchError, InvalidConfigError, PlanMismatchError, RowsOutOfRangeError
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

    def __call__(self, y) -> torch.Tensor:
        """y: (M,) or (M, cols) complex -> (R,) or (R, cols) complex64 on the device."""
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
            _lib.check(_lib.lib().pnce_process_bodies(self._plan, ctypes.c_void_p(body.data_ptr()), self.stride,
                                                      ctypes.c_void_p(taps.data_ptr()), None, None, None, 1,
                                                      _stream_ptr(self.device)))
        out = taps[0, :, 0, :].transpose(0, 1)                       # (R, cols)
        return out[:, 0] if squeeze else out


def correlate_rows(rows, y, backend: str | None = None, norm_len: int | None = None) -> torch.Tensor:
    """estimator.py:68-86: (1/norm_len) rows @ y for complex y ((M,) or (M, cols)).
    ``backend``: operand dtype "fp16" (default) or "bf16"."""
    yt = y if isinstance(y, torch.Tensor) else np.asarray(y)
    cols = 1 if yt.ndim == 1 else int(yt.shape[1])
    return RowsCorrelator(rows, cols, norm_len, dtype=backend or "fp16")(y)


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
