"""Error metrics on device estimates (pnce/metrics.py:19-25 + the north-star MSE).

The hot-path scoring is fused into the correlation epilogue (CirEstimate.stats);
these helpers score arbitrary device tensors with on-device reductions.
"""

from __future__ import annotations

import torch

from .errors import DimensionMismatchError


def _taps(x) -> torch.Tensor:
    return getattr(x, "taps", x)


def mae(truth, est) -> float:
    """metrics.py:19-25: mean |est - truth| over all antenna pairs and lags."""
    t, e = _taps(truth), _taps(est)
    if tuple(t.shape) != tuple(e.shape):
        raise DimensionMismatchError(f"shape mismatch: truth {tuple(t.shape)} vs estimate {tuple(e.shape)}")
    t = torch.as_tensor(t).to(e.device if isinstance(e, torch.Tensor) else "cpu")
    return float(torch.mean(torch.abs(torch.as_tensor(e).to(torch.complex128) - t.to(torch.complex128))).item())


def mse(truth, est) -> float:
    """mean |est - truth|^2 (north-star addition; no reference symbol)."""
    t, e = _taps(truth), _taps(est)
    if tuple(t.shape) != tuple(e.shape):
        raise DimensionMismatchError(f"shape mismatch: truth {tuple(t.shape)} vs estimate {tuple(e.shape)}")
    t = torch.as_tensor(t).to(e.device if isinstance(e, torch.Tensor) else "cpu")
    d = torch.as_tensor(e).to(torch.complex128) - t.to(torch.complex128)
    return float(torch.mean(d.real ** 2 + d.imag ** 2).item())
