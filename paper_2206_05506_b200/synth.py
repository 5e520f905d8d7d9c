"""Device-side input synthesis: channel draws and pilot sweeps.

Counterparts of `draw_channel` (pnce/channel.py:96-108) and `simulate_frame`
(channel.py:186-214) running on the GPU for whole batches of frame-sets, so benches and
SNR/tap sweeps are not bound by host-side synthesis (0.36 s per cfg3 frame-set in the
reference).  Same laws and the same deterministic structure (noiseless frames are the
exact linear convolution of each batch pilot with its CIR; noise is calibrated with
noise_reference_power), but Philox streams: statistically equivalent, not draw-for-draw
identical to numpy's PCG64.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .errors import DimensionMismatchError, InvalidSpecError


def _stream(dev: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def draw_channel(corr, n_frames: int, l_nz: int | None = None, seed: int = 0) -> torch.Tensor:
    """complex64 (F, n_r, n_t, L) CIRs with the draw_channel law (L_nz = L: dense)."""
    l_nz = corr.cfg.l if l_nz is None else int(l_nz)
    if not 1 <= l_nz <= corr.cfg.l:
        raise InvalidSpecError(f"l_nz must be in [1, L={corr.cfg.l}], got {l_nz}")
    h = torch.empty(corr.taps_shape(n_frames), dtype=torch.complex64, device=corr.device)
    with torch.cuda.device(corr.device):
        _lib.check(_lib.lib().pnce_draw_channel(corr._plan, l_nz, seed & (2**64 - 1), ctypes.c_void_p(h.data_ptr()),
                                                n_frames, _stream(corr.device)))
    return h


def simulate_frames(corr, h: torch.Tensor, snr_db: float = math.inf, seed: int = 0,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """float32 IQ (F, n_batches, n_r, P+L-1, 2) for the CIRs ``h`` (F, n_r, n_t, L) complex64."""
    if h.dim() == 3:
        h = h.unsqueeze(0)
    n_frames = int(h.shape[0])
    if tuple(h.shape) != corr.taps_shape(n_frames) or h.dtype != torch.complex64 or h.device != corr.device:
        raise DimensionMismatchError(f"h must be complex64 {corr.taps_shape(n_frames)} on {corr.device}")
    h = h.contiguous()
    if out is None:
        out = torch.empty(corr.iq_shape(n_frames), dtype=torch.float32, device=corr.device)
    elif tuple(out.shape) != corr.iq_shape(n_frames) or out.dtype != torch.float32 or not out.is_contiguous():
        raise DimensionMismatchError("out must be contiguous float32 (F, n_batches, n_r, P+L-1, 2)")
    if math.isnan(snr_db):
        raise InvalidSpecError("snr_db is NaN")
    with torch.cuda.device(corr.device):
        _lib.check(_lib.lib().pnce_simulate_frames(corr._plan, ctypes.c_void_p(h.data_ptr()), float(snr_db),
                                                   seed & (2**64 - 1), ctypes.c_void_p(out.data_ptr()), n_frames,
                                                   _stream(corr.device)))
    return out
