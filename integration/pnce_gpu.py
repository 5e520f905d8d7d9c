"""Reference-side binding: what a `pnce` maintainer adds as `pnce/gpu.py` to run the
reference's `process_frames` (pnce/experiments.py:176-208) on a B200 through
libpnce_b200.so (include/pnce_b200.h).  Plain ctypes over the C ABI; torch only for
device memory and the current stream.  This file is the one INTEGRATION.md shows, kept
executable so tests/test_gpu_integration.py runs it on the reference's own objects
(PnSequence, PilotConfig, BatchPlan, ReceivedFrame, BackendConfig) from baseline/_ref.

Drop-in contract: same signature and return type as the reference's process_frames;
`rows_per_batch` may carry a `GpuPlan` (the device counterpart of the static correlator
rows, experiments.py:157-173) so repeated calls reuse it.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from pnce.errors import (DimensionMismatchError, FrameTooShortError, InvalidConfigError, InvalidSpecError,
                         NotMaximalLengthError, PlanMismatchError, PnceError, RowsOutOfRangeError,
                         SaturationDetectedError, ZeroStateError)
from pnce.estimator import CirEstimate

_ERR = {1: InvalidConfigError, 2: InvalidSpecError, 3: ZeroStateError, 4: NotMaximalLengthError,
        5: DimensionMismatchError, 6: FrameTooShortError, 7: PlanMismatchError, 8: RowsOutOfRangeError,
        9: SaturationDetectedError}


class _Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("m", "c", "n_t", "n_r", "n_batch", "l", "degree")] + \
               [("tap_mask", ctypes.c_uint32), ("state", ctypes.c_uint32), ("dtype", ctypes.c_int32)]


_lib = ctypes.CDLL(os.environ.get("PNCE_B200_LIB", "libpnce_b200.so"))
_vp = ctypes.c_void_p
_lib.pnce_last_error.restype = ctypes.c_char_p
_lib.pnce_plan_create.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(_vp), _vp]
_lib.pnce_plan_destroy.argtypes = [_vp]
_lib.pnce_process_frames.argtypes = [_vp] * 6 + [ctypes.c_size_t, ctypes.c_int64, _vp]
_lib.pnce_process_frames_tensor16.argtypes = [_vp] * 5 + [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _vp]


def _check(rc: int) -> None:
    if rc:
        raise _ERR.get(rc, PnceError)(_lib.pnce_last_error().decode())


class GpuPlan:
    """Device correlator state for one (sequence, PilotConfig, n_r)."""

    def __init__(self, seq, cfg, n_r: int):
        spec = seq.spec
        if spec is None:
            raise InvalidConfigError("the device plan regenerates the chips from the sequence's LfsrSpec")
        mask = sum(1 << (t - 1) for t in spec.taps)
        self.key = (cfg, n_r)
        self._c = _Cfg(cfg.m, cfg.c, cfg.n_t, n_r, cfg.n_batch, cfg.l, spec.degree, mask, spec.state, 0)
        self.handle = _vp()
        _check(_lib.pnce_plan_create(ctypes.byref(self._c), ctypes.byref(self.handle), _stream()))

    def __del__(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.pnce_plan_destroy(self.handle)
            self.handle = None


def _stream() -> ctypes.c_void_p:
    return _vp(torch.cuda.current_stream().cuda_stream)


def process_frames_gpu(seq, cfg, plan, frames, backend, counters=None, rows_per_batch=None) -> CirEstimate:
    """experiments.py:176-208 on the B200: same arguments, same CirEstimate (complex128 taps,
    already x 1/M; saturated batches zeroed and counted n_r * n_tx)."""
    n_r = frames[0].n_r
    gp = rows_per_batch if isinstance(rows_per_batch, GpuPlan) and rows_per_batch.key == (cfg, n_r) \
        else GpuPlan(seq, cfg, n_r)
    if len(frames) != len(plan.batches):
        raise DimensionMismatchError(f"{len(frames)} frames for {len(plan.batches)} batches")
    # frames -> f32 (I, Q) [1][n_batches][n_r][P+L-1][2], the iqfile.py payload layout
    iq = np.stack([np.stack([f.samples.real, f.samples.imag], -1) for f in frames]).astype(np.float32)[None]
    d_iq = torch.from_numpy(iq).cuda()
    d_taps = torch.empty((1, n_r, cfg.n_t, cfg.l), dtype=torch.complex64, device="cuda")
    stats = torch.zeros((1, 4), dtype=torch.float64, device="cuda")   # .., .., non-finite, saturations
    if backend.kind == "tensor16":
        _check(_lib.pnce_process_frames_tensor16(gp.handle, d_iq.data_ptr(), d_taps.data_ptr(), None,
                                                 stats.data_ptr(), backend.chunk_len or 0,
                                                 1 if backend.accumulator == "binary16" else 0, 1, _stream()))
    else:   # reference64 / reference32: the fused fp16 path (north-star tolerance)
        _check(_lib.pnce_process_frames(gp.handle, d_iq.data_ptr(), d_taps.data_ptr(), None, stats.data_ptr(),
                                        None, 0, 1, _stream()))
    if counters is not None:
        counters.samples_moved += len(frames) * n_r * cfg.p
        counters.macs += cfg.n_t * cfg.l * cfg.m * n_r
    taps = d_taps[0].cpu().numpy().astype(np.complex128)
    return CirEstimate(taps=taps, backend=backend.kind, norm=1.0 / cfg.m,
                       saturations=int(round(float(stats[0, 3].item()))))
