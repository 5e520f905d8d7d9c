"""Device correlator front end, mirroring the reference's estimator API.

Reference seam: `process_frames` (pnce/experiments.py:176-208) calling
`correlate_rows` (pnce/estimator.py:68-86) with the static correlator state of
`correlator_rows_for_plan` (experiments.py:157-173).  Here the correlator state
is a device plan (C ABI `pnce_plan_create`: device LFSR + stacked lag-window
rows in tensor-core operand layout) and every frame-set goes through one device
path: pack (CP strip, de-interleave, fp16/bf16) -> tcgen05 correlation -> fused
1/M, demux and scoring.  There is no CPU fallback; the reference's BackendConfig
selects between the fused path and its tensor16 mode (backend.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .backend import resolve as resolve_backend
from .errors import DimensionMismatchError, FrameTooShortError, InvalidConfigError
from .pilots import BatchPlan, PilotConfig, build_batch_plan
from .pn import LfsrSpec, PnSequence

DTYPES = {"fp16": _lib.PNCE_DTYPE_FP16, "bf16": _lib.PNCE_DTYPE_BF16}


@dataclass(frozen=True, eq=False)
class CirEstimate:
    """estimator.py:27-37.  taps: complex64 device tensor (n_r, n_t, L) or (F, n_r, n_t, L).

    ``stats`` (float64 (F, 4): sum|e|, sum|e|^2, non-finite taps, saturations) is filled
    by the fused epilogue (the error sums when ground truth was supplied), and ``link_mse``
    (float32 (F, n_r, n_t) or (n_r, n_t)) with each link's mean |e|^2 over its L taps.
    """

    taps: torch.Tensor
    backend: str
    norm: float
    saturations: int = 0
    stats: torch.Tensor | None = None
    link_mse: torch.Tensor | None = None

    def mae(self) -> float:
        """metrics.py:19-25 from the fused per-frame sums."""
        if self.stats is None:
            raise InvalidConfigError("estimate was produced without ground truth")
        return float(self.stats[:, 0].sum().item()) / self.taps.numel()

    def mse(self) -> float:
        if self.stats is None:
            raise InvalidConfigError("estimate was produced without ground truth")
        return float(self.stats[:, 1].sum().item()) / self.taps.numel()


@dataclass
class WorkCounters:
    """experiments.py:98-109: samples_moved (P per batch per receiver), macs (rows x M x n_r)."""

    samples_moved: int = 0
    macs: int = 0


def remove_cp(samples, c: int, m: int):
    """estimator.py:40-47 (a view; the device path fuses it into the pack kernel)."""
    if samples.shape[-1] < c + m:
        raise FrameTooShortError(f"frame has {samples.shape[-1]} samples, need at least C+M={c + m}")
    return samples[..., c:c + m]


def _stream_ptr(dev: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _same_device(dev: torch.device, **tensors) -> None:
    """Every tensor argument must live on the plan's device: a foreign pointer would reach
    TMA descriptors and kernels of another GPU (DimensionMismatchError instead)."""
    for name, t in tensors.items():
        if t is not None and (not t.is_cuda or t.device != dev):
            raise DimensionMismatchError(f"{name} is on {t.device}, the correlator on {dev}")


class Correlator:
    """Static correlator state for one (sequence, PilotConfig, n_r, dtype).

    The device counterpart of `correlator_rows_for_plan` (experiments.py:157-173):
    all full batches share one stacked row matrix and a short last batch uses
    its row prefix, so one plan serves every batch and every frame-set.
    """

    def __init__(self, spec: LfsrSpec, cfg: PilotConfig, n_r: int, dtype: str = "fp16",
                 device: torch.device | str | None = None):
        if dtype not in DTYPES:
            raise InvalidConfigError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        if spec.period_target != cfg.m:
            raise DimensionMismatchError(f"sequence length {spec.period_target} != configured M {cfg.m}")
        if n_r < 1:
            raise InvalidConfigError(f"n_r must be >= 1, got {n_r}")
        self.spec, self.cfg, self.n_r, self.dtype = spec, cfg, n_r, dtype
        self.plan_layout: BatchPlan = build_batch_plan(cfg)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._c = _lib.CfgStruct(m=cfg.m, c=cfg.c, n_t=cfg.n_t, n_r=n_r, n_batch=cfg.n_batch,
                                 l=cfg.l, degree=spec.degree, tap_mask=spec.tap_mask,
                                 state=spec.state, dtype=DTYPES[dtype])
        L = _lib.lib()
        _lib.check(L.pnce_config_check(ctypes.byref(self._c)))
        handle = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.pnce_plan_create(ctypes.byref(self._c), ctypes.byref(handle),
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

    # ------------------------------------------------------------ shapes
    @property
    def samples(self) -> int:
        return self.cfg.samples_per_receiver

    def iq_shape(self, n_frames: int) -> tuple[int, ...]:
        """float32 (F, n_batches, n_r, P + L - 1, 2): the IQ file payload layout."""
        return (n_frames, self.cfg.n_batches, self.n_r, self.samples, 2)

    def taps_shape(self, n_frames: int) -> tuple[int, ...]:
        return (n_frames, self.n_r, self.cfg.n_t, self.cfg.l)

    def chips(self) -> torch.Tensor:
        """Device chips the plan was built from (device LFSR output)."""
        out = torch.empty(self.cfg.m, dtype=torch.float32, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_plan_chips(self._plan, ctypes.c_void_p(out.data_ptr()),
                                                  _stream_ptr(self.device)))
        return out

    def operand(self) -> torch.Tensor:
        """The plan's device-built correlation operand (fp16/bf16 [rows_alloc][K_pad], rows
        j*L + l = chips shifted by s_j + l; batched_lag_rows, estimator.py:114-117)."""
        L = _lib.lib()
        rows, kp = ctypes.c_int32(), ctypes.c_int32()
        _lib.check(L.pnce_plan_operand(self._plan, None, ctypes.byref(rows), ctypes.byref(kp), None))
        tdt = torch.float16 if self.dtype == "fp16" else torch.bfloat16
        out = torch.empty((rows.value, kp.value), dtype=tdt, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(L.pnce_plan_operand(self._plan, ctypes.c_void_p(out.data_ptr()), None, None,
                                           _stream_ptr(self.device)))
        return out

    def packed_bytes(self, n_frames: int) -> int:
        """Size of the packed 16-bit operand `pack` produces (the fused path needs none)."""
        return int(_lib.lib().pnce_workspace_bytes(self._plan, n_frames))

    # ------------------------------------------------------------ validation
    def _check_iq(self, iq: torch.Tensor) -> tuple[torch.Tensor, int]:
        if not isinstance(iq, torch.Tensor) or not iq.is_cuda:
            raise DimensionMismatchError("iq must be a CUDA tensor (use process_frames for host frames)")
        _same_device(self.device, iq=iq)
        if iq.dtype != torch.float32:
            raise DimensionMismatchError(f"iq must be float32 (I, Q) pairs, got {iq.dtype}")
        if iq.dim() == 4:
            iq = iq.unsqueeze(0)
        if iq.dim() != 5 or iq.shape[-1] != 2:
            raise DimensionMismatchError(f"iq must be (F, n_batches, n_r, samples, 2), got {tuple(iq.shape)}")
        if iq.shape[-2] < self.cfg.c + self.cfg.m:
            raise FrameTooShortError(
                f"frame has {iq.shape[-2]} samples, need at least C+M={self.cfg.c + self.cfg.m}")
        if tuple(iq.shape[1:]) != self.iq_shape(1)[1:]:
            raise DimensionMismatchError(f"iq shape {tuple(iq.shape)} != {self.iq_shape(iq.shape[0])}")
        if not iq.is_contiguous():
            iq = iq.contiguous()
        return iq, int(iq.shape[0])

    # ------------------------------------------------------------ hot path
    def process(self, iq: torch.Tensor, truth: torch.Tensor | None = None,
                out: torch.Tensor | None = None, stats: torch.Tensor | None = None):
        """Estimate every frame-set in ``iq``: returns (taps complex64 (F, n_r, n_t, L), stats|None).

        ``truth`` (complex64, same shape as taps) switches on the fused scoring
        (per-frame sum|e|, sum|e|^2, non-finite count into ``stats`` (F, 4) f64).
        """
        iq, n_frames = self._check_iq(iq)
        if out is None:
            out = torch.empty(self.taps_shape(n_frames), dtype=torch.complex64, device=self.device)
        elif tuple(out.shape) != self.taps_shape(n_frames) or out.dtype != torch.complex64 or not out.is_contiguous():
            raise DimensionMismatchError("out must be contiguous complex64 (F, n_r, n_t, L)")
        truth_ptr = None
        if truth is not None:
            if tuple(truth.shape) != self.taps_shape(n_frames) or truth.dtype != torch.complex64 or not truth.is_cuda:
                raise DimensionMismatchError("truth must be CUDA complex64 (F, n_r, n_t, L)")
            truth = truth.contiguous()
            truth_ptr = ctypes.c_void_p(truth.data_ptr())
            if stats is None:
                stats = torch.zeros((n_frames, 4), dtype=torch.float64, device=self.device)
        stats_ptr = None
        if stats is not None:
            if tuple(stats.shape) != (n_frames, 4) or stats.dtype != torch.float64 or not stats.is_contiguous():
                raise DimensionMismatchError("stats must be contiguous float64 (F, 4)")
            stats_ptr = ctypes.c_void_p(stats.data_ptr())
        _same_device(self.device, out=out, truth=truth, stats=stats)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_process_frames(
                self._plan, ctypes.c_void_p(iq.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                truth_ptr, stats_ptr, None, 0, n_frames, _stream_ptr(self.device)))
        return out, stats

    def process_gather(self, iq: torch.Tensor, csi: torch.Tensor, r0: int, peers=()) -> torch.Tensor:
        """Antenna split with the all-gather fused into the epilogue (pnce_process_frames_gather):
        this correlator's n_r receivers are rows [r0, r0 + n_r) of ``csi`` (complex64
        (F, n_r_total, n_t, L) on this device); every tap goes into ``csi`` and into each peer
        buffer (``peers``: same-shape tensors or raw device pointers mapped into this context,
        e.g. the other ranks' ``csi`` opened over CUDA IPC).  Asynchronous on the current
        stream; the ranks order themselves (stream sync + barrier) before reading."""
        iq, n_frames = self._check_iq(iq)
        n_t, L = self.cfg.n_t, self.cfg.l
        if csi.dim() != 4 or csi.shape[0] != n_frames or tuple(csi.shape[2:]) != (n_t, L) or \
                csi.dtype != torch.complex64 or not csi.is_contiguous():
            raise DimensionMismatchError("csi must be contiguous complex64 (F, n_r_total, n_t, L)")
        _same_device(self.device, csi=csi)
        n_r_total = int(csi.shape[1])
        ptrs = []
        for q in peers:
            if isinstance(q, torch.Tensor):
                if tuple(q.shape) != tuple(csi.shape) or q.dtype != csi.dtype or not q.is_contiguous():
                    raise DimensionMismatchError("peer CSI buffers must match csi")
                ptrs.append(q.data_ptr())
            else:
                ptrs.append(int(q))
        arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_process_frames_gather(
                self._plan, ctypes.c_void_p(iq.data_ptr()), ctypes.c_void_p(csi.data_ptr()), arr, len(ptrs),
                n_r_total, int(r0), n_frames, _stream_ptr(self.device)))
        return csi

    def process_scored(self, iq: torch.Tensor, truth: torch.Tensor, out: torch.Tensor | None = None,
                       stats: torch.Tensor | None = None, link_mse: torch.Tensor | None = None):
        """`process` with the fused per-link scoring (north star (4)): returns
        (taps, stats (F, 4) f64, link_mse (F, n_r, n_t) f32 = mean_l |h_est - h_true|^2)."""
        iq, n_frames = self._check_iq(iq)
        if out is None:
            out = torch.empty(self.taps_shape(n_frames), dtype=torch.complex64, device=self.device)
        elif tuple(out.shape) != self.taps_shape(n_frames) or out.dtype != torch.complex64 or not out.is_contiguous():
            raise DimensionMismatchError("out must be contiguous complex64 (F, n_r, n_t, L)")
        if truth is None or tuple(truth.shape) != self.taps_shape(n_frames) or truth.dtype != torch.complex64 \
                or not truth.is_cuda:
            raise DimensionMismatchError("truth must be CUDA complex64 (F, n_r, n_t, L)")
        truth = truth.contiguous()
        if stats is None:
            stats = torch.zeros((n_frames, 4), dtype=torch.float64, device=self.device)
        elif tuple(stats.shape) != (n_frames, 4) or stats.dtype != torch.float64:
            raise DimensionMismatchError("stats must be float64 (F, 4)")
        lshape = (n_frames, self.n_r, self.cfg.n_t)
        if link_mse is None:
            link_mse = torch.zeros(lshape, dtype=torch.float32, device=self.device)
        elif tuple(link_mse.shape) != lshape or link_mse.dtype != torch.float32 or not link_mse.is_contiguous():
            raise DimensionMismatchError("link_mse must be contiguous float32 (F, n_r, n_t), zero-filled")
        _same_device(self.device, out=out, truth=truth, stats=stats, link_mse=link_mse)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_process_frames_scored(
                self._plan, ctypes.c_void_p(iq.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                ctypes.c_void_p(truth.data_ptr()), ctypes.c_void_p(stats.data_ptr()),
                ctypes.c_void_p(link_mse.data_ptr()), n_frames, _stream_ptr(self.device)))
        return out, stats, link_mse

    def process_tensor16(self, iq: torch.Tensor, chunk_len: int | None = 256, accumulator: str = "binary32",
                         truth: torch.Tensor | None = None, out: torch.Tensor | None = None,
                         stats: torch.Tensor | None = None):
        """The reference's tensor16 backend (halfprec.py:93-125, `BackendConfig(kind="tensor16",
        chunk_len, accumulator)`) on the tensor cores: chunked binary16/binary32 partials, each
        x fp32(1/M) into an fp32 total; saturated batches scored as zeros and counted.
        Returns (taps, stats (F, 4) f64: sum|e|, sum|e|^2, non-finite, saturations)."""
        if accumulator not in ("binary32", "binary16"):
            raise InvalidConfigError(f"unknown accumulator {accumulator!r}")
        iq, n_frames = self._check_iq(iq)
        if out is None:
            out = torch.empty(self.taps_shape(n_frames), dtype=torch.complex64, device=self.device)
        elif tuple(out.shape) != self.taps_shape(n_frames) or out.dtype != torch.complex64 or not out.is_contiguous():
            raise DimensionMismatchError("out must be contiguous complex64 (F, n_r, n_t, L)")
        truth_ptr = None
        if truth is not None:
            if tuple(truth.shape) != self.taps_shape(n_frames) or truth.dtype != torch.complex64 or not truth.is_cuda:
                raise DimensionMismatchError("truth must be CUDA complex64 (F, n_r, n_t, L)")
            truth = truth.contiguous()
            truth_ptr = ctypes.c_void_p(truth.data_ptr())
        if stats is None:
            stats = torch.zeros((n_frames, 4), dtype=torch.float64, device=self.device)
        elif tuple(stats.shape) != (n_frames, 4) or stats.dtype != torch.float64 or not stats.is_contiguous():
            raise DimensionMismatchError("stats must be contiguous float64 (F, 4)")
        _same_device(self.device, out=out, truth=truth, stats=stats)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_process_frames_tensor16(
                self._plan, ctypes.c_void_p(iq.data_ptr()), ctypes.c_void_p(out.data_ptr()), truth_ptr,
                ctypes.c_void_p(stats.data_ptr()), 0 if chunk_len is None else int(chunk_len),
                1 if accumulator == "binary16" else 0, n_frames, _stream_ptr(self.device)))
        return out, stats

    def process_host(self, iq_host: torch.Tensor, taps_host: torch.Tensor, chunk: int = 8,
                     bodies_only: bool = True) -> torch.Tensor:
        """Host-buffer path (IQ ingest): pinned host IQ -> HBM by chunked
        async copies on a copy stream, correlate on the current stream, taps back to pinned
        host memory on a second copy stream; double-buffered so the PCIe transfers in both
        directions overlap the device work.  ``bodies_only``: remove_cp happens in the DMA
        (a pitched copy of the M body samples per row: 11 % fewer bytes over PCIe at cfg3).
        Asynchronous w.r.t. the host: the current stream waits for the final D2H copy."""
        if iq_host.is_cuda or taps_host.is_cuda:
            raise DimensionMismatchError("process_host takes host (pinned) tensors")
        n_frames = int(iq_host.shape[0])
        if tuple(iq_host.shape) != self.iq_shape(n_frames) or tuple(taps_host.shape) != self.taps_shape(n_frames):
            raise DimensionMismatchError("host iq/taps shapes do not match the correlator")
        if not iq_host.is_contiguous() or not taps_host.is_contiguous():
            raise DimensionMismatchError("host iq/taps must be contiguous")
        if n_frames == 0:
            return taps_host
        chunk = max(1, min(chunk, n_frames))
        stride = self.cfg.m + (self.cfg.m & 1)       # even: 16-byte aligned compact rows
        cur = torch.cuda.current_stream(self.device)
        key = (chunk, bodies_only)
        st = getattr(self, "_host_streams", None)
        if st is None or st[2] != key:
            in_shape = (chunk, self.cfg.n_batches, self.n_r, stride, 2) if bodies_only else self.iq_shape(chunk)
            bufs_in = [torch.empty(in_shape, dtype=torch.float32, device=self.device) for _ in range(2)]
            bufs_out = [torch.empty(self.taps_shape(chunk), dtype=torch.complex64, device=self.device)
                        for _ in range(2)]
            st = (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device), key, bufs_in, bufs_out)
            self._host_streams = st
        s_in, s_out, _, bufs_in, bufs_out = st
        L = _lib.lib()
        if n_frames <= chunk and bodies_only:
            # one stage (the single frame-set latency case): nothing to overlap, so copy in,
            # correlate and copy out in order on the current stream -- no side streams/events
            with torch.cuda.device(self.device):
                sp = ctypes.c_void_p(cur.cuda_stream)
                _lib.check(L.pnce_copy_bodies_h2d(self._plan, ctypes.c_void_p(iq_host.data_ptr()),
                                                  ctypes.c_void_p(bufs_in[0].data_ptr()), stride, n_frames, sp))
                _lib.check(L.pnce_process_bodies(self._plan, ctypes.c_void_p(bufs_in[0].data_ptr()), stride,
                                                 ctypes.c_void_p(bufs_out[0].data_ptr()), None, None, None,
                                                 n_frames, sp))
                taps_host.copy_(bufs_out[0][:n_frames], non_blocking=True)
            return taps_host
        in_done = [torch.cuda.Event() for _ in range(2)]
        comp_done = [torch.cuda.Event() for _ in range(2)]
        out_done = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        for i, s in enumerate(range(0, n_frames, chunk)):
            b = i & 1
            n = min(chunk, n_frames - s)
            if used[b]:
                s_in.wait_event(comp_done[b])
            with torch.cuda.device(self.device), torch.cuda.stream(s_in):
                if bodies_only:
                    _lib.check(L.pnce_copy_bodies_h2d(self._plan, ctypes.c_void_p(iq_host[s].data_ptr()),
                                                      ctypes.c_void_p(bufs_in[b].data_ptr()), stride, n,
                                                      ctypes.c_void_p(s_in.cuda_stream)))
                else:
                    bufs_in[b][:n].copy_(iq_host[s:s + n], non_blocking=True)
                in_done[b].record(s_in)
            cur.wait_event(in_done[b])
            if used[b]:
                cur.wait_event(out_done[b])
            if bodies_only:
                with torch.cuda.device(self.device):
                    _lib.check(L.pnce_process_bodies(self._plan, ctypes.c_void_p(bufs_in[b].data_ptr()), stride,
                                                     ctypes.c_void_p(bufs_out[b].data_ptr()), None, None, None, n,
                                                     ctypes.c_void_p(cur.cuda_stream)))
            else:
                self.process(bufs_in[b][:n], out=bufs_out[b][:n])
            comp_done[b].record(cur)
            s_out.wait_event(comp_done[b])
            with torch.cuda.stream(s_out):
                taps_host[s:s + n].copy_(bufs_out[b][:n], non_blocking=True)
                out_done[b].record(s_out)
            used[b] = True
        cur.wait_stream(s_out)
        return taps_host

    def capture(self, iq: torch.Tensor, out: torch.Tensor | None = None) -> tuple[torch.cuda.CUDAGraph, torch.Tensor]:
        """Record `process(iq, out)` into a CUDA graph for repeated calls on the same buffers
        (the real-time single frame-set case): `graph.replay()` re-runs the fused launch with
        one cudaGraphLaunch instead of the Python + C-ABI launch path.  Refill `iq` in place
        between replays; the taps land in the returned `out`."""
        iq, n_frames = self._check_iq(iq)
        if out is None:
            out = torch.empty(self.taps_shape(n_frames), dtype=torch.complex64, device=self.device)
        with torch.cuda.device(self.device):
            self.process(iq, out=out)                 # warm: the capture stream's resources
            torch.cuda.synchronize(self.device)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self.process(iq, out=out)
        return graph, out

    def pack(self, iq: torch.Tensor) -> torch.Tensor:
        """K2 alone: returns the packed 16-bit operand (K_pad columns; rows in 16-row blocks of
        8 links, Re rows then Im rows -- see pnce_workspace_bytes in include/pnce_b200.h)."""
        iq, n_frames = self._check_iq(iq)
        k_pad = -(-self.cfg.m // 64) * 64
        links = n_frames * self.cfg.n_batches * self.n_r
        rows = -(-links // 8) * 16
        tdt = torch.float16 if self.dtype == "fp16" else torch.bfloat16
        packed = torch.empty((rows, k_pad), dtype=tdt, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_pack_iq(self._plan, ctypes.c_void_p(iq.data_ptr()),
                                               ctypes.c_void_p(packed.data_ptr()), n_frames,
                                               _stream_ptr(self.device)))
        return packed

    def correlate(self, packed: torch.Tensor, n_frames: int, truth: torch.Tensor | None = None,
                  out: torch.Tensor | None = None, stats: torch.Tensor | None = None):
        """K3+K4 alone on a packed operand."""
        _same_device(self.device, packed=packed, out=out, truth=truth, stats=stats)
        if out is None:
            out = torch.empty(self.taps_shape(n_frames), dtype=torch.complex64, device=self.device)
        truth_ptr = ctypes.c_void_p(truth.data_ptr()) if truth is not None else None
        if truth is not None and stats is None:
            stats = torch.zeros((n_frames, 4), dtype=torch.float64, device=self.device)
        stats_ptr = ctypes.c_void_p(stats.data_ptr()) if stats is not None else None
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().pnce_correlate(self._plan, ctypes.c_void_p(packed.data_ptr()),
                                                 ctypes.c_void_p(out.data_ptr()), truth_ptr, stats_ptr,
                                                 n_frames, _stream_ptr(self.device)))
        return out, stats


def correlator_rows_for_plan(seq: PnSequence, plan: BatchPlan, cfg: PilotConfig, n_r: int,
                             dtype: str = "fp16") -> Correlator:
    """experiments.py:157-173 counterpart: the static device correlator for this plan."""
    if seq.spec is None:
        raise InvalidConfigError("device correlator needs a sequence generated from an LfsrSpec")
    if plan.m != cfg.m or plan.l != cfg.l:
        raise DimensionMismatchError("batch plan does not match the pilot configuration")
    return Correlator(seq.spec, cfg, n_r, dtype=dtype, device=seq.chips.device)


def _frames_to_iq(frames, cfg: PilotConfig) -> np.ndarray:
    """Host frames (list of (n_r, P+L-1) complex arrays or objects with .samples) -> f32 IQ.

    Same quantisation as the IQ file writer (iqfile.py:86-89)."""
    arrs = [np.asarray(getattr(f, "samples", f)) for f in frames]
    if len(arrs) != cfg.n_batches:
        raise DimensionMismatchError(f"{len(arrs)} frames for a plan of {cfg.n_batches} batches")
    n_r = arrs[0].shape[0]
    if any(a.shape[0] != n_r for a in arrs):
        raise DimensionMismatchError("frames disagree on n_r")
    if any(a.shape[-1] < cfg.c + cfg.m for a in arrs):
        raise FrameTooShortError(f"frame shorter than C+M={cfg.c + cfg.m}")
    s = cfg.samples_per_receiver
    iq = np.zeros((1, len(arrs), n_r, s, 2), dtype=np.float32)
    for b, a in enumerate(arrs):
        w = min(s, a.shape[-1])
        iq[0, b, :, :w, 0] = a.real[:, :w].astype(np.float32)
        iq[0, b, :, :w, 1] = a.imag[:, :w].astype(np.float32)
    return iq


def process_frames(seq: PnSequence, cfg: PilotConfig, plan: BatchPlan, frames, backend=None,
                   counters: WorkCounters | None = None, rows_per_batch: Correlator | None = None,
                   truth=None) -> CirEstimate:
    """experiments.py:176-208 on the device: CP removal, correlation, demux, 1/M.

    ``frames``: either the reference's per-batch list of (n_r, P+L-1) complex
    frames (host; copied to the device as f32 IQ) or a CUDA float32 IQ tensor
    (n_batches, n_r, P+L-1, 2) / (F, n_batches, n_r, P+L-1, 2).
    ``backend``: the reference's ``BackendConfig`` (ours in backend.py or pnce's own):
    reference64 / reference32 run the fused fp16 path, tensor16 runs the tensor16 mode
    with its chunk_len / accumulator (backend.py has the mapping and tolerances); or
    "fp16" / "bf16" for the fused path at that operand precision.  ``rows_per_batch``: a
    prebuilt Correlator (the static state the reference passes as rows_per_batch).
    A saturated (frame-set, batch) is scored as all-zero taps and counted as n_r * n_tx
    saturations, as the reference does (experiments.py:201-205).
    """
    mode = resolve_backend(backend, rows_per_batch.dtype if rows_per_batch is not None else None)
    single = True
    if isinstance(frames, torch.Tensor):
        iq = frames
        n_r = int(frames.shape[-3])
        single = frames.dim() == 4
    else:
        host = _frames_to_iq(frames, cfg)
        n_r = host.shape[2]
        iq = torch.from_numpy(host).to(seq.chips.device, non_blocking=False)
    corr = rows_per_batch
    if corr is None or corr.n_r != n_r or corr.dtype != mode.dtype or corr.cfg != cfg:
        corr = correlator_rows_for_plan(seq, plan, cfg, n_r, mode.dtype)
    truth_t = None
    if truth is not None:
        tt = getattr(truth, "taps", truth)
        truth_t = tt if isinstance(tt, torch.Tensor) else torch.from_numpy(np.asarray(tt, dtype=np.complex64))
        truth_t = truth_t.to(device=corr.device, dtype=torch.complex64)
        if truth_t.dim() == 3:
            truth_t = truth_t.unsqueeze(0)
    n_frames = 1 if single else int(iq.shape[0])
    # stats always: the saturation count (stats[:, 3]) comes with them
    stats = torch.zeros((n_frames, 4), dtype=torch.float64, device=corr.device)
    link_mse = None
    if mode.tensor16:
        taps, stats = corr.process_tensor16(iq, chunk_len=mode.chunk_len, accumulator=mode.accumulator,
                                            truth=truth_t, stats=stats)
    elif truth_t is not None:
        taps, stats, link_mse = corr.process_scored(iq, truth_t, stats=stats)
    else:
        taps, stats = corr.process(iq, stats=stats)
    if counters is not None:
        counters.samples_moved += n_frames * cfg.n_batches * n_r * cfg.p
        counters.macs += n_frames * cfg.n_t * cfg.l * cfg.m * n_r
    out_taps = taps[0] if single else taps
    saturations = int(round(float(stats[:, 3].sum().item())))
    if link_mse is not None and single:
        link_mse = link_mse[0]
    return CirEstimate(taps=out_taps, backend=mode.kind, norm=1.0 / cfg.m, saturations=saturations,
                       stats=stats if truth_t is not None else None, link_mse=link_mse)
