"""Multi-GPU plumbing for the estimator: one process per GPU.

Two splits, both with no data-path collective inside the estimation:

* frames -- frame-sets are independent (separate channel/noise draws,
  experiments.py:247-253): ranks take contiguous frame ranges (`frame_shard`);
  throughput scales with the rank count (weak scaling).
* antennas -- within a frame-set the receivers are independent columns of the
  correlation (estimator.py:78-79), the paper's own multi-GPU scheme: N_r / N_server
  receive antennas per GPU, then an all-gather of the CIRs (PAPER.md:150-153,
  `antenna_shard` + `allgather_csi`).  This shortens one frame-set's latency.

The collectives are the ones the north star names: error statistics are all-reduced
(a few float64s per frame-set), CSI is gathered (to one rank along frames, to all
ranks along antennas).  The backend is whatever the process group uses: NCCL over
NVLink on the GPU box; gloo for the CPU tests and for several ranks sharing one GPU
(gloo collectives run on host copies of CUDA tensors).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import DimensionMismatchError, InvalidConfigError


def frame_shard(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) frame range of ``rank``; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidConfigError(f"rank {rank} outside world of {world}")
    if n_frames < 0:
        raise DimensionMismatchError("n_frames < 0")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def antenna_shard(n_r: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [r0, r1) receive-antenna range of ``rank`` (the paper's N_r / N_server
    per GPU); sizes differ by at most one.  Every rank needs >= 1."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidConfigError(f"rank {rank} outside world of {world}")
    if n_r < world:
        raise InvalidConfigError(f"{n_r} receive antennas cannot be split over {world} ranks")
    return frame_shard(n_r, rank, world)


def _world(group) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def _host_collectives(group) -> bool:
    """gloo: run collectives on host copies (its CUDA support is partial)."""
    return dist.get_backend(group) == "gloo"


def allgather_csi(taps: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's receiver slice (F, n_r_rank, n_t, L) into the full
    (F, n_r, n_t, L) CSI on EVERY rank, receivers in rank order (PAPER.md:153 Allgather()).
    Slices may differ by one receiver (antenna_shard); they are padded for the collective."""
    world = _world(group)
    if world == 1:
        return taps
    dev = taps.device
    host = _host_collectives(group)
    cnt = torch.tensor([taps.shape[1]], dtype=torch.int64, device="cpu" if host else dev)
    cnts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt, group=group)
    cnts = [int(c.item()) for c in cnts]
    width = max(cnts)
    shape = (taps.shape[0], width) + tuple(taps.shape[2:])
    pad = torch.zeros(shape, dtype=taps.dtype, device="cpu" if host else dev)
    pad[:, : taps.shape[1]] = taps.to(pad.device)
    send = torch.view_as_real(pad) if pad.is_complex() else pad
    bufs = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(bufs, send.contiguous(), group=group)
    parts = [torch.view_as_complex(b) if pad.is_complex() else b for b in bufs]
    return torch.cat([p[:, :c] for p, c in zip(parts, cnts)], dim=1).to(dev)


class CsiGather:
    """The antenna split with the CSI all-gather fused into the estimation epilogue
    (PAPER.md:150-153): every rank allocates the full (F, n_r, n_t, L) CSI once, the ranks
    exchange CUDA-IPC handles of it, and each rank's launch (`Correlator.process_gather`)
    stores its receivers' taps straight into every rank's buffer -- NVLink stores from the
    kernel instead of a separate all-gather.  `run` is asynchronous; `wait` synchronises the
    stream and barriers the group, after which `csi` holds the gathered CSI on every rank."""

    def __init__(self, corr, n_r_total: int, n_frames: int, group=None):
        from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor

        self.group = group
        self.world = _world(group)
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.corr = corr
        self.r0, r1 = antenna_shard(n_r_total, self.rank, self.world)
        if r1 - self.r0 != corr.n_r:
            raise DimensionMismatchError(f"rank {self.rank} owns {r1 - self.r0} receivers, its correlator {corr.n_r}")
        if self.world > 8:
            raise InvalidConfigError("the fused gather addresses at most 7 peers")
        self.csi = torch.zeros((n_frames, n_r_total, corr.cfg.n_t, corr.cfg.l), dtype=torch.complex64,
                               device=corr.device)
        self.peers = []
        if self.world > 1:
            torch.cuda.synchronize(corr.device)
            mine = reduce_tensor(self.csi)[1]
            handles = [None] * self.world
            dist.all_gather_object(handles, mine, group=group)
            # open the peers' buffers; every rank must succeed (and reach each peer's device
            # directly) before any kernel stores into them -- agreed collectively, so all
            # ranks either proceed or raise together
            err = ""
            try:
                me = corr.device.index
                for i, h in enumerate(handles):
                    if i == self.rank:
                        continue
                    pdev = torch.device(h[6]).index if not isinstance(h[6], int) else h[6]
                    if pdev != me and not torch.cuda.can_device_access_peer(me, pdev):
                        raise InvalidConfigError(f"cuda:{me} cannot access cuda:{pdev} directly")
                    self.peers.append(rebuild_cuda_tensor(*h))
            except Exception as exc:  # noqa: BLE001 -- reported collectively below
                err = f"rank {self.rank}: {type(exc).__name__}: {exc}"
            errs = [None] * self.world
            dist.all_gather_object(errs, err, group=group)
            bad = [e for e in errs if e]
            if bad:
                self.peers = []
                raise InvalidConfigError("fused CSI gather unavailable: " + bad[0])

    def run(self, iq_part: torch.Tensor) -> torch.Tensor:
        return self.corr.process_gather(iq_part, self.csi, self.r0, self.peers)

    def wait(self) -> torch.Tensor:
        torch.cuda.synchronize(self.corr.device)
        if self.world > 1:
            dist.barrier(group=self.group)
        return self.csi

    def close(self) -> None:
        """Release the peer mappings (every rank, before any of them exits)."""
        self.peers = []
        torch.cuda.synchronize(self.corr.device)
        torch.cuda.ipc_collect()
        if self.world > 1:
            dist.barrier(group=self.group)


def reduce_frame_stats(stats: torch.Tensor, group=None) -> torch.Tensor:
    """Antenna split: each rank's per-frame stats (F, 4) cover its receivers only; the
    all-reduced sum is the frame-set's {sum|e|, sum|e|^2, non-finite, saturations}."""
    if stats.dim() != 2 or stats.shape[1] != 4:
        raise DimensionMismatchError(f"stats must be (F, 4), got {tuple(stats.shape)}")
    out = stats.to(torch.float64).clone()
    if _world(group) > 1:
        host = _host_collectives(group)
        buf = out.cpu() if host else out
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        out = buf.to(stats.device)
    return out


def reduce_stats(stats: torch.Tensor | None, group=None) -> torch.Tensor:
    """Sum this rank's per-frame error statistics (F, 4) into global totals (4,) float64.

    Totals are {sum|e|, sum|e|^2, non-finite taps, saturations}; every rank gets the result.
    """
    if stats is None:
        raise InvalidConfigError("no statistics to reduce (estimate without truth)")
    if stats.dim() != 2 or stats.shape[1] != 4:
        raise DimensionMismatchError(f"stats must be (F, 4), got {tuple(stats.shape)}")
    total = stats.to(torch.float64).sum(dim=0)
    if _world(group) > 1:
        buf = total.cpu() if _host_collectives(group) else total
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        total = buf.to(stats.device)
    return total


def global_metrics(stats: torch.Tensor, taps_per_frame: int, n_frames_total: int, group=None) -> dict:
    """MAE (metrics.py:19-25) and MSE over all ranks' frame-sets."""
    total = reduce_stats(stats, group)
    n = float(taps_per_frame) * float(n_frames_total)
    return {"mae": float(total[0]) / n, "mse": float(total[1]) / n, "nonfinite": int(total[2]),
            "saturations": int(total[3])}


def gather_taps(taps: torch.Tensor, dst: int = 0, group=None) -> torch.Tensor | None:
    """Gather every rank's CSI (F_rank, n_r, n_t, L) on ``dst`` in rank order (frame order).

    Ranks may hold different frame counts (frame_shard); shards are padded to the
    largest count for the collective and trimmed on ``dst``.  Returns None elsewhere.
    """
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return taps
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = taps.device
    if _host_collectives(group):
        taps = taps.cpu()
    count = torch.tensor([taps.shape[0]], dtype=torch.int64, device=taps.device)
    counts = [torch.zeros_like(count) for _ in range(world)]
    dist.all_gather(counts, count, group=group)
    counts = [int(c.item()) for c in counts]
    width = max(counts)
    padded = torch.zeros((width,) + tuple(taps.shape[1:]), dtype=taps.dtype, device=taps.device)
    padded[: taps.shape[0]] = taps
    # complex tensors travel as their real view
    send = torch.view_as_real(padded) if padded.is_complex() else padded
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    parts = [torch.view_as_complex(b) if padded.is_complex() else b for b in bufs]
    return torch.cat([p[:c] for p, c in zip(parts, counts)]).to(dev)


def max_over_ranks(values, group=None) -> list[float]:
    """Element-wise max of a few host floats over the ranks (device timings)."""
    t = torch.tensor([float(v) for v in values], dtype=torch.float64)
    if _world(group) > 1:
        if not _host_collectives(group):
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(x) for x in t.cpu().tolist()]
