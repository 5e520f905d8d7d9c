"""Multi-GPU plumbing for the estimator: one process per GPU.

Frame-sets are independent (separate channel/noise draws, experiments.py:247-253),
so the hot path shards them contiguously across ranks with no data-path
collective.  The only collectives are the ones the north star names: the
per-rank error statistics are all-reduced (a few float64s) and, optionally, the
CSI is gathered to one rank.  The backend is whatever the process group uses:
NCCL over NVLink on the GPU box, gloo for the CPU tests.
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


def reduce_stats(stats: torch.Tensor | None, group=None) -> torch.Tensor:
    """Sum this rank's per-frame error statistics (F, 4) into global totals (4,) float64.

    Totals are {sum|e|, sum|e|^2, non-finite taps, 0}; every rank gets the result.
    """
    if stats is None:
        raise InvalidConfigError("no statistics to reduce (estimate without truth)")
    if stats.dim() != 2 or stats.shape[1] != 4:
        raise DimensionMismatchError(f"stats must be (F, 4), got {tuple(stats.shape)}")
    total = stats.to(torch.float64).sum(dim=0)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
    return total


def global_metrics(stats: torch.Tensor, taps_per_frame: int, n_frames_total: int, group=None) -> dict:
    """MAE (metrics.py:19-25) and MSE over all ranks' frame-sets."""
    total = reduce_stats(stats, group)
    n = float(taps_per_frame) * float(n_frames_total)
    return {"mae": float(total[0]) / n, "mse": float(total[1]) / n, "nonfinite": int(total[2])}


def gather_taps(taps: torch.Tensor, dst: int = 0, group=None) -> torch.Tensor | None:
    """Gather every rank's CSI (F_rank, n_r, n_t, L) on ``dst`` in rank order (frame order).

    Ranks may hold different frame counts (frame_shard); shards are padded to the
    largest count for the collective and trimmed on ``dst``.  Returns None elsewhere.
    """
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return taps
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
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
    return torch.cat([p[:c] for p, c in zip(parts, counts)])
