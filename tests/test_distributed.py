"""Multi-process (gloo, world_size 2, CPU) tests of the frame sharding and the stats
collectives that the multi-GPU bench uses over NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_05506_b200 import distributed as D


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        start, stop = D.frame_shard(n_frames, rank, world)
        # deterministic per-frame "statistics" and "taps" for the frames this rank owns
        frames = torch.arange(start, stop, dtype=torch.float64)
        stats = torch.stack([frames, frames * frames, torch.zeros_like(frames), torch.zeros_like(frames)], dim=1)
        total = D.reduce_stats(stats)
        taps = (torch.arange(start, stop, dtype=torch.float32).view(-1, 1, 1, 1)
                * torch.ones(1, 2, 3, 4)).to(torch.complex64)
        gathered = D.gather_taps(taps, dst=0)
        out[rank] = {"range": (start, stop), "total": total.tolist(),
                     "gathered": None if gathered is None else gathered.real[:, 0, 0, 0].tolist()}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [0, 1, 7, 10])
def test_frame_shard_partition(n_frames):
    for world in (1, 2, 3, 8):
        ranges = [D.frame_shard(n_frames, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n_frames
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        sizes = [b - a for a, b in ranges]
        assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_reduce_and_gather():
    world, n_frames = 2, 7
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_frames, out), nprocs=world, join=True)
    want = [sum(range(n_frames)), sum(i * i for i in range(n_frames)), 0.0, 0.0]
    for r in range(world):
        assert out[r]["total"] == want                      # every rank holds the global totals
    covered = sorted(i for r in range(world) for i in range(*out[r]["range"]))
    assert covered == list(range(n_frames))                 # each frame-set exactly once
    assert out[0]["gathered"] == [float(i) for i in range(n_frames)]   # CSI in frame order
    assert out[1]["gathered"] is None


def test_single_process_passthrough():
    stats = torch.tensor([[1.0, 2.0, 0.0, 0.0], [3.0, 4.0, 1.0, 0.0]], dtype=torch.float64)
    assert D.reduce_stats(stats).tolist() == [4.0, 6.0, 1.0, 0.0]
    m = D.global_metrics(stats, taps_per_frame=2, n_frames_total=2)
    assert m == {"mae": 1.0, "mse": 1.5, "nonfinite": 1, "saturations": 0}


@pytest.mark.parametrize("n_r", [2, 5, 64, 128])
def test_antenna_shard_partition(n_r):
    for world in (1, 2, 3, 8):
        if n_r < world:
            with pytest.raises(D.InvalidConfigError):
                D.antenna_shard(n_r, 0, world)
            continue
        ranges = [D.antenna_shard(n_r, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n_r
        assert all(a[1] == b[0] and b[1] > b[0] for a, b in zip(ranges, ranges[1:]))


def _antenna_worker(rank, world, port, n_r, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, r1 = D.antenna_shard(n_r, rank, world)
        # synthetic "CSI" whose value encodes (frame, receiver, transmitter, lag)
        f, t, l = 3, 4, 5
        full = torch.arange(f * n_r * t * l, dtype=torch.float32).view(f, n_r, t, l)
        full = torch.complex(full, -full)
        got = D.allgather_csi(full[:, r0:r1].contiguous())
        stats = torch.zeros((f, 4), dtype=torch.float64)
        stats[:, 0] = torch.arange(f) * 10 + rank
        stats[:, 3] = r1 - r0
        red = D.reduce_frame_stats(stats)
        t_max = D.max_over_ranks([rank + 0.5, -rank])
        out[rank] = {"equal": bool(torch.equal(got, full)), "stats": red.tolist(), "max": t_max}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_r", [6, 7])
def test_gloo_world3_antenna_allgather(n_r):
    """The paper's split: receiver slices -> full CSI on every rank, in
    receiver order, also with uneven slices; per-frame stats summed over the slices."""
    world = 3
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_antenna_worker, args=(world, _free_port(), n_r, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r]["equal"]
        assert out[r]["stats"] == [[30.0 * k + 3.0, 0.0, 0.0, float(n_r)] for k in range(3)]
        assert out[r]["max"] == [2.5, 0.0]
