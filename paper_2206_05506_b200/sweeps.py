"""Monte-Carlo sweeps on the device, sharded over GPUs.

Counterpart of the reference harness (pnce/experiments.py:45-97, 234-348) and its
fixed-schema CSV records (pnce/records.py:15-117): the same `ExperimentConfig` grid,
`SweepResult` rows and CSV bytes, with every sweep point computed on the GPU --
channel draws and pilot sweeps by the device synthesiser (synth.py), estimation and
MAE scoring by the fused correlator -- and the points of a grid distributed round-robin
over the ranks of a process group (NCCL/gloo), gathered in grid order on rank 0.

Per point and iteration the (channel, noise) seeds derive from the master seed and the
grid key exactly as the reference does (numpy SeedSequence, experiments.py:151-154).
By default they seed the device synthesiser's Philox streams, so MAE values are
statistically -- not draw-for-draw -- equivalent.  With a ``frame_source`` (the
reference's own `simulate_frame` output for those seeds: a host callable returning
(truth taps, per-batch frames), experiments.py:217-231) every iteration estimates exactly
the frames the reference would, so the curves match the reference's draw for draw; the
frames are quantised to f32 I/Q as the IQ-file writer does (iqfile.py:86-89).
`latency_s` is the device time per frame-set of the fused scored kernel.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from .errors import InvalidConfigError, SchemaMismatchError

DEFAULT_SNR_GRID_DB = tuple(float(s) for s in range(-10, 31, 5))

CSV_COLUMNS = ("experiment", "backend", "nt", "nr", "m", "c", "l", "l_nz", "n_batch", "snr_db", "iterations",
               "seed", "mae", "latency_s", "samples_moved", "macs", "saturations")


@dataclass(frozen=True)
class ExperimentConfig:
    """experiments.py:45-80.  ``backend``: "fp16" / "bf16" (operand dtype of the fused path) or
    the reference's ``BackendConfig`` (backend.py): reference64/32 run the fused fp16 path,
    tensor16 runs the tensor16 mode with its chunk_len / accumulator (the paper's §III-B
    precision study on real tensor cores); the CSV backend column is then the kind."""

    n_t: int = 16
    n_r: int = 16
    pn_lengths: tuple[int, ...] = (511, 1023, 2047)
    c: int = 64
    l: int = 64
    l_nz: tuple[int, ...] = (64,)
    n_batch: tuple[int, ...] = (1,)
    snr_db: tuple[float, ...] = DEFAULT_SNR_GRID_DB
    iterations: int = 50
    seed: int = 0
    backend: object = "fp16"
    f_s: float = 10e6
    emit_per_iteration: bool = False
    record_latency: bool = True

    def __post_init__(self):
        if self.iterations < 1:
            raise InvalidConfigError("iterations must be >= 1")
        for m in self.pn_lengths:
            degree = (m + 1).bit_length() - 1
            if (1 << degree) - 1 != m:
                raise InvalidConfigError(f"PN length {m} is not 2**k - 1")
        if not self.pn_lengths or not self.l_nz or not self.n_batch or not self.snr_db:
            raise InvalidConfigError("grid lists must be non-empty")


@dataclass(frozen=True)
class SweepResult:
    """experiments.py:83-97: one CSV row."""

    experiment: str
    backend: str
    n_t: int
    n_r: int
    m: int
    c: int
    l: int
    l_nz: int
    n_batch: int
    snr_db: float
    iterations: int
    seed: int
    mae: float
    latency_s: float
    samples_moved: int
    macs: int
    saturations: int


def derive_seeds(master: int, *key: int) -> tuple[int, int]:
    """experiments.py:151-154: (channel seed, noise seed) from SeedSequence([master, *key])."""
    chan, noise = np.random.SeedSequence([master, *key]).generate_state(2, dtype=np.uint64)
    return int(chan), int(noise)


# ---------------------------------------------------------------- records (records.py)
def _fmt(x: float) -> str:
    return f"{x:.9g}"


def render_row(r: SweepResult) -> str:
    return ",".join([r.experiment, r.backend, str(r.n_t), str(r.n_r), str(r.m), str(r.c), str(r.l), str(r.l_nz),
                     str(r.n_batch), _fmt(r.snr_db), str(r.iterations), str(r.seed), _fmt(r.mae),
                     _fmt(r.latency_s), str(r.samples_moved), str(r.macs), str(r.saturations)])


def render_csv(rows: Iterable[SweepResult]) -> str:
    return "\n".join([",".join(CSV_COLUMNS), *(render_row(r) for r in rows)]) + "\n"


def parse_csv(text: str) -> list[SweepResult]:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise SchemaMismatchError("empty CSV: header row missing")
    header = tuple(lines[0].split(","))
    if header != CSV_COLUMNS:
        raise SchemaMismatchError(f"header {header} != expected {CSV_COLUMNS}")
    out = []
    for ln in lines[1:]:
        p = ln.split(",")
        if len(p) != len(CSV_COLUMNS):
            raise SchemaMismatchError(f"row has {len(p)} fields, expected {len(CSV_COLUMNS)}")
        out.append(SweepResult(p[0], p[1], int(p[2]), int(p[3]), int(p[4]), int(p[5]), int(p[6]), int(p[7]),
                               int(p[8]), float(p[9]), int(p[10]), int(p[11]), float(p[12]), float(p[13]),
                               int(p[14]), int(p[15]), int(p[16])))
    return out


def write_csv(path, rows: Sequence[SweepResult]) -> None:
    with open(path, "w", newline="") as fh:
        fh.write(render_csv(rows))


def read_csv(path) -> list[SweepResult]:
    with open(path) as fh:
        return parse_csv(fh.read())


# ---------------------------------------------------------------- grid + sharding
@dataclass(frozen=True)
class SweepPoint:
    experiment: str
    m: int
    n_batch: int
    l_nz: int
    snr_db: float
    si: int


def snr_sweep_points(cfg: ExperimentConfig) -> list[SweepPoint]:
    """run_snr_sweep (experiments.py:299-322) grid order."""
    return [SweepPoint("snr_sweep", m, nb, cfg.l_nz[0], snr, si)
            for m in cfg.pn_lengths for nb in cfg.n_batch for si, snr in enumerate(cfg.snr_db)]


def tap_sweep_points(cfg: ExperimentConfig) -> list[SweepPoint]:
    """run_tap_sweep (experiments.py:325-348) grid order."""
    m, nb = cfg.pn_lengths[0], cfg.n_batch[0]
    return [SweepPoint("tap_sweep", m, nb, lnz, snr, si) for lnz in cfg.l_nz for si, snr in enumerate(cfg.snr_db)]


def shard(points: Sequence, rank: int, world: int) -> list[tuple[int, object]]:
    """Round-robin (index, point) assignment: neighbouring grid points (similar cost) spread."""
    return [(i, p) for i, p in enumerate(points) if i % world == rank]


def _gather_rows(indexed_rows: list[tuple[int, list[SweepResult]]], group=None) -> list[SweepResult] | None:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [r for _, rows in sorted(indexed_rows, key=lambda x: x[0]) for r in rows]
    world = dist.get_world_size(group)
    parts = [None] * world if dist.get_rank(group) == 0 else None
    dist.gather_object(indexed_rows, parts, dst=0, group=group)
    if dist.get_rank(group) != 0:
        return None
    merged = [x for part in parts for x in part]
    return [r for _, rows in sorted(merged, key=lambda x: x[0]) for r in rows]


# ---------------------------------------------------------------- device evaluation
_CORR_CACHE: dict = {}


def _mode(cfg: ExperimentConfig):
    from .backend import resolve
    return resolve(cfg.backend)


def _correlator(cfg: ExperimentConfig, m: int, n_batch: int, device: torch.device):
    from .estimator import Correlator
    from .pilots import PilotConfig
    from .pn import default_spec
    dtype = _mode(cfg).dtype
    key = (m, n_batch, cfg.n_t, cfg.n_r, cfg.c, cfg.l, dtype, str(device))
    if key not in _CORR_CACHE:
        pilot = PilotConfig(m=m, c=cfg.c, n_t=cfg.n_t, n_batch=n_batch, l=cfg.l, f_s=cfg.f_s)
        _CORR_CACHE[key] = Correlator(default_spec((m + 1).bit_length() - 1), pilot, cfg.n_r,
                                      dtype=dtype, device=device)
    return _CORR_CACHE[key]


def _host_frames(frame_source, corr, pt: SweepPoint, seeds) -> tuple[torch.Tensor, torch.Tensor]:
    """Frames of every iteration from a host frame source -> pinned (truth c64, iq f32)."""
    import numpy as np
    from .estimator import _frames_to_iq
    it_n = len(seeds)
    h = torch.empty(corr.taps_shape(it_n), dtype=torch.complex64).pin_memory()
    iq = torch.empty(corr.iq_shape(it_n), dtype=torch.float32).pin_memory()
    for it, (cs, ns) in enumerate(seeds):
        truth, frames = frame_source(corr.cfg, corr.n_r, pt.l_nz, pt.snr_db, cs, ns)
        truth = np.asarray(getattr(truth, "taps", truth))
        if truth.shape != tuple(corr.taps_shape(1)[1:]):
            raise SchemaMismatchError(f"frame source truth shape {truth.shape} != {corr.taps_shape(1)[1:]}")
        h[it] = torch.from_numpy(truth.astype(np.complex64))
        iq[it] = torch.from_numpy(_frames_to_iq(frames, corr.cfg)[0])
    return h, iq


def evaluate_point(cfg: ExperimentConfig, pt: SweepPoint, device: torch.device,
                   frame_source=None) -> list[SweepResult]:
    """_sweep_point (experiments.py:234-296) on the device: all iterations as one batch.

    ``frame_source(pilot, n_r, l_nz, snr_db, chan_seed, noise_seed) -> (truth, frames)``:
    host frames instead of the device synthesiser (see the module docstring)."""
    from . import synth
    corr = _correlator(cfg, pt.m, pt.n_batch, device)
    it_n = cfg.iterations
    seeds = [derive_seeds(cfg.seed, pt.m, pt.n_batch, pt.l_nz, pt.si, it) for it in range(it_n)]
    if frame_source is not None:
        h_host, iq_host = _host_frames(frame_source, corr, pt, seeds)
        h = h_host.to(device, non_blocking=True)
        iq = iq_host.to(device, non_blocking=True)
    else:
        h = torch.empty(corr.taps_shape(it_n), dtype=torch.complex64, device=device)
        iq = torch.empty(corr.iq_shape(it_n), dtype=torch.float32, device=device)
        for it, (cs, ns) in enumerate(seeds):
            h[it:it + 1] = synth.draw_channel(corr, 1, l_nz=pt.l_nz, seed=cs)
            synth.simulate_frames(corr, h[it:it + 1], pt.snr_db, seed=ns, out=iq[it:it + 1])
    stream = torch.cuda.current_stream(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mode = _mode(cfg)
    ev0.record(stream)
    if mode.tensor16:   # zeroed + counted saturated batches, sums over the returned taps
        _, stats = corr.process_tensor16(iq, chunk_len=mode.chunk_len, accumulator=mode.accumulator, truth=h)
    else:
        _, stats, _ = corr.process_scored(iq, h)
    ev1.record(stream)
    torch.cuda.synchronize(device)
    per_frame = (ev0.elapsed_time(ev1) / 1e3) / it_n if cfg.record_latency else 0.0
    n_taps = cfg.n_r * cfg.n_t * cfg.l
    maes = (stats[:, 0] / n_taps).tolist()
    sats = stats[:, 3].round().long().tolist()   # n_r * n_tx per saturated batch (experiments.py:201-205)
    pil = corr.cfg
    samples_moved = pil.n_batches * cfg.n_r * pil.p
    macs = cfg.n_t * cfg.l * pt.m * cfg.n_r
    backend = mode.kind

    def row(name, iters, seed, mae_v, lat, sat):
        return SweepResult(name, backend, cfg.n_t, cfg.n_r, pt.m, cfg.c, cfg.l, pt.l_nz, pt.n_batch, pt.snr_db,
                           iters, seed, mae_v, lat, samples_moved, macs, sat)

    rows = [row(pt.experiment, it_n, cfg.seed, math.fsum(maes) / it_n, per_frame, int(sum(sats)))]
    if cfg.emit_per_iteration:
        rows += [row(f"{pt.experiment}:iter", 1, seeds[it][0], maes[it], per_frame, sats[it]) for it in range(it_n)]
    return rows


def _run(cfg: ExperimentConfig, points: Sequence[SweepPoint], device=None, group=None,
         frame_source=None) -> list[SweepResult] | None:
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if device is None:
        device = torch.device("cuda", int(os.environ.get("LOCAL_RANK", torch.cuda.current_device())))
    mine = [(i, evaluate_point(cfg, pt, device, frame_source)) for i, pt in shard(points, rank, world)]
    return _gather_rows(mine, group)


def run_snr_sweep(cfg: ExperimentConfig, device=None, group=None, frame_source=None) -> list[SweepResult] | None:
    """MAE vs SNR over the (PN length, N_batch) grid; rows on rank 0 (None elsewhere)."""
    return _run(cfg, snr_sweep_points(cfg), device, group, frame_source)


def run_tap_sweep(cfg: ExperimentConfig, device=None, group=None, frame_source=None) -> list[SweepResult] | None:
    """MAE vs SNR while varying the tap count (M, N_batch fixed to the grid heads)."""
    return _run(cfg, tap_sweep_points(cfg), device, group, frame_source)


@dataclass
class BenchPoint:
    """experiments.py:112-131: latency statistics of one (M, N_batch) point."""

    backend: str
    n_t: int
    n_r: int
    m: int
    c: int
    l: int
    l_nz: int
    n_batch: int
    snr_db: float
    reps: int
    mean_s: float
    std_s: float
    median_s: float
    samples_moved: int
    macs: int
    seed: int
    times_s: tuple = ()


@dataclass
class LatencyReport:
    points: list


def run_latency_bench(cfg: ExperimentConfig, reps: int = 10, warmup: int = 2, device=None) -> LatencyReport:
    """experiments.py:351-408 on the device: per-frame-set processing time (CUDA events around
    one fused launch on a resident synthesised frame-set) over the (M, N_batch) grid."""
    import statistics

    from . import synth
    if reps < 1:
        raise InvalidConfigError("reps must be >= 1")
    if device is None:
        device = torch.device("cuda", int(os.environ.get("LOCAL_RANK", torch.cuda.current_device())))
    points = []
    for m in cfg.pn_lengths:
        for nb in cfg.n_batch:
            corr = _correlator(cfg, m, nb, device)
            cs, ns = derive_seeds(cfg.seed, m, nb, 0)
            h = synth.draw_channel(corr, 1, l_nz=cfg.l_nz[0], seed=cs)
            iq = synth.simulate_frames(corr, h, cfg.snr_db[0], seed=ns)
            taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64, device=device)
            times = []
            for rep in range(warmup + reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(torch.cuda.current_stream(device))
                if _mode(cfg).tensor16:
                    m16 = _mode(cfg)
                    corr.process_tensor16(iq, chunk_len=m16.chunk_len, accumulator=m16.accumulator, out=taps)
                else:
                    corr.process(iq, out=taps)
                e1.record(torch.cuda.current_stream(device))
                torch.cuda.synchronize(device)
                if rep >= warmup:
                    times.append(e0.elapsed_time(e1) / 1e3)
            pil = corr.cfg
            points.append(BenchPoint(_mode(cfg).kind, cfg.n_t, cfg.n_r, m, cfg.c, cfg.l, cfg.l_nz[0], nb,
                                     cfg.snr_db[0], len(times), statistics.fmean(times),
                                     statistics.stdev(times) if len(times) > 1 else 0.0, statistics.median(times),
                                     pil.n_batches * cfg.n_r * pil.p, cfg.n_t * cfg.l * m * cfg.n_r, cfg.seed,
                                     tuple(times)))
    return LatencyReport(points=points)


def bench_rows(report: LatencyReport, record_latency: bool = True) -> list[SweepResult]:
    """experiments.py:410-435: CSV-schema rows (mae column zeroed)."""
    return [SweepResult("latency_bench", p.backend, p.n_t, p.n_r, p.m, p.c, p.l, p.l_nz, p.n_batch, p.snr_db, p.reps,
                        p.seed, 0.0, p.mean_s if record_latency else 0.0, p.samples_moved, p.macs, 0)
            for p in report.points]


def main(argv=None) -> int:
    """`python -m paper_2206_05506_b200.sweeps` (torchrun for several GPUs): the reference CLI's
    `snr-sweep` / `tap-sweep` on the device, CSV on rank 0."""
    import argparse

    import torch.distributed as dist
    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("experiment", choices=["snr", "tap", "bench"])
    ap.add_argument("--out", default="-")
    ap.add_argument("--nt", type=int, default=16)
    ap.add_argument("--nr", type=int, default=16)
    ap.add_argument("--m", type=int, nargs="+", default=[511, 1023, 2047])
    ap.add_argument("--c", type=int, default=64)
    ap.add_argument("--l", type=int, default=64)
    ap.add_argument("--l-nz", type=int, nargs="+", default=None)
    ap.add_argument("--n-batch", type=int, nargs="+", default=[1])
    ap.add_argument("--snr", type=float, nargs="+", default=list(DEFAULT_SNR_GRID_DB))
    ap.add_argument("--iterations", type=int, default=50)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--per-iteration", action="store_true")
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and not dist.is_initialized():
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    cfg = ExperimentConfig(n_t=a.nt, n_r=a.nr, pn_lengths=tuple(a.m), c=a.c, l=a.l,
                           l_nz=tuple(a.l_nz or [a.l]), n_batch=tuple(a.n_batch), snr_db=tuple(a.snr),
                           iterations=a.iterations, seed=a.seed, backend=a.dtype, emit_per_iteration=a.per_iteration)
    if a.experiment == "bench":
        rank0 = not dist.is_initialized() or dist.get_rank() == 0
        rows = bench_rows(run_latency_bench(cfg)) if rank0 else None
    else:
        rows = (run_snr_sweep if a.experiment == "snr" else run_tap_sweep)(cfg)
    if rows is not None:
        text = render_csv(rows)
        if a.out == "-":
            print(text, end="")
        else:
            with open(a.out, "w", newline="") as fh:
                fh.write(text)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
