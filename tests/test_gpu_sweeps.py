"""Device sweeps against the reference's own sweep output."""

import math
import os

import numpy as np
import pytest
import torch

from oracle import pnce_oracle as O
from paper_2206_05506_b200 import sweeps as SW

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def oracle_source(pilot, n_r, l_nz, snr_db, chan_seed, noise_seed):
    """The reference's simulate_frame for these seeds (oracle restatement, pinned to the
    reference's IQ bytes by test_oracle.py)."""
    ocfg = O.Config(m=pilot.m, c=pilot.c, n_t=pilot.n_t, n_batch=pilot.n_batch, l=pilot.l, n_r=n_r)
    return O.simulate_frame(O.sequence_for_length(pilot.m), ocfg, l_nz, snr_db, chan_seed, noise_seed)


def db(a, b):
    return abs(10 * math.log10(a / b))


def test_snr_sweep_identical_inputs_match_reference_csv(dev):
    """With the reference's own frames (frame_source) every row matches the reference's
    run_snr_sweep CSV: counters exactly, MAE within 0.01 dB (draw for draw)."""
    with open(os.path.join(GOLD, "ref_snr_sweep.csv"), newline="") as fh:
        ref = SW.parse_csv(fh.read())
    cfg = SW.ExperimentConfig(n_t=4, n_r=4, pn_lengths=(63, 127), c=16, l=16, l_nz=(16,), n_batch=(1,),
                              snr_db=(-10.0, 10.0, 30.0), iterations=4, seed=0, record_latency=False)
    rows = SW.run_snr_sweep(cfg, device=dev, frame_source=oracle_source)
    assert len(rows) == len(ref)
    for a, b in zip(rows, ref):
        assert (a.m, a.snr_db, a.samples_moved, a.macs, a.saturations) == (b.m, b.snr_db, b.samples_moved, b.macs,
                                                                          b.saturations)
        assert db(a.mae, b.mae) <= 0.01, (a, b)


def test_table1_grid_draw_for_draw(dev):
    """The paper's Table I grid at cfg2 (SNR 0..30 dB step 5 x 50 iterations, seed 0) on the
    reference's own frames: every per-iteration MAE within 0.05 dB and every point within
    0.01 dB of the REAL reference's sweep (tests/golden/ref_cfg2_table1.csv)."""
    with open(os.path.join(GOLD, "ref_cfg2_table1.csv"), newline="") as fh:
        ref = SW.parse_csv(fh.read())
    cfg = SW.ExperimentConfig(n_t=16, n_r=16, pn_lengths=(255,), c=32, l=32, l_nz=(32,), n_batch=(4,),
                              snr_db=tuple(float(s) for s in range(0, 31, 5)), iterations=50, seed=0,
                              emit_per_iteration=True, record_latency=False)
    rows = SW.run_snr_sweep(cfg, device=dev, frame_source=oracle_source)
    assert len(rows) == len(ref) == 7 * 51
    worst_it = worst_pt = 0.0
    for a, b in zip(rows, ref):
        assert (a.experiment, a.snr_db, a.iterations, a.seed, a.samples_moved, a.macs, a.saturations) == \
               (b.experiment, b.snr_db, b.iterations, b.seed, b.samples_moved, b.macs, b.saturations)
        d = db(a.mae, b.mae)
        if a.experiment == "snr_sweep":
            worst_pt = max(worst_pt, d)
        else:
            worst_it = max(worst_it, d)
    assert worst_pt <= 0.01 and worst_it <= 0.05, (worst_pt, worst_it)


def test_snr_sweep_rows_match_reference_csv(dev):
    """Same grid, schema, seeds and counters as the reference's run_snr_sweep (4x4, M 63/127);
    MAE statistically equal (4 iterations per point on each side)."""
    with open(os.path.join(GOLD, "ref_snr_sweep.csv"), newline="") as fh:
        ref = SW.parse_csv(fh.read())
    cfg = SW.ExperimentConfig(n_t=4, n_r=4, pn_lengths=(63, 127), c=16, l=16, l_nz=(16,), n_batch=(1,),
                              snr_db=(-10.0, 10.0, 30.0), iterations=4, seed=0, record_latency=False)
    rows = SW.run_snr_sweep(cfg, device=dev)
    assert len(rows) == len(ref)
    for a, b in zip(rows, ref):
        assert (a.experiment, a.n_t, a.n_r, a.m, a.c, a.l, a.l_nz, a.n_batch, a.snr_db, a.iterations, a.seed,
                a.samples_moved, a.macs, a.saturations) == \
               (b.experiment, b.n_t, b.n_r, b.m, b.c, b.l, b.l_nz, b.n_batch, b.snr_db, b.iterations, b.seed,
                b.samples_moved, b.macs, b.saturations)
        assert a.backend == "tcgen05-fp16" and a.latency_s == 0.0
        assert abs(math.log(a.mae / b.mae)) < 0.25, (a, b)
    text = SW.render_csv(rows)                      # 9-digit rendering: stable after one round trip
    assert SW.render_csv(SW.parse_csv(text)) == text


def test_cfg2_mae_curve(dev):
    """cfg2 (16x16, M=255, L=C=32, N_b=4) MAE vs SNR with 64 iterations per point against
    the reference64 anchor (8 frame-sets per point): within 8 %."""
    gold = np.load(os.path.join(GOLD, "golden.npz"))
    snrs, mae_ref = gold["curve_snr"], gold["curve_mae32"].mean(axis=1)
    cfg = SW.ExperimentConfig(n_t=16, n_r=16, pn_lengths=(255,), c=32, l=32, l_nz=(32,), n_batch=(4,),
                              snr_db=tuple(float(s) for s in snrs), iterations=64, seed=0, emit_per_iteration=True)
    rows = SW.run_snr_sweep(cfg, device=dev)
    head = [r for r in rows if r.experiment == "snr_sweep"]
    per_it = [r for r in rows if r.experiment == "snr_sweep:iter"]
    assert len(head) == len(snrs) and len(per_it) == 64 * len(snrs)
    for r, want in zip(head, mae_ref):
        assert abs(r.mae / want - 1) < 0.08, (r.snr_db, r.mae, want)
        assert r.latency_s > 0
    # the head row is the mean of its per-iteration rows
    for k, r in enumerate(head):
        its = per_it[64 * k:64 * (k + 1)]
        assert math.isclose(r.mae, math.fsum(x.mae for x in its) / 64, rel_tol=1e-12)


def test_latency_bench_rows(dev):
    cfg = SW.ExperimentConfig(n_t=16, n_r=16, pn_lengths=(255, 511), c=32, l=32, l_nz=(32,), n_batch=(1, 4),
                              snr_db=(10.0,), iterations=1, seed=0)
    rep = SW.run_latency_bench(cfg, reps=3, warmup=1, device=dev)
    assert [(p.m, p.n_batch) for p in rep.points] == [(255, 1), (255, 4), (511, 1), (511, 4)]
    rows = SW.bench_rows(rep)
    assert all(r.experiment == "latency_bench" and r.mae == 0.0 and r.latency_s > 0 and r.iterations == 3
               for r in rows)
    assert rows[0].macs == 16 * 32 * 255 * 16 and rows[0].samples_moved == 16 * 16 * (32 + 255)
    text = SW.render_csv(rows)
    assert SW.render_csv(SW.parse_csv(text)) == text


def test_tensor16_sweep_matches_reference_csv(dev):
    """The reference's tensor16 sweep (BackendConfig(kind="tensor16", chunk_len=128,
    accumulator="binary16"), the paper's precision study) run on the tensor cores with the
    reference's own frames: same rows, backend column "tensor16", counters and saturations
    exact, every per-iteration MAE within 0.05 dB of the real reference's emulation
    (tests/golden/ref_t16_sweep.csv)."""
    from paper_2206_05506_b200.backend import BackendConfig
    with open(os.path.join(GOLD, "ref_t16_sweep.csv"), newline="") as fh:
        ref = SW.parse_csv(fh.read())
    cfg = SW.ExperimentConfig(n_t=16, n_r=16, pn_lengths=(255,), c=32, l=32, l_nz=(32,), n_batch=(4,),
                              snr_db=(0.0, 15.0, 30.0), iterations=6, seed=0, emit_per_iteration=True,
                              record_latency=False,
                              backend=BackendConfig(kind="tensor16", chunk_len=128, accumulator="binary16"))
    rows = SW.run_snr_sweep(cfg, device=dev, frame_source=oracle_source)
    assert len(rows) == len(ref) == 3 * 7
    worst = 0.0
    for a, b in zip(rows, ref):
        assert (a.experiment, a.backend, a.snr_db, a.iterations, a.seed, a.samples_moved, a.macs, a.saturations) == \
               (b.experiment, b.backend, b.snr_db, b.iterations, b.seed, b.samples_moved, b.macs, b.saturations)
        worst = max(worst, db(a.mae, b.mae))
    assert worst <= 0.05, worst
