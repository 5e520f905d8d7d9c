"""Sweep records and sharding on CPU: CSV bytes against the real
reference's renderer, grid order and seeds against the reference, gloo world-2 gather."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pnce_oracle as O
from paper_2206_05506_b200 import sweeps as SW
from paper_2206_05506_b200.errors import InvalidConfigError, SchemaMismatchError

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read(name):
    with open(os.path.join(GOLD, name), newline="") as fh:
        return fh.read()


def test_csv_bytes_match_reference_renderer():
    for name in ("ref_records.csv", "ref_snr_sweep.csv"):
        text = _read(name)
        assert SW.render_csv(SW.parse_csv(text)) == text


def test_csv_schema_errors():
    with pytest.raises(SchemaMismatchError):
        SW.parse_csv("")
    with pytest.raises(SchemaMismatchError):
        SW.parse_csv("a,b\n1,2\n")
    with pytest.raises(SchemaMismatchError):
        SW.parse_csv(",".join(SW.CSV_COLUMNS) + "\n1,2,3\n")


def test_grid_order_and_counters_match_reference():
    ref = SW.parse_csv(_read("ref_snr_sweep.csv"))
    cfg = SW.ExperimentConfig(n_t=4, n_r=4, pn_lengths=(63, 127), c=16, l=16, l_nz=(16,), n_batch=(1,),
                              snr_db=(-10.0, 10.0, 30.0), iterations=4, seed=0, record_latency=False)
    pts = SW.snr_sweep_points(cfg)
    assert [(p.m, p.n_batch, p.l_nz, p.snr_db) for p in pts] == [(r.m, r.n_batch, r.l_nz, r.snr_db) for r in ref]
    tap = SW.tap_sweep_points(SW.ExperimentConfig(pn_lengths=(127,), l_nz=(4, 16), snr_db=(0.0, 10.0)))
    assert [(p.l_nz, p.snr_db, p.si) for p in tap] == [(4, 0.0, 0), (4, 10.0, 1), (16, 0.0, 0), (16, 10.0, 1)]


def test_seeds_match_reference_derivation():
    for key in [(63, 1, 16, 0, 0), (1023, 8, 64, 4, 49), (255, 4, 32, 2, 7)]:
        assert SW.derive_seeds(0, *key) == O.derive_seeds(0, *key)
        assert SW.derive_seeds(5, *key) == O.derive_seeds(5, *key)


def test_config_validation():
    with pytest.raises(InvalidConfigError):
        SW.ExperimentConfig(iterations=0)
    with pytest.raises(InvalidConfigError):
        SW.ExperimentConfig(pn_lengths=(100,))
    with pytest.raises(InvalidConfigError):
        SW.ExperimentConfig(snr_db=())


def test_shard_covers_grid_once():
    pts = list(range(11))
    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i, _ in SW.shard(pts, r, world))
        assert got == pts


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = SW.ExperimentConfig(n_t=4, n_r=4, pn_lengths=(63, 127), c=16, l=16, snr_db=(-10.0, 0.0, 10.0),
                                  iterations=2)
        pts = SW.snr_sweep_points(cfg)

        def fake_eval(i, pt):   # stands in for the device evaluation; tags the computing rank
            return [SW.SweepResult(pt.experiment, f"rank{rank}", 4, 4, pt.m, 16, 16, pt.l_nz, pt.n_batch, pt.snr_db,
                                   2, 0, float(i), 0.0, 0, 0, 0)]
        rows = SW._gather_rows([(i, fake_eval(i, pt)) for i, pt in SW.shard(pts, rank, world)])
        out[rank] = None if rows is None else [(r.m, r.snr_db, r.mae, r.backend) for r in rows]
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sweep_gather():
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[1] is None
    rows = out[0]
    assert [r[2] for r in rows] == [float(i) for i in range(6)]              # grid order restored
    assert {r[3] for r in rows} == {"rank0", "rank1"}                        # both ranks computed points
    assert [(r[0], r[1]) for r in rows] == [(m, s) for m in (63, 127) for s in (-10.0, 0.0, 10.0)]
