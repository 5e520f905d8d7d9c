"""The multi-GPU paths executed for real: two ranks (gloo process group) sharing cuda:0
(the GPU box has one GPU, so the ranks share it -- no kernel waits on
another rank, so sharing is safe).  Frame-sharded and antenna-sharded (N_r per rank,
PAPER.md:150-153) taps equal the single-rank taps bit for bit, and the all-reduced
statistics equal the single-rank sums -- the analogue of the reference's thread-count
invariance test (test_experiments.py:172-177).  The antenna split also runs with the CSI
all-gather fused into the epilogue (`CsiGather`: each rank's kernel stores its receivers'
taps into every rank's CSI buffer through CUDA-IPC mappings) and must give the same CSI."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(P, S, corr, n_frames):
    h = S.draw_channel(corr, n_frames, seed=11)
    iq = S.simulate_frames(corr, h, 10.0, seed=12)
    return h, iq


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_2206_05506_b200 as P
    from paper_2206_05506_b200 import distributed as D
    from paper_2206_05506_b200 import synth as S
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name, (n, m, l, nb, f) in {"cfg3": (64, 1023, 64, 8, 5), "cfg2": (16, 255, 32, 4, 7)}.items():
            cfg = P.PilotConfig(m=m, c=l, n_t=n, n_batch=nb, l=l, f_s=10e6)
            full = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, n, device=dev)
            h, iq = _inputs(P, S, full, f)                    # identical on every rank (seeded)
            ref_taps, ref_stats, ref_link = full.process_scored(iq, h)
            ref_total = D.reduce_stats(ref_stats.clone(), group=None) / world   # (every rank adds the same)
            # --- frames: contiguous frame ranges, no collective until the gather/reduce
            a, b = D.frame_shard(f, rank, world)
            taps, stats, _ = full.process_scored(iq[a:b].contiguous(), h[a:b].contiguous())
            gathered = D.gather_taps(taps, dst=0)
            total = D.reduce_stats(stats)
            # --- antennas: this rank's receivers only, then the all-gather of the CIRs
            r0, r1 = D.antenna_shard(n, rank, world)
            part = P.Correlator(P.default_spec((m + 1).bit_length() - 1), cfg, r1 - r0, device=dev)
            iq_r = iq[:, :, r0:r1].contiguous()
            taps_r, stats_r, link_r = part.process_scored(iq_r, h[:, r0:r1].contiguous())
            csi = D.allgather_csi(taps_r)
            fstats = D.reduce_frame_stats(stats_r)
            links = D.allgather_csi(link_r.unsqueeze(-1)).squeeze(-1)
            # --- antennas with the all-gather fused into the epilogue (CUDA-IPC peer buffers)
            gat = D.CsiGather(part, n, f)
            gat.run(iq_r)
            fused = gat.wait().clone()
            gat.close()                 # release the peer mappings before any producer exits
            res[name] = {
                "frames_taps_equal": None if gathered is None else bool(torch.equal(gathered, ref_taps)),
                "frames_total": total.tolist(), "single_total": ref_total.tolist(),
                "antenna_taps_equal": bool(torch.equal(csi, ref_taps)),
                "antenna_links_equal": bool(torch.equal(links, ref_link)),
                "fused_gather_equal": bool(torch.equal(fused, ref_taps)),
                "antenna_stats": fstats.tolist(), "single_stats": ref_stats.tolist(),
            }
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_share_one_gpu_bit_identical(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        for name, r in out[rank].items():
            if rank == 0:
                assert r["frames_taps_equal"], name
            assert r["antenna_taps_equal"], name          # CSI on every rank == single rank
            assert r["antenna_links_equal"], name
            assert r["fused_gather_equal"], name         # epilogue stores into every rank's CSI
            for x, y in zip(r["frames_total"], r["single_total"]):
                # (the per-frame float64 sums add up in another order over 3 ranks)
                assert x == pytest.approx(y, rel=1e-12 if world == 2 else 1e-8, abs=0)
            for fx, fy in zip(r["antenna_stats"], r["single_stats"]):
                for x, y in zip(fx, fy):
                    # (3 ranks: 22/21/21 receivers, so the warps' float32 partials group
                    # links differently than the single-rank launch)
                    assert x == pytest.approx(y, rel=1e-9 if world == 2 else 1e-6, abs=0)
