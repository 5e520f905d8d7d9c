"""BASELINE configs[4]: the parameter sweep grid (PN 127..4095 x CIR 8..256 x N_b 1..32) at
256 receive and 256 transmit antennas -- estimation throughput of the fused kernel at every
feasible point (L <= M, N_b <= floor(M/L), shift spacing >= L; pilots.py:39-42, 134-142),
inputs from the device synthesiser.  One GPU; points shard over GPUs like sweeps.py."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

PEAK = 1645.7e12
dev = torch.device("cuda:0")
n_t = n_r = 256
rows = []
t_start = time.perf_counter()
print(f"{'M':>5} {'L':>4} {'N_b':>4} {'F':>3} {'us/frame-set':>13} {'TFLOP/s':>8} {'tensor%':>8} {'GB/s':>7}")
for m in (127, 255, 511, 1023, 2047, 4095):
    deg = (m + 1).bit_length() - 1
    spec = P.LfsrSpec(12, (12, 6, 4, 1), 1) if deg == 12 else P.default_spec(deg)
    for l in (8, 16, 32, 64, 128, 256):
        for nb in (1, 2, 4, 8, 16, 32):
            if l > m or nb > m // l or (m // nb) < l:
                continue
            cfg = P.PilotConfig(m=m, c=l, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
            corr = P.Correlator(spec, cfg, n_r, device=dev)
            per_set = cfg.n_batches * n_r * cfg.samples_per_receiver * 8
            F = max(1, min(8, (1 << 30) // per_set))
            h = S.draw_channel(corr, F, seed=m + l + nb)
            iq = S.simulate_frames(corr, h, 20.0, seed=1)
            taps, _ = corr.process(iq)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record()
            for _ in range(reps):
                corr.process(iq, out=taps)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / (reps * F)
            flop = 4.0 * n_t * l * m * n_r
            gbs = (cfg.n_batches * n_r * m * 8 + n_r * n_t * l * 8) / t / 1e9
            rows.append((m, l, nb, F, t * 1e6, flop / t / 1e12, 100 * flop / t / PEAK, gbs))
            print(f"{m:5d} {l:4d} {nb:4d} {F:3d} {t * 1e6:13.2f} {flop / t / 1e12:8.1f} {100 * flop / t / PEAK:8.1f} {gbs:7.0f}",
                  flush=True)
            del corr, h, iq, taps
print(f"{len(rows)} feasible points in {time.perf_counter() - t_start:.1f} s; "
      f"best {max(r[6] for r in rows):.1f} % of the bf16 peak, median {sorted(r[6] for r in rows)[len(rows) // 2]:.1f} %")
