"""Randomised stress of the device path: random feasible geometries, frame counts, dtypes
and modes; every result cross-checked (plain == scored taps == packed path bit for bit,
per-link MSE consistent, tensor16 binary32 == plain within 1e-5, oracle within 1e-2 on a
sample).  Catches pipeline/barrier protocol bugs that fixed-shape tests can miss."""
import math
import random
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402
from oracle import pnce_oracle as O  # noqa: E402

dev = torch.device("cuda:0")
rng = random.Random(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 100
t0 = time.time()
fails = 0
for it in range(n_iter):
    while True:
        deg = rng.choice([6, 7, 8, 9, 10, 11])
        m = (1 << deg) - 1
        l = rng.choice([4, 8, 13, 16, 20, 32, 64, 100, 127, 128, 200, 256])
        c = l + rng.choice([0, 0, 0, 1, 3, 17])
        nb = rng.choice([1, 2, 3, 4, 5, 8, 16, 32])
        if l <= c <= m and nb <= m // c and (m // nb) >= l:
            break
    n_t = rng.choice([1, 2, 3, nb, nb + 1, 2 * nb, 3 * nb + 1])
    n_r = rng.choice([1, 2, 3, 5, 8, 16, 33, 64])
    F = rng.choice([1, 2, 3, 7, 16, 33])
    dtype = rng.choice(["fp16", "bf16"])
    tag = f"it={it} M={m} L={l} C={c} N_b={nb} n_t={n_t} n_r={n_r} F={F} {dtype}"
    try:
        cfg = P.PilotConfig(m=m, c=c, n_t=n_t, n_batch=nb, l=l, f_s=10e6)
        corr = P.Correlator(P.default_spec(deg), cfg, n_r, dtype=dtype, device=dev)
        h = S.draw_channel(corr, F, seed=it)
        iq = S.simulate_frames(corr, h, rng.choice([0.0, 10.0, 30.0, math.inf]), seed=it + 1)
        taps, _ = corr.process(iq)
        t2, st, lk = corr.process_scored(iq, h)
        assert torch.equal(taps, t2), "scored taps differ"
        tp, _ = corr.correlate(corr.pack(iq), F)
        assert torch.equal(taps, tp), "packed path differs"
        e2 = (taps - h).abs().double() ** 2
        assert torch.allclose(lk.double(), e2.mean(-1), rtol=1e-3, atol=1e-12), "link mse"
        assert torch.allclose(st[:, 1], e2.sum((1, 2, 3)), rtol=1e-3), "frame mse"
        if (64 * ((m + 63) // 64)) >= 256 and cfg.samples_per_receiver % 2 == 0:
            t16, _ = corr.process_tensor16(iq, chunk_len=None)
            assert torch.equal(t16, taps), "tensor16 single chunk differs"
        if it % 5 == 0:
            ocfg = O.Config(m=m, c=c, n_t=n_t, n_batch=nb, l=l, n_r=n_r)
            ref = O.process_frames(O.sequence_for_length(m), ocfg, O.iq_to_frames(iq[0].cpu().numpy()))[0]
            got = taps[0].cpu().numpy().astype(np.complex128)
            sc = np.abs(ref).max(axis=-1, keepdims=True)
            sc[sc == 0] = 1
            err = float((np.abs(got - ref) / sc).max())
            tol = 1e-2 if dtype == "fp16" else 2e-2
            assert err <= tol, f"oracle err {err:.2e}"
    except Exception as exc:  # report and continue
        fails += 1
        print("FAIL", tag, type(exc).__name__, str(exc)[:200], flush=True)
        if "CUDA" in str(exc) or "launch" in str(exc):
            break
print(f"{n_iter} iterations, {fails} failures, {time.time() - t0:.1f} s")
sys.exit(1 if fails else 0)
