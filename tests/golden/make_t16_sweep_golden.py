"""Golden CSV written by the REAL reference: run_snr_sweep with the tensor16 backend
(BackendConfig(kind="tensor16", chunk_len=128, accumulator="binary16")) at cfg2 geometry
(16x16, M=255, L=C=32, N_b=4), SNR {0, 15, 30} dB, 6 iterations, one row per iteration.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_t16_sweep_golden.py
"""

from __future__ import annotations

import os
import sys

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from pnce.experiments import ExperimentConfig, run_snr_sweep  # noqa: E402
from pnce.halfprec import BackendConfig  # noqa: E402
from pnce.records import render_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cfg = ExperimentConfig(n_t=16, n_r=16, pn_lengths=(255,), c=32, l=32, l_nz=(32,), n_batch=(4,),
                           snr_db=(0.0, 15.0, 30.0), iterations=6, seed=0, emit_per_iteration=True,
                           record_latency=False,
                           backend=BackendConfig(kind="tensor16", chunk_len=128, accumulator="binary16"))
    with open(os.path.join(HERE, "ref_t16_sweep.csv"), "w", newline="") as fh:
        fh.write(render_csv(run_snr_sweep(cfg)))
    print("ok")


if __name__ == "__main__":
    main()
