"""Golden CSV written by the REAL reference: the paper's Table I grid at cfg2 (SURVEY §8d:
16x16 MIMO, M=255, L=C=32, N_b=4, SNR 0..30 dB step 5, 50 iterations, seed 0), with one
row per iteration so the device sweep can be checked draw for draw.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_table1_golden.py

Writes tests/golden/ref_cfg2_table1.csv (pnce.records.render_csv of run_snr_sweep).
"""

from __future__ import annotations

import os
import sys

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from pnce.experiments import ExperimentConfig, run_snr_sweep  # noqa: E402
from pnce.records import render_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    cfg = ExperimentConfig(n_t=16, n_r=16, pn_lengths=(255,), c=32, l=32, l_nz=(32,), n_batch=(4,),
                           snr_db=tuple(float(s) for s in range(0, 31, 5)), iterations=50, seed=0,
                           emit_per_iteration=True, record_latency=False)
    with open(os.path.join(HERE, "ref_cfg2_table1.csv"), "w", newline="") as fh:
        fh.write(render_csv(run_snr_sweep(cfg)))
    print("ok")


if __name__ == "__main__":
    main()
