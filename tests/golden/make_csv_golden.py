"""Golden CSV written by the REAL reference (`pnce.records.render_csv`), for the sweep
records of SURVEY §8f row f4.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_csv_golden.py

Writes tests/golden/ref_records.csv (reference renderer, rows with awkward floats) and
tests/golden/ref_snr_sweep.csv (the reference's run_snr_sweep at 4x4, M in {63, 127},
L=C=16, N_b=1, SNR {-10, 10, 30}, 4 iterations, seed 0, latency recording off).
"""

from __future__ import annotations

import os
import sys

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from pnce.experiments import ExperimentConfig, SweepResult, run_snr_sweep  # noqa: E402
from pnce.records import render_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rows = [
        SweepResult("snr_sweep", "reference64", 16, 16, 255, 32, 32, 32, 4, -10.0, 50, 0, 0.0108282512345,
                    1.23456789e-3, 4608, 2088960, 0),
        SweepResult("tap_sweep", "tensor16", 4, 4, 127, 16, 16, 3, 1, 2.5, 1, 12345678901234567890,
                    1e-12, 0.0, 560, 32512, 7),
        SweepResult("latency_bench", "reference32", 64, 64, 1023, 64, 64, 64, 8, 30.0, 10, 0, 0.0,
                    0.0136, 589312, 268173312, 0),
    ]
    with open(os.path.join(HERE, "ref_records.csv"), "w", newline="") as fh:
        fh.write(render_csv(rows))
    cfg = ExperimentConfig(n_t=4, n_r=4, pn_lengths=(63, 127), c=16, l=16, l_nz=(16,), n_batch=(1,),
                           snr_db=(-10.0, 10.0, 30.0), iterations=4, seed=0, record_latency=False)
    with open(os.path.join(HERE, "ref_snr_sweep.csv"), "w", newline="") as fh:
        fh.write(render_csv(run_snr_sweep(cfg)))
    print("ok")


if __name__ == "__main__":
    main()
