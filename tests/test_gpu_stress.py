"""Randomised cross-mode stress (tools/stress.py) as a GPU test: random feasible geometries,
frame counts, dtypes and SNRs; plain == scored == packed bit for bit, per-link and frame
MSE consistent, tensor16 single chunk == plain, oracle parity on a sample."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_random_stress():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress.py"), "7", "80"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
