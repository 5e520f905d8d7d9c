"""Pipeline variants that must not change a single bit: the split drain (first accumulator
half released early), the A-stage reuse across lag-row groups (L2 scratch), and the
LDGSTS truth ring of the scored drain, the narrow lag-row groups of few-tile launches and
their LDG converters, the 256-column tiling of 5-9 frame-set launches, the LDG converters
of plain launches with >= 3 groups (cfg4') --
each run in a subprocess with its knob off and
compared with the default build of the same launch (same MMAs in the same K order, same
epilogue arithmetic).  Covers one group (cfg3), two groups (scored / tensor16 tilings) and
four groups (cfg4')."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2206_05506_b200 as P
from paper_2206_05506_b200 import synth as S
dev = torch.device("cuda:0")
out = {}
for name, m, l, nt, nb, nr, deg, F in (("cfg3", 1023, 64, 64, 8, 64, 10, 9), ("cfg3_1", 1023, 64, 64, 8, 64, 10, 1),
                                       ("cfg4", 2047, 127, 128, 16, 128, 11, 3),
                                       ("odd", 1023, 40, 24, 10, 40, 10, 5)):
    cfg = P.PilotConfig(m=m, c=l, n_t=nt, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(P.default_spec(deg), cfg, nr, device=dev)
    h = S.draw_channel(corr, F, seed=5)
    iq = S.simulate_frames(corr, h, 12.0, seed=6)
    taps, _ = corr.process(iq)
    out[name + "_plain"] = taps.cpu().numpy()
    taps_s, st, lk = corr.process_scored(iq, h)
    out[name + "_scored"] = taps_s.cpu().numpy()
    out[name + "_stats"] = st.cpu().numpy()
    out[name + "_link"] = lk.cpu().numpy()
    t16, st16 = corr.process_tensor16(iq, chunk_len=256, accumulator="binary16")
    out[name + "_t16"] = t16.cpu().numpy()
    torch.cuda.synchronize()
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, tag, env_extra):
    path = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT, path], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return np.load(path)


@pytest.fixture(scope="module")
def default_run(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _run(tmp_path_factory.mktemp("knobs"), "default", {})


@pytest.mark.parametrize("knob,value", [("PNCE_TUNE_SPLIT_DRAIN", "0"), ("PNCE_TUNE_A_REUSE", "0"),
                                        ("PNCE_TUNE_A_REUSE", "2"),
                                        ("PNCE_TUNE_TRUTH_SLOTS", "0"), ("PNCE_TUNE_TRUTH_SLOTS", "3"),
                                        ("PNCE_TUNE_NARROW", "0"), ("PNCE_TUNE_NARROW_LDG", "0"), ("PNCE_TUNE_MID", "0"),
                                        ("PNCE_TUNE_SCORED_G", "256"), ("PNCE_TUNE_SCORED_EPI", "4"),
                                        ("PNCE_TUNE_T16_EPI", "4"), ("PNCE_TUNE_WIDE_LDG", "0")])
def test_variant_bit_identical(default_run, tmp_path, knob, value):
    other = _run(tmp_path, knob + value, {knob: value})
    for key in default_run.files:
        a, b = default_run[key], other[key]
        if key.endswith("_stats") or key.endswith("_link"):
            # float atomics: the summation order of the per-frame / per-link partials may differ
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-12, err_msg=f"{knob}: {key}")
        else:
            assert np.array_equal(a, b), f"{knob}: {key} differs"
