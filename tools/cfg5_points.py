"""A few BASELINE configs[4] points (256x256) timed through the C ABI directly (no Python
wrapper in the timed loop): for A/B of library builds (PNCE_LIB)."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import _lib  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
L = _lib.lib()
for (m, l, nb) in ((4095, 256, 8), (4095, 128, 16), (2047, 64, 16), (4095, 64, 32), (1023, 64, 8), (127, 8, 1)):
    deg = (m + 1).bit_length() - 1
    spec = P.LfsrSpec(12, (12, 6, 4, 1), 1) if deg == 12 else P.default_spec(deg)
    cfg = P.PilotConfig(m=m, c=l, n_t=256, n_batch=nb, l=l, f_s=10e6)
    corr = P.Correlator(spec, cfg, 256, device=dev)
    per_set = cfg.n_batches * 256 * cfg.samples_per_receiver * 8
    F = max(1, min(8, (1 << 30) // per_set))
    h = S.draw_channel(corr, F, seed=m + l + nb)
    iq = S.simulate_frames(corr, h, 20.0, seed=1)
    taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64, device=dev)
    st = torch.cuda.current_stream(dev)
    args = (corr._plan, iq.data_ptr(), taps.data_ptr(), None, None, None, 0, F, st.cuda_stream)
    for _ in range(3):
        L.pnce_process_frames(*args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        L.pnce_process_frames(*args)
    e1.record(st)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / (10 * F)
    print(f"M={m} L={l} N_b={nb} F={F}: {t * 1e6:.2f} us/frame-set", flush=True)
    del corr, h, iq, taps
