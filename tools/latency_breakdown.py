"""Single cfg3 frame-set end-to-end latency, broken into its parts (GPU box).

H2D of the CP-stripped bodies, the fused kernel, D2H of the taps -- each timed alone with
CUDA events, then back to back on one stream (no host work between), then through
`Correlator.process_host(chunk=1)` (wall clock), and a receiver-split pipeline estimate:
the frame-set's receivers in G groups (a correlator with n_r/G antennas per group, inputs
pre-arranged per group), H2D / kernel / D2H of the groups overlapped on three streams.
"""
import ctypes
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import _lib  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

REPS = 50
dev = torch.device("cuda", 0)
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
L = _lib.lib()
iq = torch.empty(corr.iq_shape(1), dtype=torch.float32, device=dev)
h = S.draw_channel(corr, 1, seed=1)
S.simulate_frames(corr, h, 10.0, seed=2, out=iq)
h_iq = iq.cpu().pin_memory()
h_taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64).pin_memory()
stride = cfg.m + (cfg.m & 1)
bodies = torch.empty((1, cfg.n_batches, 64, stride, 2), dtype=torch.float32, device=dev)
taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64, device=dev)
s = torch.cuda.current_stream(dev)


def ev_time(fn):
    out = []
    for i in range(REPS + 5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        if i >= 5:
            out.append(a.elapsed_time(b) * 1e3)
    return statistics.median(out), min(out)


def h2d():
    _lib.check(L.pnce_copy_bodies_h2d(corr._plan, ctypes.c_void_p(h_iq.data_ptr()),
                                      ctypes.c_void_p(bodies.data_ptr()), stride, 1, ctypes.c_void_p(s.cuda_stream)))


def kern():
    _lib.check(L.pnce_process_bodies(corr._plan, ctypes.c_void_p(bodies.data_ptr()), stride,
                                     ctypes.c_void_p(taps.data_ptr()), None, None, None, 1,
                                     ctypes.c_void_p(s.cuda_stream)))


def d2h():
    h_taps.copy_(taps, non_blocking=True)


res = {}
res["h2d_bodies"] = ev_time(h2d)
res["kernel"] = ev_time(kern)
res["d2h_taps"] = ev_time(d2h)
res["serial_one_stream"] = ev_time(lambda: (h2d(), kern(), d2h()))
ref_taps = h_taps.clone()

te = []
for i in range(REPS + 5):
    torch.cuda.synchronize(dev)
    w0 = time.perf_counter()
    corr.process_host(h_iq, h_taps, chunk=1)
    torch.cuda.synchronize(dev)
    if i >= 5:
        te.append((time.perf_counter() - w0) * 1e6)
res["process_host_wall"] = (statistics.median(te), min(te))
assert torch.equal(h_taps, ref_taps)

for G in (2, 4):
    nr = 64 // G
    sub = P.Correlator(P.default_spec(10), cfg, nr, device=dev)
    # per-group host bodies already compact ([G][n_batches][nr][stride][2]) -- the best case
    hb = bodies.cpu().view(1, cfg.n_batches, G, nr, stride, 2).permute(2, 0, 1, 3, 4, 5).contiguous().pin_memory()
    db = [torch.empty((1, cfg.n_batches, nr, stride, 2), dtype=torch.float32, device=dev) for _ in range(G)]
    dt = torch.empty((G, 1, nr, 64, 64), dtype=torch.complex64, device=dev)
    ht = torch.empty((G, 1, nr, 64, 64), dtype=torch.complex64).pin_memory()
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def pipe():
        evi = [torch.cuda.Event() for _ in range(G)]
        evk = [torch.cuda.Event() for _ in range(G)]
        s_in.wait_stream(s)
        s_out.wait_stream(s)
        for g in range(G):
            with torch.cuda.stream(s_in):
                db[g].copy_(hb[g], non_blocking=True)
                evi[g].record(s_in)
        for g in range(G):
            s.wait_event(evi[g])
            _lib.check(L.pnce_process_bodies(sub._plan, ctypes.c_void_p(db[g].data_ptr()), stride,
                                             ctypes.c_void_p(dt[g].data_ptr()), None, None, None, 1,
                                             ctypes.c_void_p(s.cuda_stream)))
            evk[g].record(s)
            s_out.wait_event(evk[g])
            with torch.cuda.stream(s_out):
                ht[g].copy_(dt[g], non_blocking=True)
        s.wait_stream(s_out)

    res[f"rx_split_G{G}"] = ev_time(pipe)
    got = ht.permute(1, 0, 2, 3, 4).reshape(1, 64, 64, 64)
    res[f"rx_split_G{G}_bit_identical"] = bool(torch.equal(got, ref_taps))
    res[f"rx_split_G{G}_kernel_alone"] = ev_time(
        lambda: _lib.check(L.pnce_process_bodies(sub._plan, ctypes.c_void_p(db[0].data_ptr()), stride,
                                                 ctypes.c_void_p(dt[0].data_ptr()), None, None, None, 1,
                                                 ctypes.c_void_p(s.cuda_stream))))

for k, v in res.items():
    if isinstance(v, tuple):
        print(f"{k:28s} median {v[0]:8.1f} us   min {v[1]:8.1f} us")
    else:
        print(f"{k:28s} {v}")
