"""cfg4' fused launch for the cycle-accounting build (PNCE_LIB=tools/bin/libpnce_diag_prof.so,
PNCE_PROF_FILE=...): the last launch's counters are dumped."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2206_05506_b200 as P  # noqa: E402
from paper_2206_05506_b200 import synth as S  # noqa: E402

dev = torch.device("cuda:0")
F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = P.PilotConfig(m=2047, c=127, n_t=128, n_batch=16, l=127, f_s=10e6)
corr = P.Correlator(P.default_spec(11), cfg, 128, device=dev)
h = S.draw_channel(corr, F, seed=77)
iq = S.simulate_frames(corr, h, 10.0, seed=78)
taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64, device=dev)
mode = sys.argv[2] if len(sys.argv) > 2 else "fused"
if mode == "packed":  # the GEMM on the packed fp16 operand instead
    packed = corr.pack(iq)
    run = lambda: corr.correlate(packed, F, out=taps)  # noqa: E731
elif mode == "scored":  # fused + per-frame sums and per-link MSE against the drawn channel
    stats = torch.zeros((F, 4), dtype=torch.float64, device=dev)
    link = torch.zeros((F, 128, 128), dtype=torch.float32, device=dev)
    run = lambda: corr.process_scored(iq, h, out=taps, stats=stats, link_mse=link)  # noqa: E731
else:
    run = lambda: corr.process(iq, out=taps)  # noqa: E731
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    run()
e0.record()
run()
e1.record()
torch.cuda.synchronize()
print(f"cfg4' {mode} {e0.elapsed_time(e1) * 1e3 / F:.2f} us/frame-set")
