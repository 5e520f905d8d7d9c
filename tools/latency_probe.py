import statistics, sys, time, subprocess
import torch
sys.path.insert(0, ".")
import paper_2206_05506_b200 as P
from paper_2206_05506_b200 import synth as S
dev = torch.device("cuda", 0)
cfg = P.PilotConfig(m=1023, c=64, n_t=64, n_batch=8, l=64, f_s=10e6)
corr = P.Correlator(P.default_spec(10), cfg, 64, device=dev)
iq = torch.empty(corr.iq_shape(4), dtype=torch.float32, device=dev)
h = S.draw_channel(corr, 4, seed=1); S.simulate_frames(corr, h, 10.0, seed=2, out=iq)
def loop(tag, h_iq, h_taps):
    te = []
    for i in range(55):
        torch.cuda.synchronize(dev); w0 = time.perf_counter()
        corr.process_host(h_iq, h_taps, chunk=1)
        torch.cuda.synchronize(dev)
        if i >= 5: te.append((time.perf_counter() - w0) * 1e6)
    print(f"{tag:40s} median {statistics.median(te):7.1f} min {min(te):7.1f}", flush=True)
a = iq[:1].cpu().pin_memory(); t = torch.empty(corr.taps_shape(1), dtype=torch.complex64).pin_memory()
loop("tool-style buffers", a, t)
b = torch.empty(corr.iq_shape(1), dtype=torch.float32).pin_memory(); b.copy_(iq[:1].cpu())
t2 = torch.empty(corr.taps_shape(1), dtype=torch.complex64).pin_memory()
loop("bench-style buffers", b, t2)
p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
time.sleep(1.0)
loop("with nvidia-smi -lms 100 running", b, t2)
p.terminate(); p.wait()
loop("after nvidia-smi terminated", b, t2)
time.sleep(2.0)
loop("2 s later", b, t2)
