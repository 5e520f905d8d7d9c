"""Benchmark: PN-correlation channel estimation at 64x64 MIMO, PN 1023 (BASELINE cfg3).

One step = one pass of the hot path over a batch of F frame-sets already resident in
HBM: ONE fused kernel launch (CP strip + fp16 quantise + tcgen05 correlation with the
PN circulant + 1/M + per-transmitter demux into complex64 taps) (default F = 10,000, the
BASELINE headline: 47 GB of received IQ, far larger than L2).  value = CSI
estimates/s = link CIRs (frame, rx, tx) per second over all ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Under torchrun each rank estimates its own F frame-sets (weak scaling, no
hot-path collective); the step time is the max over ranks (NCCL all_reduce MAX of
the CUDA-event time) and the per-rank error statistics are all_reduced at the end.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs[2] (headline single-GPU bench)
WORKLOAD = dict(name="cfg3", n_t=64, n_r=64, m=1023, l=64, c=64, n_batch=8, snr_db=10.0)
# the `config` object both arms print, textually identical (the per-step sample sizes and the
# parallelism of each arm are reported beside it, under "run")
CONFIG = {"workload": "cfg3 64x64 MIMO, PN 1023, L=C=64, N_batch=8, 10 dB (BASELINE configs[2])",
          "metric_unit": "CSI estimates/s (link CIRs of L taps per second)",
          "l2": "GPU arm: inputs (f32 IQ, 4.7 MB per frame-set) far larger than the 126 MB L2, no flush"}
def _baseline_metric() -> str:
    """BASELINE.json's metric string, verbatim (fallback: the same text)."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "BASELINE.json")) as fh:
            return json.load(fh)["metric"]
    except Exception:
        return "CSI estimates/sec & \u00b5s/frame at 64\u00d764 MIMO, PN 1023; tensor-pipe % of peak"


METRIC = _baseline_metric()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def algorithmic_per_frame(w):
    """FLOP = 4*macs (macs = n_t*L*M*n_r, experiments.py:200).
    bytes_gemm  = fp16 body in + complex64 taps out (packed-operand GEMM, §8d);
    bytes_fused = f32 (I,Q) CP-stripped body in + complex64 taps out (the fused kernel)."""
    n_batches = -(-w["n_t"] // w["n_batch"])
    macs = w["n_t"] * w["l"] * w["m"] * w["n_r"]
    flop = 4 * macs
    taps = w["n_r"] * w["n_t"] * w["l"] * 8
    bytes_gemm = w["n_r"] * n_batches * w["m"] * 2 * 2 + taps
    bytes_fused = w["n_r"] * n_batches * w["m"] * 8 + taps
    return flop, bytes_gemm, bytes_fused


class ClockSampler:
    """Samples nvidia-smi SM clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        limit = None
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=power.limit",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            limit = float(out.stdout.strip().splitlines()[0])
        except Exception:
            pass
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if r[4 + i].lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": limit}


def cpu_reference_rate(w, seconds, threads=None):
    """Time the oracle port of process_frames (reference64, experiments.py:176-208) on the
    host cores over a bounded sample; returns (CSI estimates/s, cores, sample description)."""
    import numpy as np
    from oracle import pnce_oracle as O
    cfg = O.Config(m=w["m"], c=w["c"], n_t=w["n_t"], n_batch=w["n_batch"], l=w["l"], n_r=w["n_r"])
    chips = O.sequence_for_length(w["m"])
    plan = O.build_batch_plan(cfg)
    rows = O.correlator_rows_for_plan(chips, plan, cfg.l)
    # two distinct pre-simulated frame-sets (experiments.py:373: synthesis is untimed)
    pool = []
    for it in range(2):
        cs, ns = O.derive_seeds(0, cfg.m, cfg.n_batch, cfg.l, 0, it)
        _, frames = O.simulate_frame(chips, cfg, cfg.l, w["snr_db"], cs, ns)
        pool.append(O.iq_to_frames(O.frames_to_iq(frames)))
    for f in pool:   # warm-up (run_latency_bench warmup=2)
        O.process_frames(chips, cfg, f, rows_per_batch=rows)
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 3:
        f = pool[len(times) % 2]
        t0 = time.perf_counter()
        O.process_frames(chips, cfg, f, rows_per_batch=rows)
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    cores = threads or os.cpu_count()
    rate = w["n_r"] * w["n_t"] / med
    sample = (f"{len(times)} frame-sets of cfg3 through the numpy oracle port of process_frames "
              f"(reference64), median {med * 1e3:.2f} ms/frame-set, {cores} BLAS threads")
    return rate, cores, sample, med


def cpu_backend_times(w, seconds=3.0):
    """SURVEY §8d CPU baseline detail: the oracle port of process_frames with the
    reference's other backends (reference32; tensor16, the paper-arithmetic emulation with
    256-sample chunks and binary16 partials) on all host threads, and reference64 on ONE
    BLAS thread; median ms per cfg3 frame-set over a bounded sample each."""
    from threadpoolctl import threadpool_limits
    from oracle import pnce_oracle as O
    cfg = O.Config(m=w["m"], c=w["c"], n_t=w["n_t"], n_batch=w["n_batch"], l=w["l"], n_r=w["n_r"])
    chips = O.sequence_for_length(w["m"])
    rows = O.correlator_rows_for_plan(chips, O.build_batch_plan(cfg), cfg.l)
    cs, ns = O.derive_seeds(0, cfg.m, cfg.n_batch, cfg.l, 0, 0)
    _, frames = O.simulate_frame(chips, cfg, cfg.l, w["snr_db"], cs, ns)
    frames = O.iq_to_frames(O.frames_to_iq(frames))

    def med_ms(**kw):
        O.process_frames(chips, cfg, frames, rows_per_batch=rows, **kw)   # warm-up
        ts, t_end = [], time.perf_counter() + seconds
        while time.perf_counter() < t_end or len(ts) < 2:
            t0 = time.perf_counter()
            O.process_frames(chips, cfg, frames, rows_per_batch=rows, **kw)
            ts.append(time.perf_counter() - t0)
        return {"ms_per_frame_set": statistics.median(ts) * 1e3, "samples": len(ts)}

    out = {"threads": os.cpu_count(),
           "reference32": med_ms(backend="reference32"),
           "tensor16": med_ms(backend="tensor16", chunk_len=256, accumulator="binary16")}
    with threadpool_limits(limits=1):
        out["reference64_1_thread"] = med_ms(backend="reference64")
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    w = WORKLOAD
    per_step = []
    sample = None
    cores = os.cpu_count()
    for i in range(args.warmup + args.steps):
        rate, cores, sample, med = cpu_reference_rate(w, seconds=args.ref_seconds)
        if i >= args.warmup:
            per_step.append(med)
    med = statistics.median(per_step)
    value = w["n_r"] * w["n_t"] / med
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "CSI estimates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": med * 1e3, "us_per_frame": med * 1e6, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(CONFIG),
        "run": {"frames_per_step": 1, "parallelism": "host threads (OpenBLAS)",
                "sample": "each step: the median of a bounded sample of cfg3 frame-sets (--ref-seconds)"},
        "cpu_baseline": {"value": value, "unit": "CSI estimates/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "CSI estimates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        line["cpu_backends"] = cpu_backend_times(w)
    except Exception as exc:  # informational only
        line["cpu_backends"] = {"skipped": f"{type(exc).__name__}: {exc}"[:200]}
    print(json.dumps(line), flush=True)
    return 0


def ingest_leg(corr, iq, taps, w, Ff, rank):
    """IQ file written (untimed) to a local temp dir, then estimated through
    iqfile.estimate_file (page cache -> pinned -> HBM -> pinned taps); host wall clock."""
    import tempfile

    import torch
    from paper_2206_05506_b200 import iqfile as IQ
    hdr = IQ.IqFileHeader(n_t=w["n_t"], n_r=w["n_r"], p=w["c"] + w["m"], l=w["l"], m=w["m"], c=w["c"],
                          n_batch=w["n_batch"], frame_count=Ff * corr.cfg.n_batches, seed=1234 + rank)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "frames.iq")
        IQ.write_iq_tensor(path, hdr, iq[:Ff])
        taps_f = torch.empty(corr.taps_shape(Ff), dtype=torch.complex64).pin_memory()
        IQ.estimate_file(path, corr, taps_host=taps_f)            # warm-up (page cache, pools)
        t0 = time.perf_counter()
        IQ.estimate_file(path, corr, taps_host=taps_f)
        tf = time.perf_counter() - t0
        ok = torch.equal(taps_f[:min(Ff, 4)], taps[:min(Ff, 4)].cpu())
        size = os.path.getsize(path)
    return {"value": Ff / tf * w["n_r"] * w["n_t"], "unit": "CSI estimates/s", "frames": Ff, "file_bytes": size,
            "us_per_frame": tf / Ff * 1e6, "GB_per_s": size / tf / 1e9, "taps_match_resident_path": bool(ok),
            "timing": "host wall clock, file in page cache"}


def cfg4_leg(P, S, dev, stream, F4, steps, tf_burst, tf_sust):
    """BASELINE configs[3] (cfg4': 128x128 MIMO, PN 2047, L=C=127, N_b=16 -> 2032 lag rows,
    four 512-column groups): the tensor-bound configuration.  Fused kernel (f32 IQ in) and
    the GEMM on the pre-packed fp16 operand, device-synthesised inputs, CUDA events."""
    import torch
    cfg = P.PilotConfig(m=2047, c=127, n_t=128, n_batch=16, l=127, f_s=10e6)
    corr = P.Correlator(P.default_spec(11), cfg, 128, device=dev)
    h = S.draw_channel(corr, F4, seed=77)
    iq = S.simulate_frames(corr, h, 10.0, seed=78)
    del h
    taps = torch.empty(corr.taps_shape(F4), dtype=torch.complex64, device=dev)
    flop = 4.0 * cfg.n_t * cfg.l * cfg.m * 128

    def timed(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / 1e3 / steps / F4

    tf = timed(lambda: corr.process(iq, out=taps))
    packed = corr.pack(iq)
    tp = timed(lambda: corr.correlate(packed, F4, out=taps))
    del packed, iq, taps
    out = {"workload": "cfg4' 128x128 MIMO, PN 2047, L=C=127, N_batch=16 (BASELINE configs[3])", "frames": F4,
           "flop_per_frame": flop}
    for name, t in (("fused", tf), ("gemm", tp)):
        out[name] = {"us_per_frame": t * 1e6, "tflops": flop / t / 1e12, "frac_of_bf16_peak": flop / t / 1e12 / tf_burst,
                     "frac_of_bf16_sustained": (flop / t / 1e12 / tf_sust) if tf_sust else None}
    return out


def antenna_leg(P, D, dev, stream, w, iq1, reps, rank, world):
    """One cfg3 frame-set split over the ranks by receive antenna, the paper's scheme
    (PAPER.md:150-153): each rank estimates its N_r / N_ranks receivers in one fused launch,
    then the CIRs are all-gathered so every rank holds the full CSI.  Per rep: barrier, CUDA
    events on the launching stream around the launch (kernel) and around launch + all-gather
    (total); each figure is the max over ranks, then the median over reps."""
    import statistics as st

    import torch
    import torch.distributed as dist
    r0, r1 = D.antenna_shard(w["n_r"], rank, world)
    cfg = P.PilotConfig(m=w["m"], c=w["c"], n_t=w["n_t"], n_batch=w["n_batch"], l=w["l"], f_s=10e6)
    part = P.Correlator(P.default_spec(10), cfg, r1 - r0, device=dev)
    iq_r = iq1[:, :, r0:r1].contiguous()
    taps_r = torch.empty(part.taps_shape(1), dtype=torch.complex64, device=dev)
    kern, tot = [], []
    for i in range(reps + 5):
        if world > 1:
            dist.barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize(dev)
        e0.record(stream)
        part.process(iq_r, out=taps_r)
        e1.record(stream)
        csi = D.allgather_csi(taps_r)
        e2.record(stream)
        torch.cuda.synchronize(dev)
        k, t = D.max_over_ranks([e0.elapsed_time(e1) * 1e3, e0.elapsed_time(e2) * 1e3])
        if i >= 5:
            kern.append(k)
            tot.append(t)
    assert csi.shape == (1, w["n_r"], w["n_t"], w["l"])
    # the same split with the all-gather fused into the epilogue: each rank's kernel stores its
    # receivers' taps into every rank's CSI buffer (CUDA-IPC mappings, NVLink stores)
    fused = None
    try:
        gat = D.CsiGather(part, w["n_r"], 1)
        fg = []
        for i in range(reps + 5):
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record(stream)
            gat.run(iq_r)
            e1.record(stream)
            gat.wait()
            (t,) = D.max_over_ranks([e0.elapsed_time(e1) * 1e3])
            if i >= 5:
                fg.append(t)
        fused_ok = bool(torch.equal(gat.csi, csi))
        gat.close()
        fused = {"us_median": st.median(fg), "csi_equal_to_allgather": fused_ok}
    except Exception as exc:  # noqa: BLE001 -- the leg reports, the bench line survives
        fused = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    return {"ranks": world, "receivers_per_rank": r1 - r0, "frames": 1, "reps": reps,
            "kernel_us_median": st.median(kern), "with_allgather_us_median": st.median(tot),
            "fused_gather": fused,
            "allgather_bytes": w["n_r"] * w["n_t"] * w["l"] * 8,
            "note": "per rep: max over ranks of CUDA-event time (launch; launch + all-gather of the CIRs)"}


def run_gpu(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2206_05506_b200 as P
    from paper_2206_05506_b200 import _lib

    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; with more ranks than GPUs (a gloo smoke run of the multi-rank
    # path on a 1-GPU box) ranks share devices round-robin
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    w = dict(WORKLOAD)
    F = args.frames
    cfg = P.PilotConfig(m=w["m"], c=w["c"], n_t=w["n_t"], n_batch=w["n_batch"], l=w["l"], f_s=10e6)
    corr = P.Correlator(P.default_spec(10), cfg, w["n_r"], dtype=args.dtype, device=dev)

    # --- resident synthetic input: F distinct frame-sets synthesised on the device by the
    # library's own channel draw + pilot sweep + AWGN (untimed input synthesis)
    from paper_2206_05506_b200 import synth as S
    Fq = min(F, args.scored_frames) if not args.no_quality else 0
    ts0 = time.perf_counter()
    iq = torch.empty(corr.iq_shape(F), dtype=torch.float32, device=dev)
    h_q = None
    chunk = 2048
    for s0 in range(0, F, chunk):
        e0 = min(F, s0 + chunk)
        h = S.draw_channel(corr, e0 - s0, seed=(1234 + rank) * 1_000_003 + s0)
        S.simulate_frames(corr, h, w["snr_db"], seed=(4321 + rank) * 1_000_003 + s0, out=iq[s0:e0])
        if s0 < Fq:
            h_q = h[:Fq - s0].clone() if h_q is None else torch.cat([h_q, h[:Fq - s0]])
        del h
    torch.cuda.synchronize(dev)
    synth_s = time.perf_counter() - ts0
    taps = torch.empty(corr.taps_shape(F), dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)
    L = _lib.lib()

    launch_frames = args.launch_frames if args.launch_frames > 0 else F
    iq_stride = iq[0].numel() * 4 if F > 0 else 0
    taps_stride = taps[0].numel() * 8 if F > 0 else 0

    def step():
        # the hot path: fused launches (CP strip + quantise + tcgen05 correlate + demux + 1/M),
        # one per `launch_frames` frame-sets (default: ONE launch over all F)
        for f0 in range(0, F, launch_frames):
            n = min(launch_frames, F - f0)
            _lib.check(L.pnce_process_frames(corr._plan, iq.data_ptr() + f0 * iq_stride,
                                             taps.data_ptr() + f0 * taps_stride, None, None, None, 0, n,
                                             stream.cuda_stream))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.25)
    launches0 = L.pnce_kernel_launches()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize(dev)
    evs[0].record(stream)
    for i in range(args.steps):
        step()
        evs[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    launches = L.pnce_kernel_launches() - launches0
    clocks = sampler.stop()
    t_total = evs[0].elapsed_time(evs[-1]) / 1e3                      # s, device time
    t_step = [evs[i].elapsed_time(evs[i + 1]) / 1e3 for i in range(args.steps)]
    t_kernel = sum(t_step) / args.steps                                # one launch per step
    from paper_2206_05506_b200 import distributed as D
    if world > 1:
        t_total, t_kernel = D.max_over_ranks([t_total, t_kernel])
    ms_per_step = t_total / args.steps * 1e3
    frames_total = F * world
    frames_per_s = frames_total * args.steps / t_total
    value = frames_per_s * w["n_r"] * w["n_t"]

    # --- roofline of the dominant (only) kernel: fused k_correlate<true>
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    flop_f, bytes_gemm_f, bytes_fused_f = algorithmic_per_frame(w)
    achieved_tf = flop_f * F / t_kernel / 1e12
    achieved_gbs = bytes_fused_f * F / t_kernel / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as fh:
                per_frame = json.load(fh).get("k_correlate_fused_dram_bytes_per_frame")
                traffic = per_frame * F if per_frame else None
        except Exception:
            traffic = None

    # --- estimate quality on the synthetic input: fused scoring + NCCL all-reduce of the
    # per-rank error sums (the only collective of the path)
    quality = None
    if not args.no_quality:
        # fused scoring (taps + per-frame sums + per-link MSE) over the first Fq frame-sets
        # against their true channels
        q_stats = torch.zeros((Fq, 4), dtype=torch.float64, device=dev)
        q_link = torch.zeros((Fq, w["n_r"], w["n_t"]), dtype=torch.float32, device=dev)
        corr.process_scored(iq[:Fq], h_q, out=taps[:Fq], stats=q_stats, link_mse=q_link)  # warm-up
        q_stats.zero_()
        q_link.zero_()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record()
        corr.process_scored(iq[:Fq], h_q, out=taps[:Fq], stats=q_stats, link_mse=q_link)
        q1.record()
        torch.cuda.synchronize()
        quality = D.global_metrics(q_stats, w["n_r"] * w["n_t"] * w["l"], Fq * world)
        quality["mse_db"] = 10 * math.log10(quality["mse"]) if quality["mse"] > 0 else None
        worst = float(q_link.max().item())
        quality["worst_link_mse_db"] = 10 * math.log10(worst) if worst > 0 else None
        quality["frames"] = Fq * world
        quality["scored_us_per_frame"] = q0.elapsed_time(q1) * 1e3 / Fq
        quality["scored_bytes_per_frame"] = bytes_fused_f + w["n_r"] * w["n_t"] * w["l"] * 8
        del h_q, q_stats, q_link

    # --- tensor16 leg: the reference's tensor16 backend on the tensor cores,
    # binary16 partials per 256-sample chunk folded into an fp32 total in TMEM
    t16 = None
    if not args.no_quality:
        Ft = min(F, args.scored_frames)
        st16 = torch.zeros((Ft, 4), dtype=torch.float64, device=dev)
        corr.process_tensor16(iq[:Ft], chunk_len=256, accumulator="binary16", out=taps[:Ft], stats=st16)
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st16.zero_()
        t0e.record()
        corr.process_tensor16(iq[:Ft], chunk_len=256, accumulator="binary16", out=taps[:Ft], stats=st16)
        t1e.record()
        torch.cuda.synchronize(dev)
        t16 = {"chunk_len": 256, "accumulator": "binary16", "frames": Ft,
               "us_per_frame": t0e.elapsed_time(t1e) * 1e3 / Ft,
               "saturations": int(st16[:, 3].sum().item()), "nonfinite": int(st16[:, 2].sum().item())}
        del st16

    # --- GEMM-only leg (K3 on the pre-packed fp16 operand): the north-star tensor-% number
    gemm = None
    if not args.no_gemm_leg:
        Fg = min(F, args.gemm_frames)
        packed = corr.pack(iq[:Fg])
        taps_g = taps[:Fg]
        for _ in range(3):
            _lib.check(L.pnce_correlate(corr._plan, packed.data_ptr(), taps_g.data_ptr(), None, None, Fg,
                                        stream.cuda_stream))
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        g0.record(stream)
        for _ in range(args.steps):
            _lib.check(L.pnce_correlate(corr._plan, packed.data_ptr(), taps_g.data_ptr(), None, None, Fg,
                                        stream.cuda_stream))
        g1.record(stream)
        torch.cuda.synchronize(dev)
        tg = g0.elapsed_time(g1) / 1e3 / args.steps
        gemm = {"kernel": "k_correlate<packed>", "frames": Fg, "us_per_frame": tg / Fg * 1e6,
                "tflops": flop_f * Fg / tg / 1e12, "frac_of_bf16_peak": flop_f * Fg / tg / 1e12 / tf_burst,
                "frac_of_bf16_sustained": (flop_f * Fg / tg / 1e12 / tf_sust) if tf_sust else None,
                "gbs": bytes_gemm_f * Fg / tg / 1e9}
        del packed

    # --- single frame-set latency: one fused launch on ONE resident frame-set
    # (CUDA events, launch included), and end to end through the public host-buffer API
    # (pinned host IQ -> HBM -> taps back in pinned host memory, wall clock)
    lat = None
    if args.latency_reps > 0:
        one_iq, one_taps = iq[:1], taps[:1]
        ts = []
        # the C-ABI call with its (constant) arguments evaluated before the start event
        largs = (corr._plan, one_iq.data_ptr(), one_taps.data_ptr(), None, None, None, 0, 1, stream.cuda_stream)
        for i in range(args.latency_reps + 5):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            rc = L.pnce_process_frames(*largs)
            a1.record(stream)
            _lib.check(rc)
            a1.synchronize()
            if i >= 5:
                ts.append(a0.elapsed_time(a1) * 1e3)
        # the same launch replayed from a CUDA graph (Correlator.capture): the real-time
        # single frame-set loop without the Python/ctypes launch path
        graph, _ = corr.capture(one_iq, out=one_taps)
        tg = []
        for i in range(args.latency_reps + 5):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            graph.replay()
            a1.record(stream)
            a1.synchronize()
            if i >= 5:
                tg.append(a0.elapsed_time(a1) * 1e3)
        del graph
        h_iq = torch.empty(corr.iq_shape(1), dtype=torch.float32).pin_memory()
        h_iq.copy_(one_iq.cpu())
        h_taps = torch.empty(corr.taps_shape(1), dtype=torch.complex64).pin_memory()
        te = []
        # host-side warm-up: the first few hundred calls of a fresh process run 1.5-2x slower
        # (tools/latency_probe.py, profiles/r01/latency_probe_v21.txt), so warm for >= 0.5 s
        e2e_warm = 0
        w_end = time.perf_counter() + 0.5
        while time.perf_counter() < w_end or e2e_warm < 5:
            corr.process_host(h_iq, h_taps, chunk=1)
            torch.cuda.synchronize(dev)
            e2e_warm += 1
        for i in range(args.latency_reps):
            torch.cuda.synchronize(dev)
            w0 = time.perf_counter()
            corr.process_host(h_iq, h_taps, chunk=1)
            torch.cuda.synchronize(dev)
            te.append((time.perf_counter() - w0) * 1e6)
        # the paper's real-time criterion: processing time <= pilot
        # propagation time P*N_t/(N_batch*F_s); P = C + M + L - 1 samples per received batch
        p_samples = w["c"] + w["m"] + w["l"] - 1
        n_batches = -(-w["n_t"] // w["n_batch"])
        prop_10mhz_us = p_samples * n_batches / 10e6 * 1e6
        lat = {"frames": 1, "device_us_median": statistics.median(ts), "device_us_min": min(ts),
               "graph_replay_us_median": statistics.median(tg), "graph_replay_us_min": min(tg),
               "propagation_time_us_at_10MHz": prop_10mhz_us,
               "realtime_up_to_fs_mhz": {"device": p_samples * n_batches / statistics.median(ts),
                                         "e2e": p_samples * n_batches / statistics.median(te),
                                         "amortised": p_samples * n_batches / (ms_per_step * 1e3 / F)},
               "e2e_us_median": statistics.median(te), "e2e_us_min": min(te), "reps": args.latency_reps,
               "e2e_warmup_calls": e2e_warm,
               "note": "device: one fused launch on one resident cfg3 frame-set (narrow tiling, 16 CTA pairs), "
                       "CUDA events around the ctypes call; graph_replay: the same launch from a CUDA graph; "
                       "e2e: pinned host IQ -> H2D (CP stripped in the DMA) -> kernel -> D2H taps, wall clock"}

    # --- the paper's multi-GPU split of one frame-set: receivers over ranks + CSI all-gather
    ant = None
    if args.antenna_reps > 0:
        ant = antenna_leg(P, D, dev, stream, w, iq[:1], args.antenna_reps, rank, world)

    # --- BASELINE configs[3] (cfg4', tensor-bound): fused and packed-GEMM tensor fractions
    c4 = None
    if args.cfg4_frames > 0:
        c4 = cfg4_leg(P, S, dev, stream, args.cfg4_frames, args.steps, tf_burst, tf_sust)

    # --- e2e through the public API with pinned host buffers (H2D in, D2H taps out)
    e2e = None
    if not args.no_e2e:
        Fe = min(args.e2e_frames, F)
        host_iq = torch.empty(corr.iq_shape(Fe), dtype=torch.float32).pin_memory()
        host_iq.copy_(iq[:Fe].cpu())
        host_taps = torch.empty(corr.taps_shape(Fe), dtype=torch.complex64).pin_memory()
        for _ in range(2):
            corr.process_host(host_iq, host_taps, chunk=args.e2e_chunk)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        reps = max(2, args.steps // 2)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(reps):
            corr.process_host(host_iq, host_taps, chunk=args.e2e_chunk)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        te = t0.elapsed_time(t1) / 1e3
        if world > 1:
            te = D.max_over_ranks([te])[0]
        e2e = {"value": Fe * world * reps / te * w["n_r"] * w["n_t"], "unit": "CSI estimates/s",
               "h2d_bytes_per_step": Fe * corr.cfg.n_batches * w["n_r"] * w["m"] * 8,   # body-only pitched DMA
               "d2h_bytes_per_step": host_taps.numel() * 8,
               "frames_per_step": Fe, "chunk": args.e2e_chunk, "us_per_frame": te / (Fe * reps) * 1e6}

    # --- IQ-file ingest: reference-format file -> pinned chunks -> HBM ->
    # taps in pinned host memory (N=1 only: a host-I/O leg with per-rank temp files)
    ingest = None
    if not args.no_e2e and args.file_frames > 0:
        if world > 1:
            ingest = {"skipped": "host-I/O leg measured at N=1 only (per-rank temp files)"}
        else:
            try:
                ingest = ingest_leg(corr, iq, taps, w, min(args.file_frames, F), rank)
            except OSError as exc:   # no room for the temp file: report, do not fail the bench
                ingest = {"skipped": f"{type(exc).__name__}: {exc}"[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, cores, sample, _ = cpu_reference_rate(w, seconds=args.cpu_seconds)
        cpu = {"value": rate, "unit": "CSI estimates/s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "CSI estimates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "us_per_frame": ms_per_step * 1e3 / F, "frames_per_s": frames_per_s,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.dtype,
            "data": f"synthetic: {F} distinct frame-sets from the device synthesiser (draw_channel law, "
                    f"pilot sweep, {w['snr_db']:g} dB AWGN; {synth_s:.2f} s, untimed)",
            "config": dict(CONFIG),
            "run": {"frames_per_step": F, "launch_frames": launch_frames, "input_bytes_per_step": iq.numel() * 4,
                       "parallelism": f"dp{world} (frames sharded, no hot-path collective)",
                       "dist_backend": args.dist_backend if world > 1 else None,
                       "distinct_devices": min(world, torch.cuda.device_count())},
            "tensor_pct_of_peak": 100 * achieved_tf / tf_burst,
            "kernels": {"k_correlate_fused_ms": t_kernel * 1e3, "tflops": achieved_tf, "gbs": achieved_gbs},
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": achieved_gbs / hbm, "traffic": traffic,
                         "peak_source": f"{peak_src} HBM copy bandwidth",
                         "tensor_frac": achieved_tf / tf_burst,
                         "tensor_frac_sustained": (achieved_tf / tf_sust) if tf_sust else None,
                         "algorithmic": {"flop_per_frame": flop_f, "bytes_per_frame": bytes_fused_f,
                                         "bytes": "f32 CP-stripped body in + complex64 taps out",
                                         "frames_per_launch": F}},
            "gemm_leg": gemm,
            "estimate_quality": quality,
            "tensor16_leg": t16,
            "cfg4_leg": c4,
            "latency": lat,
            "antenna_split": ant,
            "cpu_baseline": cpu, "e2e": e2e, "ingest_iq_file": ingest, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=10000, help="frame-sets per step per GPU")
    ap.add_argument("--dtype", default="fp16", choices=["fp16", "bf16"])
    ap.add_argument("--e2e-frames", type=int, default=512)
    ap.add_argument("--e2e-chunk", type=int, default=8, help="frame-sets per H2D/compute/D2H pipeline stage")
    ap.add_argument("--file-frames", type=int, default=256, help="frame-sets in the IQ-file ingest leg (0: off)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gemm-leg", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="skip the fused-scoring quality pass")
    ap.add_argument("--scored-frames", type=int, default=2048, help="frame-sets in the fused-scoring pass")
    ap.add_argument("--gemm-frames", type=int, default=4096)
    ap.add_argument("--cfg4-frames", type=int, default=256, help="frame-sets in the cfg4' leg (0: off)")
    ap.add_argument("--latency-reps", type=int, default=50, help="single frame-set latency samples (0: off)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend under torchrun (gloo: several ranks may share one GPU)")
    ap.add_argument("--antenna-reps", type=int, default=50, help="antenna-sharded latency samples (0: off)")
    ap.add_argument("--launch-frames", type=int, default=0, help="frame-sets per fused launch in a step (0: all)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
        dist.init_process_group(args.dist_backend)
    try:
        return run_gpu(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
