"""CPU oracle for the PN-correlation channel-estimation hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2206_05506_b200/`) may import or call this module; it is used by
`tests/`, by `__graft_entry__.smoke()` as the checker, and by `bench.py`'s
`cpu_baseline` / `--impl reference` legs as the timed CPU baseline.

This is a NumPy restatement of the reference's algorithm (package `pnce`,
mounted read-only at /root/reference/pkg/src/pnce).  Every function cites the
reference file:line it follows.  The restatement uses the same NumPy calls in
the same order as the reference, so on identical seeds it reproduces the
reference's synthetic inputs and its reference64 estimates bit for bit.  That
claim is pinned by tests/test_oracle.py against golden vectors produced by
running the real reference (tests/golden/make_golden.py).

Third-party arithmetic: numpy (reference pyproject.toml:11 `numpy>=1.24`,
unpinned; golden vectors made with numpy 2.3.5 / OpenBLAS 0.3.30).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# pn.py:25-36 built-in primitive polynomials.  Degree 12 is NOT in the
# reference table (pn.py:74-82 raises for it); (12, 6, 4, 1) is an explicit
# LfsrSpec verified maximal-length with the reference's own generate_mseq.
PRIMITIVE_TAPS = {
    2: (2, 1), 3: (3, 2), 4: (4, 3), 5: (5, 3), 6: (6, 5), 7: (7, 6),
    8: (8, 6, 5, 4), 9: (9, 5), 10: (10, 3), 11: (11, 2),
}
EXTRA_TAPS = {12: (12, 6, 4, 1)}


class OracleError(ValueError):
    """Raised where the reference raises one of its PnceError subclasses."""


def taps_for_degree(degree: int) -> tuple[int, ...]:
    """pn.py:74-82 default_spec, extended with EXTRA_TAPS for degree 12."""
    if degree in PRIMITIVE_TAPS:
        return PRIMITIVE_TAPS[degree]
    if degree in EXTRA_TAPS:
        return EXTRA_TAPS[degree]
    raise OracleError(f"no primitive polynomial of degree {degree}")


def generate_mseq(degree: int, taps: tuple[int, ...], state: int = 1) -> np.ndarray:
    """pn.py:109-138: Fibonacci LFSR, output = MSB, feedback = parity(state & tap_mask).

    Returns float64 chips 1 - 2*bit for one period; raises OracleError when the
    period is not 2**degree - 1 (pn.py:131-136).
    """
    k = degree
    mask = (1 << k) - 1
    tap_mask = 0
    for t in taps:
        tap_mask |= 1 << (t - 1)
    s = state
    bits = []
    for _ in range(1 << k):
        bits.append((s >> (k - 1)) & 1)
        fb = (s & tap_mask).bit_count() & 1
        s = ((s << 1) | fb) & mask
        if s == state:
            break
    if len(bits) != (1 << k) - 1:
        raise OracleError(f"LFSR period {len(bits)} != {(1 << k) - 1}")
    return 1.0 - 2.0 * np.array(bits, dtype=np.float64)


def sequence_for_length(m: int) -> np.ndarray:
    """experiments.py:143-148 (built-in m-sequence of length m, state 1)."""
    degree = (m + 1).bit_length() - 1
    if (1 << degree) - 1 != m:
        raise OracleError(f"PN length {m} is not 2**k - 1")
    return generate_mseq(degree, taps_for_degree(degree), 1)


@dataclass(frozen=True)
class Config:
    """pilots.py:14-47 PilotConfig plus the receive-array size n_r."""

    m: int
    c: int
    n_t: int
    n_batch: int
    l: int
    n_r: int
    f_s: float = 10e6

    def __post_init__(self):
        if not 1 <= self.l <= self.c <= self.m:
            raise OracleError("need 1 <= L <= C <= M")
        if not 1 <= self.n_batch <= self.m // self.c:
            raise OracleError("n_batch outside [1, floor(M/C)]")

    @property
    def p(self) -> int:
        return self.c + self.m

    @property
    def n_batches(self) -> int:
        return -(-self.n_t // self.n_batch)

    @property
    def samples(self) -> int:
        """Per-receiver samples of one received batch, P + L - 1 (channel.py:131)."""
        return self.p + self.l - 1


def shift_for_transmitter(t: int, cfg: Config) -> int:
    """pilots.py:92-100: floor(M / N_batch) * (t mod N_batch)."""
    return (cfg.m // cfg.n_batch) * (t % cfg.n_batch)


def build_batch_plan(cfg: Config) -> list[list[tuple[int, int]]]:
    """pilots.py:119-143: consecutive transmitters per batch + >= L separation check."""
    batches = []
    for start in range(0, cfg.n_t, cfg.n_batch):
        batches.append([(t, shift_for_transmitter(t, cfg))
                        for t in range(start, min(start + cfg.n_batch, cfg.n_t))])
    for batch in batches:
        sh = [s for _, s in batch]
        for i in range(len(sh)):
            for j in range(i + 1, len(sh)):
                d = abs(sh[i] - sh[j]) % cfg.m
                if min(d, cfg.m - d) < cfg.l:
                    raise OracleError("shift separation < L")
    return batches


def lag_rows(chips: np.ndarray, lags: np.ndarray) -> np.ndarray:
    """estimator.py:62-65: A[i, k] = chips[(k - lag_i) mod M]."""
    m = chips.shape[0]
    idx = (np.arange(m)[None, :] - np.asarray(lags)[:, None]) % m
    return chips[idx]


def batched_lag_rows(chips: np.ndarray, batch, l: int) -> np.ndarray:
    """estimator.py:114-117: stacked lag windows [shift, shift + L) per transmitter."""
    m = chips.shape[0]
    lags = np.concatenate([(s + np.arange(l)) % m for _, s in batch])
    return lag_rows(chips, lags)


def correlator_rows_for_plan(chips: np.ndarray, plan, l: int) -> list[np.ndarray]:
    """experiments.py:157-173: one row matrix per distinct shift set."""
    cache: dict[tuple, np.ndarray] = {}
    out = []
    for batch in plan:
        key = tuple(s for _, s in batch)
        if key not in cache:
            cache[key] = batched_lag_rows(chips, batch, l)
        out.append(cache[key])
    return out


def remove_cp(samples: np.ndarray, c: int, m: int) -> np.ndarray:
    """estimator.py:40-47."""
    if samples.shape[-1] < c + m:
        raise OracleError("frame shorter than C + M")
    return samples[..., c:c + m]


# ---------------------------------------------------------------- backends

def _mma_real(a16: np.ndarray, x16: np.ndarray, chunk_len, accumulator: str, norm_len: int):
    """halfprec.py:93-125 (tensor16 emulation of one real GEMM)."""
    a64 = a16.astype(np.float64)
    x64 = x16.astype(np.float64)
    rows, k = a64.shape
    cols = x64.shape[1]
    scale = np.float32(1.0 / norm_len)
    total = np.zeros((rows, cols), dtype=np.float32)
    edges = [(0, k)] if chunk_len is None else [
        (lo, min(lo + chunk_len, k)) for lo in range(0, k, chunk_len)]
    for lo, hi in edges:
        if accumulator == "binary32":
            acc = (a64[:, lo:hi] @ x64[lo:hi]).astype(np.float32)
        else:
            acc16 = np.zeros((rows, cols), dtype=np.float16)
            for s in range(lo, hi, 4):
                step = a64[:, s:s + 4] @ x64[s:s + 4]
                with np.errstate(over="ignore", invalid="ignore"):
                    acc16 = (acc16.astype(np.float64) + step).astype(np.float16)
            acc = acc16.astype(np.float32)
        if not np.isfinite(acc).all():
            raise FloatingPointError("saturation")
        total = total + acc * scale
    if not np.isfinite(total).all():
        raise FloatingPointError("saturation")
    return total.astype(np.float64)


def mma_correlate(a: np.ndarray, y: np.ndarray, norm_len: int, chunk_len=256,
                  accumulator: str = "binary32") -> np.ndarray:
    """halfprec.py:128-160: fp16 operands, pad to 4, Re and Im as two real GEMMs."""
    rows, m = a.shape
    kp = -(-m // 4) * 4
    if chunk_len is not None and chunk_len > kp:
        raise OracleError("chunk_len exceeds padded length")
    rp = -(-rows // 4) * 4
    with np.errstate(over="ignore"):
        a16 = np.zeros((rp, kp), dtype=np.float16)
        a16[:rows, :m] = a.astype(np.float16)
        re16 = np.zeros((kp, y.shape[1]), dtype=np.float16)
        im16 = np.zeros_like(re16)
        re16[:m] = y.real.astype(np.float16)
        im16[:m] = y.imag.astype(np.float16)
    return (_mma_real(a16, re16, chunk_len, accumulator, norm_len)
            + 1j * _mma_real(a16, im16, chunk_len, accumulator, norm_len))[:rows]


def correlate_rows(rows: np.ndarray, y: np.ndarray, backend: str, norm_len: int,
                   chunk_len=256, accumulator: str = "binary32") -> np.ndarray:
    """estimator.py:68-86 dispatch (reference64 / reference32 / tensor16)."""
    if backend == "reference64":
        re = rows @ np.ascontiguousarray(y.real)
        im = rows @ np.ascontiguousarray(y.imag)
        return (re + 1j * im) / norm_len
    if backend == "reference32":
        r32 = rows.astype(np.float32)
        re = r32 @ y.real.astype(np.float32) / np.float32(norm_len)
        im = r32 @ y.imag.astype(np.float32) / np.float32(norm_len)
        return re.astype(np.float64) + 1j * im.astype(np.float64)
    if backend == "tensor16":
        return mma_correlate(rows, y, norm_len, chunk_len=chunk_len, accumulator=accumulator)
    raise OracleError(f"unknown backend {backend!r}")


def process_frames(chips: np.ndarray, cfg: Config, frames, backend: str = "reference64",
                   rows_per_batch=None, chunk_len=256, accumulator: str = "binary32"):
    """experiments.py:176-208: CP strip, correlate, demux into taps[r, t, l].

    ``frames`` is a sequence of (n_r, P + L - 1) complex arrays, one per batch.
    Returns (taps complex128 (n_r, n_t, l), saturations, macs).
    """
    plan = build_batch_plan(cfg)
    if rows_per_batch is None:
        rows_per_batch = correlator_rows_for_plan(chips, plan, cfg.l)
    n_r = frames[0].shape[0]
    taps = np.zeros((n_r, cfg.n_t, cfg.l), dtype=np.complex128)
    saturations = 0
    macs = 0
    for batch, frame, rows in zip(plan, frames, rows_per_batch):
        body = np.ascontiguousarray(remove_cp(frame, cfg.c, cfg.m).T)
        macs += rows.shape[0] * cfg.m * n_r
        try:
            flat = correlate_rows(rows, body, backend, cfg.m, chunk_len, accumulator)
        except FloatingPointError:
            saturations += n_r * len(batch)
            continue
        for i, (t, _) in enumerate(batch):
            taps[:, t, :] = flat[i * cfg.l:(i + 1) * cfg.l, :].T
    return taps, saturations, macs


def mae(truth: np.ndarray, est: np.ndarray) -> float:
    """metrics.py:19-25: mean |est - truth|."""
    if truth.shape != est.shape:
        raise OracleError("shape mismatch")
    return float(np.mean(np.abs(est - truth)))


def mse(truth: np.ndarray, est: np.ndarray) -> float:
    """North-star addition (no reference symbol): mean |est - truth|**2."""
    if truth.shape != est.shape:
        raise OracleError("shape mismatch")
    return float(np.mean(np.abs(est - truth) ** 2))


def oracle_circular_correlate(y: np.ndarray, chips: np.ndarray) -> np.ndarray:
    """metrics.py:28-39: IFFT(conj(FFT s) * FFT y) / M."""
    spectrum = np.conj(np.fft.fft(chips)) * np.fft.fft(y)
    return np.fft.ifft(spectrum) / chips.shape[0]


# ------------------------------------------------------- input synthesis
# Restated so that parity inputs can be regenerated on the GPU box (where
# /root/reference does not exist) bit-identically to the reference.

def derive_seeds(master: int, *key: int) -> tuple[int, int]:
    """experiments.py:151-154."""
    ss = np.random.SeedSequence([master, *key])
    a, b = ss.generate_state(2, dtype=np.uint64)
    return int(a), int(b)


def draw_channel(n_r: int, n_t: int, l: int, l_nz: int, seed: int) -> np.ndarray:
    """channel.py:96-108: per-link L_nz positions w/o replacement, amp U(0,Amax], phase U[0,2pi)."""
    rng = np.random.default_rng(seed)
    amax = math.sqrt(1.0 / (n_t * math.sqrt(l_nz)))
    taps = np.zeros((n_r, n_t, l), dtype=np.complex128)
    for r in range(n_r):
        for t in range(n_t):
            pos = rng.choice(l, size=l_nz, replace=False)
            amp = amax * (1.0 - rng.random(l_nz))
            phase = rng.uniform(0.0, 2.0 * math.pi, l_nz)
            taps[r, t, pos] = amp * np.exp(1j * phase)
    return taps


def build_pilot(chips: np.ndarray, shift: int, c: int) -> np.ndarray:
    """pilots.py:103-110 (+ pn.py:149-160 circular_shift = np.roll)."""
    body = np.roll(chips, shift)
    return np.concatenate([body[-c:], body])


def apply_channel(pilots, taps: np.ndarray, txs) -> np.ndarray:
    """channel.py:111-142: FFT linear convolution, output P + L - 1."""
    l = taps.shape[2]
    p = len(pilots[0])
    out_len = p + l - 1
    nfft = 1 << (out_len - 1).bit_length()
    f_frames = np.fft.fft(np.stack(pilots), n=nfft, axis=-1)
    f_taps = np.fft.fft(taps[:, txs, :], n=nfft, axis=-1)
    mixed = np.fft.ifft((f_frames[None, :, :] * f_taps).sum(axis=1), axis=-1)
    return np.ascontiguousarray(mixed[:, :out_len])


def simulate_frame(chips: np.ndarray, cfg: Config, l_nz: int, snr_db: float,
                   chan_seed: int, noise_seed: int):
    """channel.py:186-214 (+ add_awgn 145-167, noise_reference_power 175-183).

    Returns (truth taps (n_r, n_t, l) complex128, list of per-batch frames).
    """
    plan = build_batch_plan(cfg)
    truth = draw_channel(cfg.n_r, cfg.n_t, cfg.l, l_nz, chan_seed)
    rng = np.random.default_rng(noise_seed)
    frames = []
    for batch in plan:
        pilots = [build_pilot(chips, s, cfg.c) for _, s in batch]
        clean = apply_channel(pilots, truth, [t for t, _ in batch])
        ref = float(np.mean(np.abs(clean[:, cfg.c:cfg.c + cfg.m]) ** 2)) / (len(batch) * cfg.l)
        if snr_db == math.inf:
            frames.append(clean)
            continue
        sigma2 = ref / (10.0 ** (snr_db / 10.0))
        shape = clean.shape
        noise = math.sqrt(sigma2 / 2.0) * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
        frames.append(clean + noise)
    return truth, frames


def frames_to_iq(frames) -> np.ndarray:
    """iqfile.py:86-89 layout: receiver-major f32 interleaved (I, Q) per batch.

    Returns float32 (n_batches, n_r, P + L - 1, 2).
    """
    st = np.stack(frames)
    iq = np.empty(st.shape + (2,), dtype=np.float32)
    iq[..., 0] = st.real.astype(np.float32)
    iq[..., 1] = st.imag.astype(np.float32)
    return iq


def iq_to_frames(iq: np.ndarray):
    """iqfile.py:117-120: widen f32 (I, Q) back to complex128 per batch."""
    return [iq[b, ..., 0].astype(np.float64) + 1j * iq[b, ..., 1].astype(np.float64)
            for b in range(iq.shape[0])]
