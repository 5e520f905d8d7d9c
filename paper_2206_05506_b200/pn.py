"""PN (m-sequence) generation on the device, mirroring pnce/pn.py.

`generate_mseq` runs the Fibonacci LFSR of pn.py:109-138 on the GPU through
the C ABI (pnce_generate_mseq); the chips stay resident in HBM as float32
+1/-1 (bit 0 -> +1, bit 1 -> -1, pn.py:137).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .errors import InvalidSpecError, ZeroStateError

# pn.py:25-36 (degree 12 is deliberately absent, exactly as in the reference;
# pass LfsrSpec(12, (12, 6, 4, 1)) explicitly for M = 4095).
PRIMITIVE_TAPS: dict[int, tuple[int, ...]] = {
    2: (2, 1), 3: (3, 2), 4: (4, 3), 5: (5, 3), 6: (6, 5), 7: (7, 6),
    8: (8, 6, 5, 4), 9: (9, 5), 10: (10, 3), 11: (11, 2),
}
MAX_DEGREE = 16


@dataclass(frozen=True)
class LfsrSpec:
    """pn.py:39-71: feedback taps (exponents, must include degree) + nonzero start state."""

    degree: int
    taps: tuple[int, ...]
    state: int = 1

    def __post_init__(self):
        if self.degree < 2:
            raise InvalidSpecError(f"degree must be >= 2, got {self.degree}")
        if self.degree > MAX_DEGREE:
            raise InvalidSpecError(f"degree must be <= {MAX_DEGREE} on the device LFSR")
        taps = tuple(sorted(set(int(t) for t in self.taps), reverse=True))
        object.__setattr__(self, "taps", taps)
        if not taps or any(t < 1 or t > self.degree for t in taps):
            raise InvalidSpecError(f"taps must lie in [1, {self.degree}], got {taps}")
        if self.degree not in taps:
            raise InvalidSpecError(f"tap set must include the degree {self.degree}")
        if self.state == 0:
            raise ZeroStateError("initial LFSR state must be nonzero")
        if not 0 < self.state < (1 << self.degree):
            raise InvalidSpecError(f"state must be a nonzero {self.degree}-bit value, got {self.state}")

    @property
    def period_target(self) -> int:
        return (1 << self.degree) - 1

    @property
    def tap_mask(self) -> int:
        mask = 0
        for t in self.taps:
            mask |= 1 << (t - 1)
        return mask


def default_spec(degree: int, state: int = 1) -> LfsrSpec:
    """pn.py:74-82."""
    try:
        taps = PRIMITIVE_TAPS[degree]
    except KeyError:
        raise InvalidSpecError(
            f"no built-in primitive polynomial of degree {degree}; supply taps explicitly") from None
    return LfsrSpec(degree=degree, taps=taps, state=state)


@dataclass(frozen=True, eq=False)
class PnSequence:
    """pn.py:85-106: bipolar chips (device float32 tensor) with their LfsrSpec."""

    chips: torch.Tensor
    spec: LfsrSpec | None = None

    def __len__(self) -> int:
        return int(self.chips.shape[0])

    @property
    def m(self) -> int:
        return int(self.chips.shape[0])

    def numpy(self):
        return self.chips.detach().cpu().double().numpy()


def generate_mseq(spec: LfsrSpec, device: torch.device | str | None = None) -> PnSequence:
    """pn.py:109-138 on the GPU; raises NotMaximalLengthError for non-primitive taps."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    m = spec.period_target
    chips = torch.empty(m, dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().pnce_generate_mseq(spec.degree, spec.tap_mask, spec.state,
                                                 ctypes.c_void_p(chips.data_ptr()), m,
                                                 ctypes.c_void_p(stream)))
    return PnSequence(chips=chips, spec=spec)


def sequence_for_length(m: int, device=None) -> PnSequence:
    """experiments.py:143-148: built-in m-sequence of length m."""
    degree = (m + 1).bit_length() - 1
    if (1 << degree) - 1 != m:
        raise InvalidSpecError(f"PN length {m} is not 2**k - 1")
    return generate_mseq(default_spec(degree), device)


def circular_autocorrelation(seq: PnSequence, lag: int) -> float:
    """pn.py:141-146: (1/M) sum_m s[m] s[(m + lag) mod M]."""
    from .errors import LagOutOfRangeError
    m = seq.m
    if not 0 <= lag < m:
        raise LagOutOfRangeError(f"lag {lag} outside [0, {m})")
    c = seq.chips.double()
    return float(torch.dot(c, torch.roll(c, -lag)).item() / m)


def circular_shift(seq: PnSequence, shift: int) -> PnSequence:
    """pn.py:149-160: cyclic delay by ``shift`` chips (chip 0 moves to index ``shift``)."""
    from .errors import ShiftOutOfRangeError
    m = seq.m
    if not 0 <= shift < m:
        raise ShiftOutOfRangeError(f"shift {shift} outside [0, {m})")
    return PnSequence(chips=torch.roll(seq.chips, shift), spec=seq.spec)
