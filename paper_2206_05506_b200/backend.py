"""Backend selection at the reference seam (pnce/halfprec.py:24-55 `BackendConfig`).

The reference dispatches `correlate_rows` / `process_frames` on
``BackendConfig.kind`` in {"reference64", "reference32", "tensor16"}.  Here there is
one device path with two arithmetic modes, so a reference caller's backend maps as:

* ``reference64`` / ``reference32`` -> the fused fp16 (or bf16) tensor-core path with
  fp32 accumulation and one x(1/M) in the epilogue.  Not bit-equal to float64/float32
  BLAS: the north-star tolerance applies (per tap |h - h_ref64| <= 1e-2 * max_l
  |h_ref64[r, t, :]|, MSE within 0.1 dB; measured ~1e-4 / < 0.001 dB with fp16).
* ``tensor16`` -> the tensor16 mode (halfprec.py:93-125 on real tensor cores):
  ``chunk_len``-sample chunks accumulated as binary32 or binary16 partials, each
  x fp32(1/M) into an fp32 total; a saturated (frame-set, batch) is scored as zeros and
  counted (n_r * n_tx) exactly as experiments.py:201-205 does.  Device chunks are whole
  64-sample K-blocks: ``chunk_len`` must be a multiple of 64 (the reference allows
  multiples of 4; others raise InvalidConfigError).

Plain strings "fp16" / "bf16" select the operand precision of the fused path directly.
Objects of the reference's own ``pnce.halfprec.BackendConfig`` class are accepted as
they are (duck-typed on ``kind``, ``chunk_len``, ``accumulator``).
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidConfigError

TILE = 4
KINDS = ("reference64", "reference32", "tensor16")
ACCUMULATORS = ("binary32", "binary16")
DTYPES = ("fp16", "bf16")


@dataclass(frozen=True)
class BackendConfig:
    """halfprec.py:29-55, same fields, defaults and validation."""

    kind: str = "reference64"
    tile: int = TILE
    chunk_len: int | None = 256
    accumulator: str = "binary32"

    def __post_init__(self):
        if self.kind not in KINDS:
            raise InvalidConfigError(f"unknown backend kind {self.kind!r}")
        if self.accumulator not in ACCUMULATORS:
            raise InvalidConfigError(f"unknown accumulator {self.accumulator!r}")
        if self.tile != TILE:
            raise InvalidConfigError(f"tile size is fixed at {TILE}")
        if self.chunk_len is not None:
            if self.chunk_len < self.tile or self.chunk_len % self.tile != 0:
                raise InvalidConfigError(
                    f"chunk_len must be a positive multiple of {self.tile}, got {self.chunk_len}")


REFERENCE64 = BackendConfig(kind="reference64")
REFERENCE32 = BackendConfig(kind="reference32")
TENSOR16 = BackendConfig(kind="tensor16")


@dataclass(frozen=True)
class Resolved:
    """What the device path runs for a requested backend."""

    kind: str                 # the reference kind reported in CirEstimate.backend
    dtype: str                # operand precision
    tensor16: bool
    chunk_len: int | None = None
    accumulator: str = "binary32"


def resolve(backend, dtype: str | None = None) -> Resolved:
    """Map None / "fp16" / "bf16" / a BackendConfig (ours or the reference's) to a device mode.

    ``dtype`` (e.g. a prebuilt Correlator's operand precision) overrides the default fp16
    for the reference kinds."""
    dt = dtype or "fp16"
    if dt not in DTYPES:
        raise InvalidConfigError(f"dtype must be one of {DTYPES}, got {dt!r}")
    if backend is None:
        return Resolved(kind=f"tcgen05-{dt}", dtype=dt, tensor16=False)
    if isinstance(backend, str):
        if backend in DTYPES:
            return Resolved(kind=f"tcgen05-{backend}", dtype=backend, tensor16=False)
        if backend in KINDS:
            backend = BackendConfig(kind=backend)
        else:
            raise InvalidConfigError(f"unknown backend {backend!r}")
    kind = getattr(backend, "kind", None)
    if kind not in KINDS:
        raise InvalidConfigError(f"unknown backend kind {kind!r}")
    if kind != "tensor16":
        return Resolved(kind=kind, dtype=dt, tensor16=False)
    acc = getattr(backend, "accumulator", "binary32")
    if acc not in ACCUMULATORS:
        raise InvalidConfigError(f"unknown accumulator {acc!r}")
    return Resolved(kind=kind, dtype=dt, tensor16=True, chunk_len=getattr(backend, "chunk_len", 256),
                    accumulator=acc)
