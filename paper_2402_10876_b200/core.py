"""Host-side carriers shared by prune, compress and matmul.

Restates the parts of ``tilesparse.core`` that sit on the TW/TEW path:

* :func:`as_matrix`   -- reference core.py:32-43 (float32 C-contiguous 2-D carrier)
* :func:`floor_count` -- reference core.py:46-60 (exact-rational floor with a 2**-48 guard)
* :class:`TileConfig` -- reference core.py:63-76
* :class:`IndexMask`  -- reference core.py:79-115
* :func:`synthetic_matrix` -- reference cli.py:52-56 (Philox Gaussian inputs, streams cli.py:47-49)

Everything here is plain numpy on the host: these are the offline prune /
compress steps whose integer outputs (masks, indices) must be bit-exact
with the reference.  Nothing on the GPU hot path lives in this module.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .errors import InvalidInputError

VALUE_DTYPE = np.dtype(np.float32)   # reference core.py:24
ACC_DTYPE = np.dtype(np.float64)     # reference core.py:25

# Philox stream ids used by the reference CLI (cli.py:47-49).
STREAM_WEIGHTS = 0
STREAM_INPUT = 1
STREAM_GRAD = 2

_GUARD_SHIFT = 48


def as_matrix(values) -> np.ndarray:
    """Return ``values`` as a C-contiguous float32 matrix with dims >= 1.

    Same contract as reference core.py:32-43; raises InvalidInputError.
    """
    out = np.ascontiguousarray(values, dtype=VALUE_DTYPE)
    if out.ndim != 2:
        raise InvalidInputError(f"matrix must be 2-D, got ndim={out.ndim}")
    rows, cols = out.shape
    if rows < 1 or cols < 1:
        raise InvalidInputError(f"matrix dims must be >= 1, got {out.shape}")
    return out


def floor_count(fraction: float, n: int) -> int:
    """``floor(fraction * n)`` in exact rational arithmetic (core.py:46-60).

    The float is converted exactly (``Fraction(float)``); if the product lies
    within ``product / 2**48`` *below* the next integer, that integer is
    returned instead, so decimal-intended fractions such as 0.37 count 37 of
    100.
    """
    if n < 0:
        raise InvalidInputError(f"count must be non-negative, got {n}")
    exact = Fraction(float(fraction)) * int(n)
    lower = math.floor(exact)
    if exact > 0:
        gap = lower + 1 - exact
        if gap <= exact / (1 << _GUARD_SHIFT):
            return lower + 1
    return lower


@dataclass(frozen=True)
class TileConfig:
    """Tile width ``granularity_g`` along N and the reference's input-row
    blocking ``input_tile_t`` (only recorded; never changes pruning)."""

    granularity_g: int = 128
    input_tile_t: int = 32

    def __post_init__(self):
        for name in ("granularity_g", "input_tile_t"):
            if int(getattr(self, name)) < 1:
                raise InvalidInputError(f"{name} must be >= 1, got {getattr(self, name)}")


@dataclass(frozen=True)
class IndexMask:
    """Strictly increasing kept indices out of ``domain_len`` slots."""

    domain_len: int
    kept: np.ndarray

    def __post_init__(self):
        if self.domain_len < 1:
            raise InvalidInputError(f"domain_len must be >= 1, got {self.domain_len}")
        idx = np.asarray(self.kept, dtype=np.int64).ravel()
        if idx.size:
            bad = idx[0] < 0 or idx[-1] >= self.domain_len or bool(np.any(idx[1:] <= idx[:-1]))
            if bad:
                raise InvalidInputError(
                    "kept indices must be strictly increasing and within the domain")
        idx.setflags(write=False)
        object.__setattr__(self, "kept", idx)

    @classmethod
    def from_bool(cls, flags) -> "IndexMask":
        flags = np.asarray(flags, dtype=bool).ravel()
        return cls(flags.size, np.flatnonzero(flags))

    @classmethod
    def full(cls, domain_len: int) -> "IndexMask":
        return cls(domain_len, np.arange(domain_len, dtype=np.int64))

    def to_bool(self) -> np.ndarray:
        out = np.zeros(self.domain_len, dtype=bool)
        out[self.kept] = True
        return out

    @property
    def n_kept(self) -> int:
        return int(self.kept.size)

    @property
    def density(self) -> float:
        return self.kept.size / self.domain_len


def synthetic_matrix(seed: int, rows: int, cols: int, stream: int = STREAM_WEIGHTS) -> np.ndarray:
    """Standard-normal float32 matrix from ``Philox(key=[seed, stream])``.

    Same generator, key layout and draw order as reference cli.py:52-56, so
    the same (seed, shape, stream) yields the same bytes on every host.
    """
    gen = np.random.Generator(np.random.Philox(key=np.array([seed, stream], dtype=np.uint64)))
    return gen.standard_normal((rows, cols)).astype(np.float32)


def round_to(values: np.ndarray, dtype: str = "fp16") -> np.ndarray:
    """Round float32 values once to fp16/bf16 and widen back to float32.

    The parity protocol feeds this rounded copy to both
    the reference and the GPU path, so masks are computed on identical data
    and the GEMM products are exact in fp32.
    """
    v = np.ascontiguousarray(values, dtype=np.float32)
    if dtype == "fp16":
        return v.astype(np.float16).astype(np.float32)
    if dtype == "bf16":
        bits = v.view(np.uint32).astype(np.uint64)
        # round-to-nearest-even on the upper 16 bits (NaNs stay NaN)
        rounded = ((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16
        out = rounded.astype(np.uint32).view(np.float32)
        return np.where(np.isnan(v), v, out).astype(np.float32)
    if dtype == "fp32":
        return v.copy()
    raise InvalidInputError(f"unknown dtype {dtype!r}; expected fp16, bf16 or fp32")
