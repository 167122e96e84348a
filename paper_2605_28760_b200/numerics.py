"""Keyed direction streams, digests and the canonical mean -- the
``zoserve.numerics`` surface (numerics.py:17-37) on the B200 engine.

* ``sample_gaussian`` / ``gaussian_vector`` run the bit-exact device sampler
  (csrc/sampler.cu): SeedSequence -> Philox4x64-10 -> numpy's ziggurat.
* digests are FNV-1a-64 in libzob200's host code (thread-safe, GIL released).
* ``sample_indices`` is host data prep (16 indices per step) and uses numpy's
  Generator exactly as the reference does (numerics.py:177-181).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib
from .errors import ConfigError, DimensionError, InputError  # noqa: F401  (re-exported)

FNV_OFFSET_BASIS = 0xCBF29CE484222325
_MASK = (1 << 64) - 1

__all__ = [
    "DimensionError", "ConfigError", "InputError", "Role", "StreamKey", "sample_gaussian",
    "gaussian_vector", "sample_indices", "FNV_OFFSET_BASIS", "digest_bytes", "digest_array",
    "digest_text", "digest_hex", "canonical_mean",
]


# ---------------------------------------------------------------- digests
def digest_bytes(data: bytes, h: int = FNV_OFFSET_BASIS) -> int:
    """FNV-1a-64 over raw bytes chained from ``h`` (numerics.py:96-99)."""
    b = bytes(data)
    return int(lib().zo_fnv1a64(ctypes.c_char_p(b), len(b), h & _MASK))


def digest_array(a: np.ndarray, h: int = FNV_OFFSET_BASIS) -> int:
    """FNV-1a-64 over the little-endian float64 bytes of ``a`` (numerics.py:102-111)."""
    arr = np.ascontiguousarray(a, dtype="<f8")
    return int(lib().zo_fnv1a64(arr.ctypes.data, arr.nbytes, h & _MASK))


def digest_text(s: str, h: int = FNV_OFFSET_BASIS) -> int:
    return digest_bytes(s.encode("utf-8"), h)


def digest_hex(h: int) -> str:
    return f"{h & _MASK:016x}"


# ---------------------------------------------------------------- streams
class Role(enum.IntEnum):
    """Stream purpose, part of the key (numerics.py:128-136)."""
    U = 0
    V = 1
    DENSE_Z = 2
    MINIBATCH = 3
    INIT = 4


@dataclass(frozen=True)
class StreamKey:
    """(seed, step, layer_id, role) address of one stream (numerics.py:139-158)."""
    seed: int
    step: int
    layer_id: str
    role: Role

    def __post_init__(self) -> None:
        if self.seed < 0 or self.step < 0:
            raise ConfigError("seed and step must be non-negative")

    @property
    def lid_hash(self) -> int:
        return digest_text(self.layer_id)

    def generator(self) -> np.random.Generator:
        """Host numpy generator of the same stream (used for host data prep)."""
        ent = [self.seed, self.step, self.lid_hash, int(self.role)]
        return np.random.Generator(np.random.Philox(np.random.SeedSequence(ent)))


def _device_stream(key: StreamKey, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    check(lib().zo_sample_stream(None, key.seed, key.step, key.lid_hash, int(key.role), n, out.ctypes.data))
    return out


def sample_gaussian(key: StreamKey, rows: int, cols: int) -> np.ndarray:
    """Standard-normal (rows, cols) float64 matrix for ``key``, sampled on the
    GPU bit-identically to numpy's Philox/ziggurat stream (numerics.py:161-168)."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"gaussian sample needs rows, cols >= 1, got {rows}x{cols}")
    return _device_stream(key, rows * cols).reshape(rows, cols)


def gaussian_vector(key: StreamKey, n: int) -> np.ndarray:
    if n < 1:
        raise DimensionError(f"gaussian vector needs n >= 1, got {n}")
    return _device_stream(key, n)


def sample_indices(key: StreamKey, count: int, upper: int) -> np.ndarray:
    """``count`` int64 indices uniform over [0, upper) (numerics.py:177-181)."""
    if count < 1 or upper < 1:
        raise DimensionError("index sample needs count >= 1 and upper >= 1")
    return key.generator().integers(0, upper, size=count, dtype=np.int64)


# ---------------------------------------------------------------- reductions
def canonical_mean(values) -> float:
    """Float64 mean by recursive halving (left half = n // 2), so a batch
    concatenated with itself has the same mean bit for bit (numerics.py:271-284).
    The device coefficient kernel (csrc/zo_kernels.cu k_coefficient) uses the
    same tree."""
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    if v.size == 0:
        raise DimensionError("canonical_mean of empty batch")

    def tree(lo: int, n: int) -> float:
        if n == 1:
            return float(v[lo])
        h = n // 2
        return tree(lo, h) + tree(lo + h, n - h)

    return tree(0, v.size) / v.size
