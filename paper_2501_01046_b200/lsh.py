"""LSH banding -- mirror of the reference's lsh.hpp.

  BandingConfig          lsh.hpp:14-21
  BucketKey              lsh.hpp:24-29
  choose_bucket_count    lsh.hpp:33   (host C++, exact integer arithmetic)
  band_bucket_ids        lsh.hpp:38   (device; normally fused into the K1 epilogue)
  BandRange / band_partition  lsh.hpp:43-53
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from ._lib import check, u32p
from .device import Context, default_context


def _ratio(r) -> tuple[int, int]:
    if isinstance(r, tuple):
        return int(r[0]), int(r[1])
    f = Fraction(r).limit_denominator(10**9) if not isinstance(r, Fraction) else r
    return f.numerator, f.denominator


@dataclass
class BandingConfig:
    bands: int = 0
    rows: int = 0
    bucket_count: int = 0
    bucket_scale: tuple[int, int] = (2, 1)

    def hash_count(self) -> int:
        return self.bands * self.rows


@dataclass(frozen=True, order=True)
class BucketKey:
    band: int = 0
    bucket: int = 0


@dataclass(frozen=True)
class BandRange:
    first: int = 0
    last: int = 0

    def size(self) -> int:
        return self.last - self.first


def choose_bucket_count(doc_count: int, scale=(2, 1)) -> int:
    """K = max(1, ceil(scale * sqrt(N))) in exact integers (lsh.cpp:26-40)."""
    num, den = _ratio(scale)
    out = C.c_uint32()
    check(_lib.load().nd_choose_bucket_count(doc_count, num, den, C.byref(out)))
    return out.value


def band_bucket_ids(signatures, bands: int, rows: int, bucket_count: int,
                    ctx: Context | None = None) -> np.ndarray:
    """Band ids of one signature (1-D) or a batch (n x H) -- (sum of rows) mod K."""
    sig = np.ascontiguousarray(signatures, dtype=np.uint32)
    one = sig.ndim == 1
    sig2 = sig.reshape(1, -1) if one else sig
    if bucket_count == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "bucket count must be positive")
    ctx = ctx or default_context()
    out = np.empty((sig2.shape[0], bands), np.uint32)
    ctx.check(ctx.lib.nd_band_keys(ctx.h, sig2.ctypes.data_as(u32p), sig2.shape[0], sig2.shape[1],
                                   bands, rows, bucket_count, out.ctypes.data_as(u32p)))
    return out[0] if one else out


def band_partition(bands: int, workers: int) -> list[BandRange]:
    """lsh.cpp:62-72: contiguous balanced ranges; extra workers get empty ranges."""
    r = (C.c_uint32 * (2 * max(workers, 1)))()
    check(_lib.load().nd_band_partition(bands, workers, r))
    return [BandRange(r[2 * w], r[2 * w + 1]) for w in range(workers)]


def cell_partition(bands: int, bucket_count: int, shards: int) -> list[int]:
    """Owner ranges of cells (band*K + bucket) over shards (multi-GPU exchange)."""
    fc = (C.c_uint64 * (shards + 1))()
    check(_lib.load().nd_cell_partition(bands, bucket_count, shards, fc))
    return list(fc)
