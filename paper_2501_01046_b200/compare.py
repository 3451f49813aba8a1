"""Candidate comparison -- mirror of the reference's compare.hpp.

  DuplicatePair         compare.hpp:15-21
  signature_match_count compare.hpp:24   (host helper, test use)
  SimilarityThreshold   compare.hpp:28-37 (exact integer rule m*den > num*H)
  compare_bucket        compare.hpp:43   -> K3 kernel on one cell
  compare_pass          compare.hpp:49   -> K3 over all cells + sort/unique (K4a)
  write/read_pair_file  compare.hpp:56-57 (20-byte LE records)
GatheredBucket / GatherResult mirror sigstore.hpp:114-131.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import u32p, u64p
from .device import Context, default_context
from .lsh import BucketKey, _ratio


@dataclass(frozen=True)
class DuplicatePair:
    lo: int
    hi: int
    match_count: int


@dataclass
class SimilarityThreshold:
    value: tuple[int, int] = (4, 5)

    def __post_init__(self):
        self.value = _ratio(self.value)
        if self.value[1] == 0:
            raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "ratio denominator must be positive")

    def accepts(self, match_count: int, hash_count: int) -> bool:
        num, den = self.value
        return match_count * den > num * hash_count

    def min_matches(self, hash_count: int) -> int:
        num, den = self.value
        return int(_lib.load().nd_min_matches(hash_count, num, den))


def signature_match_count(a, b) -> int:
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                               f"signature length mismatch: {a.size} vs {b.size}")
    return int((a == b).sum())


@dataclass
class GatheredBucket:
    key: BucketKey = field(default_factory=BucketKey)
    doc_ids: list[int] = field(default_factory=list)
    signatures: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


@dataclass
class GatherResult:
    buckets: list[GatheredBucket] = field(default_factory=list)


def _compare_cells(buckets, hash_count: int, threshold: SimilarityThreshold, ctx):
    """K3 + K4a over the given cells; returns sorted distinct DuplicatePairs.

    Each distinct doc id becomes one signature row (rows ranked by doc id), so
    the same pair met in several cells collapses in the device-side unique and
    row order equals (lo, hi) doc-id order."""
    ctx = ctx or default_context()
    if hash_count <= 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "hash count must be positive")
    by_id: dict[int, np.ndarray] = {}
    cells = []
    for b in buckets:
        n = len(b.doc_ids)
        sig = np.ascontiguousarray(b.signatures, dtype=np.uint32).reshape(-1)
        if sig.size != n * hash_count:
            raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "gathered bucket shape mismatch")
        ids = [int(d) for d in b.doc_ids]
        for k, d in enumerate(ids):
            row = sig[k * hash_count:(k + 1) * hash_count]
            prev = by_id.setdefault(d, row)
            if prev is not row and not np.array_equal(prev, row):
                raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                                       f"doc {d} carries different signatures in two cells")
        cells.append(ids)
    if not by_id:
        return []
    order = sorted(by_id)
    rank = {d: i for i, d in enumerate(order)}
    sigs = np.ascontiguousarray(np.stack([by_id[d] for d in order]), dtype=np.uint32)
    offs = [0]
    rows = []
    for ids in cells:
        rows.extend(rank[d] for d in ids)
        offs.append(len(rows))
    offs_a = np.array(offs, np.uint64)
    rows_a = np.array(rows, np.uint32)
    npairs = C.c_uint64()
    num, den = threshold.value
    ctx.check(ctx.lib.nd_compare_cells(ctx.h, sigs.ctypes.data_as(u32p), sigs.shape[0], hash_count,
                                       offs_a.ctypes.data_as(u64p), rows_a.ctypes.data_as(u32p),
                                       len(offs) - 1, num, den, C.byref(npairs)))
    k = npairs.value
    lo = np.empty(k, np.uint32)
    hi = np.empty(k, np.uint32)
    m = np.empty(k, np.uint32)
    ctx.check(ctx.lib.nd_pairs_fetch(ctx.h, lo.ctypes.data_as(u32p), hi.ctypes.data_as(u32p),
                                     m.ctypes.data_as(u32p)))
    ids = np.array(order, np.uint64)
    return [DuplicatePair(int(a), int(b), int(c)) for a, b, c in zip(ids[lo], ids[hi], m)]


def compare_bucket(bucket: GatheredBucket, hash_count: int, threshold: SimilarityThreshold,
                   tile_size: int = 32, ctx: Context | None = None) -> list[DuplicatePair]:
    """compare.cpp:24-67: all accepted pairs (lo < hi) of one cell.  tile_size is
    accepted for API parity; the kernel's tiling is fixed (128 rows x 64 cols)."""
    if tile_size == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "tile size must be positive")
    return _compare_cells([bucket], hash_count, threshold, ctx)


def compare_pass(gathered: GatherResult, hash_count: int, threshold: SimilarityThreshold,
                 tile_size: int = 32, ctx: Context | None = None) -> list[DuplicatePair]:
    """compare.cpp:69-86: every cell, then sort by (lo, hi) and drop repeats."""
    if tile_size == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "tile size must be positive")
    return _compare_cells(gathered.buckets, hash_count, threshold, ctx)


def write_pair_file(path: str, pairs) -> None:
    """compare.cpp:88-99: bare little-endian (lo u64, hi u64, match u32) records."""
    with open(path, "wb") as f:
        for p in pairs:
            f.write(struct.pack("<QQI", p.lo, p.hi, p.match_count))


def read_pair_file(path: str) -> list[DuplicatePair]:
    """compare.cpp:101-113."""
    data = open(path, "rb").read()
    if len(data) % 20:
        raise _lib.IoError(_lib.ND_ERR_IO,
                           f"'{path}' is corrupt: size is not a multiple of the pair record")
    return [DuplicatePair(*struct.unpack_from("<QQI", data, o)) for o in range(0, len(data), 20)]
