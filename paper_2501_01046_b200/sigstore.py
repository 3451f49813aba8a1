"""Signature store -- mirror of the reference's sigstore.hpp (+ the pair files
of compare.hpp).  The byte formats are written and parsed by the C++ side of
libneardup_b200 (csrc/host_feds.cpp), identical to the reference's:

  SignatureFileHeader      sigstore.hpp:24-42 (72-byte LE header "FEDS" v1)
  write_signature_file     sigstore.cpp:143-151 (SignatureFileWriter)
  read_signature_file      sigstore.cpp:153-163 (SignatureFileReader, size + bucket checks)
  plan_gather              sigstore.cpp:288-329
  write_pair_file / read_pair_file   compare.cpp:88-113 (20-byte records)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import NdFedsHeader, check, u32p, u64p
from .lsh import _ratio
from .minhash import ShingleUnit

SIGNATURE_MAGIC = b"FEDS"
SIGNATURE_VERSION = 1
SIGNATURE_HEADER_BYTES = 72


@dataclass
class SignatureFileHeader:
    hash_count: int = 0
    bands: int = 0
    rows: int = 0
    bucket_count: int = 0
    shingle_len: int = 0
    unit: ShingleUnit = ShingleUnit.BYTE
    family_seed: int = 0
    bucket_scale: tuple[int, int] = (2, 1)
    record_count: int = 0
    source_ordinal: int = 0

    def record_bytes(self) -> int:
        return 8 + 4 * self.hash_count + 4 * self.bands

    def run_compatible(self, other: "SignatureFileHeader") -> bool:
        from math import gcd

        def norm(r):
            n, d = _ratio(r)
            g = gcd(n, d) or 1
            n, d = n // g, d // g
            return (n, 1) if n == 0 else (n, d)

        return (self.hash_count, self.bands, self.rows, self.bucket_count, self.shingle_len,
                int(self.unit), self.family_seed, norm(self.bucket_scale)) == \
               (other.hash_count, other.bands, other.rows, other.bucket_count, other.shingle_len,
                int(other.unit), other.family_seed, norm(other.bucket_scale))

    def to_c(self) -> NdFedsHeader:
        n, d = _ratio(self.bucket_scale)
        return NdFedsHeader(hash_count=self.hash_count, bands=self.bands, rows=self.rows,
                            bucket_count=self.bucket_count, shingle_len=self.shingle_len,
                            unit=int(self.unit), family_seed=self.family_seed, scale_num=n,
                            scale_den=d, record_count=self.record_count,
                            source_ordinal=self.source_ordinal)

    @classmethod
    def from_c(cls, h: NdFedsHeader) -> "SignatureFileHeader":
        return cls(h.hash_count, h.bands, h.rows, h.bucket_count, h.shingle_len,
                   ShingleUnit(h.unit), h.family_seed, (h.scale_num, h.scale_den),
                   h.record_count, h.source_ordinal)


@dataclass
class SignatureRecord:
    doc_id: int
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    buckets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


def write_signature_file(path: str, header: SignatureFileHeader, doc_ids, values, buckets,
                         fsync_on_close: bool = False) -> None:
    """Columnar form: doc_ids[n] u64, values[n, H] u32, buckets[n, bands] u32."""
    ids = np.ascontiguousarray(doc_ids, np.uint64)
    v = np.ascontiguousarray(values, np.uint32).reshape(len(ids), header.hash_count)
    b = np.ascontiguousarray(buckets, np.uint32).reshape(len(ids), header.bands)
    check(_lib.load().nd_feds_write(path.encode(), C.byref(header.to_c()),
                                    ids.ctypes.data_as(u64p), v.ctypes.data_as(u32p),
                                    b.ctypes.data_as(u32p), len(ids), int(fsync_on_close)))


def read_signature_header(path: str) -> SignatureFileHeader:
    h = NdFedsHeader()
    check(_lib.load().nd_feds_read_header(path.encode(), C.byref(h)))
    return SignatureFileHeader.from_c(h)


def read_signature_file(path: str):
    """-> (header, doc_ids[n] u64, values[n, H] u32, buckets[n, bands] u32)."""
    h = read_signature_header(path)
    n = h.record_count
    ids = np.empty(n, np.uint64)
    v = np.empty((n, h.hash_count), np.uint32)
    b = np.empty((n, h.bands), np.uint32)
    check(_lib.load().nd_feds_read(path.encode(), ids.ctypes.data_as(u64p), v.ctypes.data_as(u32p),
                                   b.ctypes.data_as(u32p)))
    return h, ids, v, b


@dataclass
class GatherPlan:
    buckets_per_pass: int
    passes_per_worker: list[int]


def plan_gather(total_signature_bytes: int, bucket_count: int, bands: int, workers: int,
                memory_budget: int, override_buckets_per_pass: int | None = None) -> GatherPlan:
    """sigstore.cpp:288-329 over band_partition(bands, workers) (lsh.cpp:62-72)."""
    if override_buckets_per_pass is not None and override_buckets_per_pass < 1:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "buckets-per-pass override must be at least 1")
    c = C.c_uint32()
    passes = (C.c_uint32 * max(workers, 1))()
    check(_lib.load().nd_plan_gather(total_signature_bytes, bucket_count, bands, workers,
                                     memory_budget, override_buckets_per_pass or 0, C.byref(c),
                                     passes))
    return GatherPlan(c.value, list(passes)[:workers])


def write_pair_file(path: str, lo, hi, match_count, fsync_file: bool = False) -> None:
    lo = np.ascontiguousarray(lo, np.uint64)
    hi = np.ascontiguousarray(hi, np.uint64)
    m = np.ascontiguousarray(match_count, np.uint32)
    check(_lib.load().nd_pairs_write(path.encode(), lo.ctypes.data_as(u64p), hi.ctypes.data_as(u64p),
                                     m.ctypes.data_as(u32p), len(lo), int(fsync_file)))


def read_pair_file(path: str):
    """-> (lo u64, hi u64, match_count u32) columns."""
    lib = _lib.load()
    n = C.c_uint64(0)
    check(lib.nd_pairs_read(path.encode(), None, None, None, C.byref(n)))
    lo = np.empty(n.value, np.uint64)
    hi = np.empty(n.value, np.uint64)
    m = np.empty(n.value, np.uint32)
    if n.value:
        check(lib.nd_pairs_read(path.encode(), lo.ctypes.data_as(u64p), hi.ctypes.data_as(u64p),
                                m.ctypes.data_as(u32p), C.byref(n)))
    return lo, hi, m


def scan_gather(paths, expected: SignatureFileHeader, bands, bucket_first: int, bucket_last: int):
    """sigstore.cpp:228-286: one scan of the signature files keeping, per band in
    `bands` (an lsh.BandRange), the documents whose bucket lies in
    [bucket_first, bucket_last); cells of a single document are dropped.  Files
    must come in source order (doc ids ascending).  Returns a compare.GatherResult
    (buckets sorted by key, doc ids ascending).  Host reference-API form; the
    compare stage itself groups every cell on the GPU (nd_compare_stage)."""
    from .compare import GatheredBucket, GatherResult
    from .lsh import BucketKey

    if bucket_last > expected.bucket_count or bucket_first > bucket_last:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "gather bucket interval out of range")
    if bands.last > expected.bands or bands.first > bands.last:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "gather band range out of range")
    width, rng = bucket_last - bucket_first, bands.last - bands.first
    if width == 0 or rng == 0:
        return GatherResult([])
    ids_l, sig_l, band_l = [], [], []
    for p in paths:
        h, ids, v, b = read_signature_file(p)
        if not h.run_compatible(expected):
            raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                                   f"'{p}' was written with different parameters than this run")
        ids_l.append(ids)
        sig_l.append(v)
        band_l.append(b)
    H = expected.hash_count
    ids = np.concatenate(ids_l) if ids_l else np.zeros(0, np.uint64)
    sig = np.concatenate(sig_l) if sig_l else np.zeros((0, H), np.uint32)
    band = np.concatenate(band_l) if band_l else np.zeros((0, expected.bands), np.uint32)
    out = []
    for j in range(bands.first, bands.last):
        col = band[:, j]
        for k in range(bucket_first, bucket_last):
            rows = np.flatnonzero(col == k)
            if len(rows) < 2:
                continue
            if (np.diff(ids[rows].astype(np.int64)) <= 0).any():
                raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "signature files are not in ascending "
                                                           "doc_id order; pass them in manifest order")
            out.append(GatheredBucket(BucketKey(j, k), ids[rows].tolist(), sig[rows].reshape(-1)))
    return GatherResult(out)
