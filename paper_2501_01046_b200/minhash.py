"""MinHash signatures on the GPU -- mirror of the reference's minhash.hpp.

Reference interface (include/neardup/minhash.hpp):
  HashFunctionParams  :17-25   -> HashFunctionParams (ctypes, byte-identical)
  HashFamily          :27-33   -> HashFamily
  derive_family       :42-43   -> derive_family        (host C++, libneardup_b200)
  Signature           :58-61   -> Signature
  ShortDocumentError  :63-66   -> ShortDocumentError
  signature_of_document :71    -> signature_of_document (K1 kernel, batch of one)
  signature_batch     :76-78   -> signature_batch       (K1 kernel)
The per-window helpers hash_window_direct / roll_next (:47, :53) are fused
into the K1 kernel (csrc/k_signature.cu) and have no standalone entry point.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import NdHashFn as HashFunctionParams
from ._lib import ShortDocumentError, check, u8p, u32p, u64p
from .device import Context, default_context

__all__ = ["ShingleUnit", "HashFunctionParams", "HashFamily", "derive_family", "CleanDocument",
           "mod_pow", "is_prime_u32", "hash_window_direct", "roll_next",
           "Signature", "ShortDocumentError", "signature_of_document", "signature_batch",
           "pack_documents", "signatures_packed", "signatures_device", "text_units"]


class ShingleUnit(enum.IntEnum):
    BYTE = 0       # ShingleUnit::kByte (text.hpp:23-26)
    CODEPOINT = 1  # ShingleUnit::kCodepoint (decoded on the GPU, k_utf8.cu)


@dataclass
class HashFamily:
    hash_count: int
    shingle_len: int
    unit: ShingleUnit
    seed: int
    functions: C.Array  # HashFunctionParams * hash_count

    def params(self) -> list[tuple[int, int, int, int, int]]:
        return [(f.modulus, f.base, f.base_inverse, f.base_power, f.reduce_factor)
                for f in self.functions]


def mod_pow(base: int, exp: int, mod: int) -> int:
    """minhash.cpp:10-20 (ConfigError for a zero modulus)."""
    out = C.c_uint64()
    check(_lib.load().nd_mod_pow(base, exp, mod, C.byref(out)))
    return out.value


def is_prime_u32(n: int) -> bool:
    """minhash.cpp:22-50: Miller-Rabin with bases {2, 3, 5, 7}."""
    return bool(_lib.load().nd_is_prime_u32(n))


def hash_window_direct(window, f: "HashFunctionParams") -> int:
    """minhash.cpp:111-119: sum c_i q^i mod p by Horner from the last unit."""
    w = np.ascontiguousarray(window, np.uint32)
    out = C.c_uint32()
    check(_lib.load().nd_hash_window_direct(w.ctypes.data_as(u32p), len(w), C.byref(f),
                                            C.byref(out)))
    return out.value


def roll_next(state: int, outgoing: int, incoming: int, f: "HashFunctionParams") -> int:
    """minhash.cpp:121-131: the Eq. 5 update."""
    return int(_lib.load().nd_roll_next(state, outgoing, incoming, C.byref(f)))


def derive_family(seed: int, hash_count: int, shingle_len: int,
                  unit: ShingleUnit = ShingleUnit.BYTE) -> HashFamily:
    """minhash.cpp:71-105 -- bit-identical family from mt19937_64(seed)."""
    lib = _lib.load()
    fns = (HashFunctionParams * max(hash_count, 1))()
    check(lib.nd_derive_family(seed, hash_count, shingle_len, int(unit), fns))
    return HashFamily(hash_count, shingle_len, ShingleUnit(unit), seed, fns)


@dataclass
class CleanDocument:
    """corpus.hpp:26-30 (text is NFC UTF-8; bytes or str)."""

    doc_id: int
    text: bytes | str
    char_count: int = 0


@dataclass
class Signature:
    doc_id: int
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


def _as_bytes(t: bytes | str) -> bytes:
    return t.encode("utf-8") if isinstance(t, str) else bytes(t)


def pack_documents(docs: Iterable[CleanDocument]):
    """Packed batch (the paper's text buffer + index buffer)."""
    texts = [_as_bytes(d.text) for d in docs]
    lens = np.fromiter((len(t) for t in texts), dtype=np.uint64, count=len(texts))
    offsets = np.zeros(len(texts) + 1, np.uint64)
    np.cumsum(lens, out=offsets[1:])
    data = np.frombuffer(b"".join(texts), dtype=np.uint8).copy() if texts else np.zeros(0, np.uint8)
    return data, offsets


def signatures_packed(data: np.ndarray, offsets: np.ndarray, family: HashFamily, bands: int = 0,
                      rows: int = 0, bucket_count: int = 0, ctx: Context | None = None,
                      sig_out: np.ndarray | None = None, band_out: np.ndarray | None = None,
                      want_bands: bool = True):
    """K1 over a host packed batch; returns (sig[n,H] u32, band[n,bands] u32 or None).

    bucket_count == 0 returns raw band row sums (K-independent)."""
    ctx = ctx or default_context()
    ctx.upload_family(family)
    data = np.ascontiguousarray(data, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = len(offsets) - 1
    H = family.hash_count
    sig = sig_out if sig_out is not None else np.empty((n, H), np.uint32)
    band = None
    if want_bands and bands:
        band = band_out if band_out is not None else np.empty((n, bands), np.uint32)
    dp = data.ctypes.data_as(u8p) if data.size else C.cast(C.c_char_p(b"\0"), u8p)
    ctx.check(ctx.lib.nd_signatures(ctx.h, dp, offsets.ctypes.data_as(u64p), n, bands, rows,
                                    bucket_count, sig.ctypes.data_as(u32p),
                                    band.ctypes.data_as(u32p) if band is not None else None))
    return sig, band


def signatures_device(d_bytes: int, d_offsets: int, n: int, family: HashFamily, d_sig: int,
                      d_band: int = 0, bands: int = 0, rows: int = 0, bucket_count: int = 0,
                      ctx: Context | None = None) -> None:
    """K1 on device-resident buffers (raw device pointers), async on ctx's stream."""
    ctx = ctx or default_context()
    ctx.upload_family(family)
    ctx.check(ctx.lib.nd_signatures_device(ctx.h, C.c_void_p(d_bytes), C.c_void_p(d_offsets), n,
                                           bands, rows, bucket_count, C.c_void_p(d_sig),
                                           C.c_void_p(d_band) if d_band else None))


def text_units(data: np.ndarray, offsets: np.ndarray, unit: ShingleUnit,
               ctx: Context | None = None, counts_only: bool = False):
    """text_units (text.hpp:32, text.cpp:101-122) over a packed batch, decoded on
    the GPU: returns (unit_offsets[n+1] u64, units u32 or None)."""
    ctx = ctx or default_context()
    data = np.ascontiguousarray(data, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = len(offsets) - 1
    uoff = np.zeros(n + 1, np.uint64)
    dp = data.ctypes.data_as(u8p) if data.size else C.cast(C.c_char_p(b"\0"), u8p)
    ctx.check(ctx.lib.nd_text_units(ctx.h, dp, offsets.ctypes.data_as(u64p), n, int(unit),
                                    uoff.ctypes.data_as(u64p), None))
    if counts_only:
        return uoff, None
    units = np.empty(int(uoff[-1]), np.uint32)
    if units.size:
        ctx.check(ctx.lib.nd_text_units(ctx.h, dp, offsets.ctypes.data_as(u64p), n, int(unit),
                                        uoff.ctypes.data_as(u64p), units.ctypes.data_as(u32p)))
    return uoff, units


def _unit_counts(docs: Sequence[CleanDocument], unit: ShingleUnit, ctx) -> np.ndarray:
    if unit == ShingleUnit.BYTE:
        return np.fromiter((len(_as_bytes(d.text)) for d in docs), np.uint64, len(docs))
    data, offsets = pack_documents(docs)
    uoff, _ = text_units(data, offsets, unit, ctx=ctx, counts_only=True)
    return np.diff(uoff)


def signature_batch(docs: Sequence[CleanDocument], family: HashFamily,
                    on_short: Callable[[int], None] | None = None,
                    ctx: Context | None = None) -> list[Signature]:
    """minhash.cpp:164-177: order preserved; short documents are skipped and
    reported through on_short, never emitted with sentinel values."""
    keep = []
    counts = _unit_counts(docs, family.unit, ctx) if docs else []
    for d, units in zip(docs, counts):
        if units < family.shingle_len:
            if on_short:
                on_short(d.doc_id)
            continue
        keep.append(d)
    if not keep:
        return []
    data, offsets = pack_documents(keep)
    sig, _ = signatures_packed(data, offsets, family, ctx=ctx, want_bands=False)
    return [Signature(d.doc_id, sig[i].copy()) for i, d in enumerate(keep)]


def signature_of_document(doc: CleanDocument, family: HashFamily,
                          ctx: Context | None = None) -> Signature:
    """minhash.cpp:133-162; raises ShortDocumentError without a full window."""
    n = int(_unit_counts([doc], family.unit, ctx)[0])
    if n < family.shingle_len:
        raise ShortDocumentError(_lib.ND_ERR_SHORT,
                                 f"document {doc.doc_id} has {n} units, needs {family.shingle_len}")
    return signature_batch([doc], family, ctx=ctx)[0]
