"""Full-scale parity checks of one in-memory GPU dedup against the CPU side
(TEST INFRASTRUCTURE ONLY: tests/test_gpu_scale.py and scripts/verify_full.py).

  gpu_dedup_device   nd_dedup_device on device-resident text, then every
                     signature row, band id, distinct pair and group fetched
  check_signatures   signature rows + band ids recomputed by the REFERENCE
                     ITSELF (oracle/_ref: signature_of_document +
                     band_bucket_ids through parallel_for_index), all rows or
                     every `stride`-th row, chunk by chunk from the same bytes
  check_pairs        cells rebuilt on the CPU from the band ids (oracle/verify.c
                     ov_cells = scan_gather's grouping, sigstore.cpp:228-286),
                     every candidate pair of every cell compared by the C
                     oracle (compare_bucket with the reference oracle's exact
                     early exit, compare.cpp:24-67 / oracle.cpp:81-92), distinct
                     (lo, hi, match) vs the GPU's; candidate_pairs vs the GPU's
                     counter (pipeline.cpp:406-411)
  check_groups       components by the oracle's union-find (dedup_graph.cpp:48-81)
                     vs the GPU's groups (rep = min member)
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from oracle_bind import Oracle, Ref, u32p, u64p


def gpu_dedup_device(ctx, lib, _lib, d_text, d_offs, docs, params, H, B):
    stats = _lib.NdDedupStats()
    ctx.check(lib.nd_dedup_device(ctx.h, C.c_void_p(d_text.data_ptr()), C.c_void_p(d_offs.data_ptr()),
                                  None, docs, C.byref(params), C.byref(stats)))
    sig = np.empty((docs, H), np.uint32)
    band = np.empty((docs, B), np.uint32)
    ctx.check(lib.nd_dedup_fetch_signatures(ctx.h, sig.ctypes.data_as(u32p),
                                            band.ctypes.data_as(u32p)))
    d = stats.distinct_pairs
    plo, phi = np.empty(d, np.uint64), np.empty(d, np.uint64)
    pm = np.empty(d, np.uint32)
    ctx.check(lib.nd_dedup_fetch_pairs(ctx.h, plo.ctypes.data_as(u64p), phi.ctypes.data_as(u64p),
                                       pm.ctypes.data_as(u32p)))
    gmem = np.empty(stats.near_duplicates, np.uint64)
    gst = np.empty(stats.duplicate_groups + 1, np.uint64)
    ctx.check(lib.nd_dedup_fetch_groups(ctx.h, gmem.ctypes.data_as(u64p), gst.ctypes.data_as(u64p)))
    return stats, sig, band, (plo, phi, pm), (gmem, gst)


def check_signatures(text_chunk, offs, sig, band, H, B, rows, K, stride=1, chunk=500_000,
                     threads=None, seed=5, L=5):
    """text_chunk(c0, c1) -> host bytes of docs [c0, c1) (offsets relative to
    offs[c0]).  Returns (rows checked, rows differing, band rows differing)."""
    ref = Ref()
    threads = threads or os.cpu_count()
    docs = len(offs) - 1
    checked = bad_sig = bad_band = 0
    for c0 in range(0, docs, chunk):
        c1 = min(docs, c0 + chunk)
        text = text_chunk(c0, c1)
        co = (offs[c0:c1 + 1] - offs[c0]).astype(np.int64)
        sel = np.arange(c0 + (-c0) % stride, c1, stride) - c0
        if stride == 1:
            sub, so = text, co.astype(np.uint64)
        else:
            lens = co[sel + 1] - co[sel]
            so = np.zeros(len(sel) + 1, np.uint64)
            np.cumsum(lens, out=so[1:])
            sub = np.concatenate([text[co[i]:co[i + 1]] for i in sel]) if len(sel) else text[:0]
        rs, rb = ref.signatures(np.ascontiguousarray(sub), so, seed=seed, H=H, L=L, bands=B,
                                rows=rows, K=K, workers=threads)
        checked += len(sel)
        bad_sig += int((rs != sig[c0 + sel]).any(axis=1).sum())
        bad_band += int((rb != band[c0 + sel]).any(axis=1).sum())
    return checked, bad_sig, bad_band


def check_pairs(sig, band, K, num, den, pairs, threads=None):
    """Every candidate pair through the C oracle; returns a dict."""
    threads = threads or os.cpu_count()
    o = Oracle()
    L = o.lib
    L.ov_cells.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint32, u64p, u32p]
    L.ov_compare_cells.argtypes = [u32p, C.c_uint32, u64p, u32p, C.c_uint64, C.c_uint64,
                                   C.c_uint64, C.c_int, C.POINTER(u32p), C.POINTER(u32p),
                                   C.POINTER(u32p), u64p]
    L.ov_compare_cells.restype = C.c_int64
    L.ov_free.argtypes = [C.c_void_p]
    docs, B = band.shape
    H = sig.shape[1]
    t = time.time()
    cells = B * K
    coff = np.empty(cells + 1, np.uint64)
    rows = np.empty(docs * B, np.uint32)
    assert L.ov_cells(band.ctypes.data_as(u32p), docs, B, K, coff.ctypes.data_as(u64p),
                      rows.ctypes.data_as(u32p)) == 0
    lo_p, hi_p, m_p, cand = u32p(), u32p(), u32p(), C.c_uint64()
    k = L.ov_compare_cells(sig.ctypes.data_as(u32p), H, coff.ctypes.data_as(u64p),
                           rows.ctypes.data_as(u32p), cells, num, den, threads, C.byref(lo_p),
                           C.byref(hi_p), C.byref(m_p), C.byref(cand))
    assert k >= 0
    olo = np.ctypeslib.as_array(lo_p, (max(k, 1),))[:k].astype(np.uint64)
    ohi = np.ctypeslib.as_array(hi_p, (max(k, 1),))[:k].astype(np.uint64)
    om = np.ctypeslib.as_array(m_p, (max(k, 1),))[:k].copy()
    for p in (lo_p, hi_p, m_p):
        L.ov_free(p)
    key = (olo << np.uint64(32)) | ohi
    order = np.argsort(key, kind="stable")
    key, om = key[order], om[order]
    first = np.r_[True, key[1:] != key[:-1]] if len(key) else np.zeros(0, bool)
    key, om = key[first], om[first]
    plo, phi, pm = pairs
    gkey = (plo << np.uint64(32)) | phi
    return {"candidate_pairs_oracle": int(cand.value), "emitted_pairs_oracle": int(k),
            "distinct_pairs_oracle": int(len(key)),
            "pairs_identical": bool(np.array_equal(key, gkey) and np.array_equal(om, pm)),
            "oracle_compare_seconds": time.time() - t, "_keys": key}


def check_groups(keys, docs, groups):
    o = Oracle()
    lab = np.empty(docs, np.uint32)
    lo32 = (keys >> np.uint64(32)).astype(np.uint32)
    hi32 = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    o.lib.or_components(lo32.ctypes.data_as(u32p), hi32.ctypes.data_as(u32p), len(keys), docs,
                        lab.ctypes.data_as(u32p))
    gmem, gst = groups
    glab = np.full(docs, 0xFFFFFFFF, np.uint32)
    sizes = np.diff(gst).astype(np.int64)
    reps = gmem[gst[:-1].astype(np.int64)]
    glab[gmem.astype(np.int64)] = np.repeat(reps, sizes).astype(np.uint32)
    return {"groups_oracle": int(len(np.unique(lab[lab != 0xFFFFFFFF]))),
            "groups_identical": bool(np.array_equal(lab, glab))}
