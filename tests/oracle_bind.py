"""ctypes bindings for the parity checkers under oracle/ (TEST INFRASTRUCTURE ONLY).

``Oracle`` wraps oracle/liboracle.so (the C restatement, oracle/oracle.c).
``Ref`` wraps oracle/_ref/libneardup_ref.so (the reference's own sources
compiled in place by oracle/Makefile, bridged by oracle/ref_shim/ref_capi.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libneardup_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class HashFn(C.Structure):
    """Mirrors HashFunctionParams (minhash.hpp:17-25) and nd_hash_fn."""

    _fields_ = [
        ("modulus", C.c_uint32),
        ("base", C.c_uint32),
        ("base_inverse", C.c_uint32),
        ("base_power", C.c_uint32),
        ("reduce_factor", C.c_uint64),
    ]


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def family_array(fns) -> np.ndarray:
    """(H, 6) uint32 view: p, q, q^-1, q^(L-1), reduce_lo, reduce_hi."""
    raw = (C.c_uint8 * (24 * len(fns))).from_buffer_copy(bytes(fns))
    return np.frombuffer(raw, dtype=np.uint32).reshape(len(fns), 6).copy()


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build_oracle()
        L = C.CDLL(ORACLE_SO)
        L.or_derive_family.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(HashFn)]
        L.or_hash_window_direct.argtypes = [u32p, C.c_uint32, C.POINTER(HashFn)]
        L.or_hash_window_direct.restype = C.c_uint32
        L.or_roll_next.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(HashFn)]
        L.or_roll_next.restype = C.c_uint32
        L.or_signature_batch.argtypes = [u8p, u64p, C.c_uint64, C.POINTER(HashFn), C.c_uint32,
                                         C.c_uint32, u32p]
        L.or_signature_batch_unit.argtypes = [u8p, u64p, C.c_uint64, C.POINTER(HashFn),
                                              C.c_uint32, C.c_uint32, C.c_uint32, u32p]
        L.or_decode_codepoints.argtypes = [u8p, C.c_uint64, u32p, C.c_uint64]
        L.or_decode_codepoints.restype = C.c_uint64
        L.or_choose_bucket_count.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_choose_bucket_count.restype = C.c_uint32
        L.or_band_bucket_ids.argtypes = [u32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
        L.or_min_matches.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64]
        L.or_min_matches.restype = C.c_uint32
        L.or_accepts.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64]
        L.or_compare_cell.argtypes = [u32p, C.c_uint32, u32p, C.c_uint64, C.c_uint64, C.c_uint64,
                                      u32p, u32p, u32p, C.c_uint64]
        L.or_compare_cell.restype = C.c_uint64
        L.or_components.argtypes = [u32p, u32p, C.c_uint64, C.c_uint32, u32p]
        L.or_is_prime_u32.argtypes = [C.c_uint32]
        L.or_mod_pow.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_mod_pow.restype = C.c_uint64
        L.or_bounded_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u32p]
        self.lib = L

    def bounded_stream(self, seed: int, bound: int, n: int) -> np.ndarray:
        """n draws bounded_random(mt19937_64(seed), bound) (util.cpp:70-79)."""
        out = np.empty(n, np.uint32)
        self.lib.or_bounded_stream(seed, bound, n, _ptr(out, u32p))
        return out

    def derive_family(self, seed: int, H: int, L: int = 5):
        fns = (HashFn * H)()
        if self.lib.or_derive_family(seed, H, L, fns) != 0:
            raise ValueError("derive_family failed")
        return fns

    def signatures(self, data: np.ndarray, offsets: np.ndarray, fns, L: int = 5,
                   unit: int = 0) -> np.ndarray:
        n = len(offsets) - 1
        H = len(fns)
        out = np.zeros((n, H), dtype=np.uint32)
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        if unit == 0:
            rc = self.lib.or_signature_batch(_ptr(data, u8p), _ptr(offsets, u64p), n, fns, H, L,
                                             _ptr(out, u32p))
        else:
            rc = self.lib.or_signature_batch_unit(_ptr(data, u8p), _ptr(offsets, u64p), n, fns, H,
                                                  L, unit, _ptr(out, u32p))
        if rc != 0:
            raise ValueError("short document")
        return out

    def decode_codepoints(self, b: bytes) -> list[int]:
        a = np.frombuffer(b, np.uint8).copy() if b else np.zeros(1, np.uint8)
        out = np.zeros(max(1, len(b)), np.uint32)
        n = self.lib.or_decode_codepoints(_ptr(a, u8p), len(b), _ptr(out, u32p), len(out))
        return out[:n].tolist()

    def band_ids(self, sigs: np.ndarray, bands: int, rows: int, K: int) -> np.ndarray:
        sigs = np.ascontiguousarray(sigs, dtype=np.uint32)
        out = np.zeros((sigs.shape[0], bands), dtype=np.uint32)
        for i in range(sigs.shape[0]):
            self.lib.or_band_bucket_ids(_ptr(sigs[i], u32p), bands, rows, K, _ptr(out[i], u32p))
        return out

    def compare_cell(self, sigs: np.ndarray, rows: np.ndarray, num: int, den: int):
        sigs = np.ascontiguousarray(sigs, dtype=np.uint32)
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        n = len(rows)
        cap = max(1, n * (n - 1) // 2)
        lo = np.zeros(cap, np.uint32)
        hi = np.zeros(cap, np.uint32)
        m = np.zeros(cap, np.uint32)
        got = self.lib.or_compare_cell(_ptr(sigs, u32p), sigs.shape[1], _ptr(rows, u32p), n, num,
                                       den, _ptr(lo, u32p), _ptr(hi, u32p), _ptr(m, u32p), cap)
        return lo[:got], hi[:got], m[:got]

    def components(self, lo: np.ndarray, hi: np.ndarray, nnodes: int) -> np.ndarray:
        lo = np.ascontiguousarray(lo, np.uint32)
        hi = np.ascontiguousarray(hi, np.uint32)
        out = np.zeros(max(nnodes, 1), np.uint32)
        self.lib.or_components(_ptr(lo, u32p), _ptr(hi, u32p), len(lo), nnodes, _ptr(out, u32p))
        return out[:nnodes]


class Ref:
    """The reference implementation itself (oracle/_ref)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            build_oracle()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_derive_family.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.POINTER(HashFn)]
        L.ref_choose_bucket_count.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_choose_bucket_count.restype = C.c_uint32
        L.ref_min_matches.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64]
        L.ref_min_matches.restype = C.c_uint32
        L.ref_signatures.argtypes = [u8p, u64p, u64p, C.c_uint64, C.c_uint64, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                     C.c_uint, u32p, u32p]
        L.ref_compare_cells.argtypes = [u32p, u64p, C.c_uint32, u64p, u32p, C.c_uint64,
                                        C.c_uint64, C.c_uint64, C.c_uint32,
                                        C.POINTER(u64p), C.POINTER(u64p), C.POINTER(u32p),
                                        u64p]
        L.ref_all_pairs_dupset.argtypes = [u32p, u64p, C.c_uint64, C.c_uint32, C.c_uint64,
                                           C.c_uint64, C.c_uint, u64p, u64p]
        L.ref_union.argtypes = [u64p, u64p, C.c_uint64, C.POINTER(u64p), C.POINTER(u64p), u64p,
                                u64p]
        dp = C.POINTER(C.c_double)
        L.ref_compare_cells_timed.argtypes = [u32p, C.c_uint32, u64p, u32p, C.c_uint64,
                                              C.c_uint64, C.c_uint64, C.c_uint, dp, dp, dp, u64p,
                                              u64p, C.POINTER(u64p), C.POINTER(u64p)]
        L.ref_union_timed.argtypes = [u64p, u64p, C.c_uint64, dp, u64p, u64p]
        L.ref_generate_synthetic.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                             C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                             C.c_uint64, C.c_uint32, C.c_char_p, C.c_char_p,
                                             C.POINTER(u8p), C.POINTER(u64p), u64p]
        L.ref_run_dedup.argtypes = [C.c_char_p, C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.c_uint64, C.c_uint, C.c_uint64,
                                    C.POINTER(C.c_double), u64p, C.c_uint32]
        L.ref_eval_accuracy.argtypes = [C.c_char_p, C.c_char_p, C.c_uint, C.c_int]
        L.ref_load_corpus.argtypes = [C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_char_p, u64p, u64p, C.POINTER(u8p), C.POINTER(u64p),
                                      C.POINTER(u64p), C.POINTER(u64p)]
        self.lib = L

    def load_corpus(self, input_path, rejects_path, text_field="text", min_chars=200, L=5,
                    unit=0):
        """-> (records, surviving, data u8, offsets u64, doc_ids u64, char_counts u64)."""
        r, s = C.c_uint64(), C.c_uint64()
        b, o, i, c = u8p(), u64p(), u64p(), u64p()
        self._check(self.lib.ref_load_corpus(input_path.encode(), text_field.encode(), min_chars,
                                             L, unit, rejects_path.encode(), C.byref(r),
                                             C.byref(s), C.byref(b), C.byref(o), C.byref(i),
                                             C.byref(c)))
        n = s.value
        offs = np.ctypeslib.as_array(o, (n + 1,)).copy()
        data = np.ctypeslib.as_array(b, (int(offs[-1]) + 1,))[:int(offs[-1])].copy()
        ids = np.ctypeslib.as_array(i, (n + 1,))[:n].copy()
        ch = np.ctypeslib.as_array(c, (n + 1,))[:n].copy()
        for p in (b, o, i, c):
            self.lib.ref_free(p)
        return r.value, n, data, offs, ids, ch

    def eval_accuracy(self, input_path, workspace, workers=1, override=False):
        self._check(self.lib.ref_eval_accuracy(input_path.encode(), workspace.encode(), workers,
                                               int(override)))

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def derive_family(self, seed: int, H: int, L: int = 5, unit: int = 0):
        fns = (HashFn * H)()
        self._check(self.lib.ref_derive_family(seed, H, L, unit, fns))
        return fns

    def signatures(self, data, offsets, seed=5, H=128, L=5, bands=16, rows=8, K=0, workers=1,
                   doc_ids=None, unit=0):
        n = len(offsets) - 1
        sig = np.zeros((n, H), np.uint32)
        band = np.zeros((n, bands), np.uint32)
        ids = None if doc_ids is None else _ptr(np.ascontiguousarray(doc_ids, np.uint64), u64p)
        self._check(self.lib.ref_signatures(_ptr(data, u8p), _ptr(offsets, u64p), ids, n, seed, H,
                                            L, unit, bands, rows, K, workers, _ptr(sig, u32p),
                                            _ptr(band, u32p)))
        return sig, band

    def compare_cells(self, sigs, cell_offsets, cell_rows, num, den, tile=32, doc_ids=None):
        sigs = np.ascontiguousarray(sigs, np.uint32)
        co = np.ascontiguousarray(cell_offsets, np.uint64)
        cr = np.ascontiguousarray(cell_rows, np.uint32)
        lo, hi, m, n = u64p(), u64p(), u32p(), C.c_uint64()
        ids = None if doc_ids is None else _ptr(np.ascontiguousarray(doc_ids, np.uint64), u64p)
        self._check(self.lib.ref_compare_cells(_ptr(sigs, u32p), ids, sigs.shape[1], _ptr(co, u64p),
                                               _ptr(cr, u32p), len(co) - 1, num, den, tile,
                                               C.byref(lo), C.byref(hi), C.byref(m), C.byref(n)))
        k = n.value
        out = (np.ctypeslib.as_array(lo, (k + 1,))[:k].copy(),
               np.ctypeslib.as_array(hi, (k + 1,))[:k].copy(),
               np.ctypeslib.as_array(m, (k + 1,))[:k].copy())
        for p in (lo, hi, m):
            self.lib.ref_free(p)
        return out

    def compare_cells_timed(self, sigs, cell_offsets, cell_rows, num, den, workers):
        """compare_bucket over every cell, parallel over cells (kernel-only CPU
        baseline): returns dict of seconds + counts and the distinct (lo, hi) rows."""
        sigs = np.ascontiguousarray(sigs, np.uint32)
        co = np.ascontiguousarray(cell_offsets, np.uint64)
        cr = np.ascontiguousarray(cell_rows, np.uint32)
        g, c, u = C.c_double(), C.c_double(), C.c_double()
        em, di = C.c_uint64(), C.c_uint64()
        lo, hi = u64p(), u64p()
        self._check(self.lib.ref_compare_cells_timed(
            _ptr(sigs, u32p), sigs.shape[1], _ptr(co, u64p), _ptr(cr, u32p), len(co) - 1, num, den,
            workers, C.byref(g), C.byref(c), C.byref(u), C.byref(em), C.byref(di), C.byref(lo),
            C.byref(hi)))
        k = di.value
        plo = np.ctypeslib.as_array(lo, (k + 1,))[:k].copy()
        phi = np.ctypeslib.as_array(hi, (k + 1,))[:k].copy()
        self.lib.ref_free(lo)
        self.lib.ref_free(hi)
        return ({"gather_s": g.value, "compare_s": c.value, "unique_s": u.value,
                 "emitted": em.value, "distinct": k}, plo, phi)

    def union_timed(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.uint64)
        hi = np.ascontiguousarray(hi, np.uint64)
        t, g, m = C.c_double(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_union_timed(_ptr(lo, u64p), _ptr(hi, u64p), len(lo), C.byref(t),
                                             C.byref(g), C.byref(m)))
        return {"seconds": t.value, "groups": g.value, "members": m.value}

    def all_pairs_dupset(self, sigs, num, den, workers=8, doc_ids=None):
        sigs = np.ascontiguousarray(sigs, np.uint32)
        n = sigs.shape[0]
        out = np.zeros(n + 1, np.uint64)
        k = C.c_uint64()
        ids = None if doc_ids is None else _ptr(np.ascontiguousarray(doc_ids, np.uint64), u64p)
        self._check(self.lib.ref_all_pairs_dupset(_ptr(sigs, u32p), ids, n, sigs.shape[1], num, den,
                                                  workers, _ptr(out, u64p), C.byref(k)))
        return out[: k.value]

    def union(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.uint64)
        hi = np.ascontiguousarray(hi, np.uint64)
        rep, mem, nrows, ngroups = u64p(), u64p(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_union(_ptr(lo, u64p), _ptr(hi, u64p), len(lo), C.byref(rep),
                                       C.byref(mem), C.byref(nrows), C.byref(ngroups)))
        k = nrows.value
        out = (np.ctypeslib.as_array(rep, (k + 1,))[:k].copy(),
               np.ctypeslib.as_array(mem, (k + 1,))[:k].copy())
        self.lib.ref_free(rep)
        self.lib.ref_free(mem)
        return out

    def generate_synthetic(self, doc_count, group_count, gmin=2, gmax=2, edit=(1, 100),
                           len_min=600, len_max=1200, seed=1, L=5, corpus_path=None,
                           truth_path=None):
        b, o, nb = u8p(), u64p(), C.c_uint64()
        cp = corpus_path.encode() if corpus_path else None
        tp = truth_path.encode() if truth_path else None
        self._check(self.lib.ref_generate_synthetic(doc_count, group_count, gmin, gmax, edit[0],
                                                    edit[1], len_min, len_max, seed, L, cp, tp,
                                                    C.byref(b), C.byref(o), C.byref(nb)))
        data = np.ctypeslib.as_array(b, (nb.value + 1,))[: nb.value].copy()
        offs = np.ctypeslib.as_array(o, (doc_count + 1,)).copy()
        self.lib.ref_free(b)
        self.lib.ref_free(o)
        return data, offs

    def run_dedup(self, input_path, workspace, H=128, bands=16, rows=8, L=5, thr=(4, 5),
                  scale=(2, 1), min_chars=200, seed=5, workers=1, memory_budget=0, unit=0):
        t = (C.c_double * 3)()
        cand = C.c_uint64()
        self._check(self.lib.ref_run_dedup(input_path.encode(), workspace.encode(), H, bands, rows,
                                           L, thr[0], thr[1], scale[0], scale[1], min_chars, seed,
                                           workers, memory_budget, t, C.byref(cand), unit))
        return list(t), cand.value
