"""Pins the CPU oracle (oracle/oracle.c) before it is trusted as the checker.

Sources of truth, in order: the reference's own unit-test vectors
(tests/unit/test_*.cpp), SURVEY App. A known answers produced by running the
reference, and the reference itself (oracle/_ref, compiled from
/root/reference/proj/src in place) on seeded random inputs.
"""
import numpy as np
import pytest

from oracle_bind import HashFn


def _toy(L):
    # test_minhash.cpp:16-24: modulus 97, base 10
    f = HashFn()
    f.modulus, f.base, f.base_inverse = 97, 10, 68
    f.base_power = pow(10, L - 1, 97)
    f.reduce_factor = (1 << 64) // 97
    return f


def _u32(vals):
    a = np.array(vals, np.uint32)
    return a, a.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_uint32))


def test_worked_examples(oracle):
    f = _toy(3)
    a, p = _u32([1, 2, 3])
    assert oracle.lib.or_hash_window_direct(p, 3, f) == 30  # test_minhash.cpp:58-64
    assert oracle.lib.or_roll_next(30, 1, 4, f) == 44  # test_minhash.cpp:66-74
    b, q = _u32([2, 3, 4])
    assert oracle.lib.or_hash_window_direct(q, 3, f) == 44


def test_primality_and_mod_pow(oracle):
    for p in [2, 3, 5, 7, 11, 257, 65521, 2097143, 8388593, 2147483647]:
        assert oracle.lib.or_is_prime_u32(p)
    for c in [0, 1, 4, 9, 100, 561, 2097151, 25326001, 65536]:
        assert not oracle.lib.or_is_prime_u32(c)
    assert oracle.lib.or_mod_pow(10, 0, 97) == 1
    assert oracle.lib.or_mod_pow(10, 2, 97) == 3
    assert oracle.lib.or_mod_pow(2, 10, 1000) == 24
    assert oracle.lib.or_mod_pow(5, 96, 97) == 1


def _fnv_family(fns):
    h = 14695981039346656037
    for f in fns:
        blob = (f.modulus.to_bytes(4, "little") + f.base.to_bytes(4, "little")
                + f.base_inverse.to_bytes(4, "little") + f.base_power.to_bytes(4, "little")
                + f.reduce_factor.to_bytes(8, "little"))
        for c in blob:
            h ^= c
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_family_known_answers(oracle):
    fam = oracle.derive_family(5, 128)
    assert (fam[0].modulus, fam[0].base, fam[0].base_inverse, fam[0].base_power) == (
        2288003, 8707, 735514, 466318)
    assert (fam[1].modulus, fam[1].base) == (3872677, 20627)
    assert (fam[2].modulus, fam[2].base) == (4640171, 3517)
    assert (fam[127].modulus, fam[127].base) == (6343609, 2731)
    assert _fnv_family(fam) == 0x73CA9E5DABE35E33
    fam256 = oracle.derive_family(5, 256)
    assert _fnv_family(fam256) == 0x47A9B9351659D55D
    assert (fam256[255].modulus, fam256[255].base) == (3815281, 23357)
    assert bytes(fam256)[: 24 * 128] == bytes(fam)  # prefix-stable in H


def test_fox_signature_known_answers(oracle):
    t = b"the quick brown fox jumps over the lazy dog"
    data = np.frombuffer(t, np.uint8).copy()
    offs = np.array([0, len(t)], np.uint64)
    sig = oracle.signatures(data, offs, oracle.derive_family(5, 128))
    assert sig[0, :8].tolist() == [66895, 242299, 135669, 105208, 5044, 26899, 34271, 98201]
    h = 14695981039346656037
    for c in sig[0].astype("<u4").tobytes():
        h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    assert h == 0xAD23996632428A07
    assert oracle.band_ids(sig, 16, 8, 10955)[0].tolist() == [
        2411, 7077, 4901, 2848, 7971, 2997, 9, 6230, 1121, 6549, 1771, 7319, 10449, 7294, 10693,
        9499]


def test_bucket_counts(oracle):
    c = oracle.lib.or_choose_bucket_count
    assert c(1_000_000, 2, 1) == 2000
    assert c(30_000_000, 2, 1) == 10955
    assert c(25, 2, 1) == 10
    assert c(4, 3, 2) == 3
    assert c(2, 1, 1) == 2
    assert c(1, 2, 1) == 2
    assert c(100, 1, 100) == 1
    assert c(0, 2, 1) == 1
    assert c(1 << 40, 1, 1) == 1 << 20
    assert c(10_000, 2, 1) == 200 and c(2_000_000, 2, 1) == 2829


def test_band_ids_worked_example(oracle):
    sig = np.array([[5, 7, 100, 3, 9, 9, 0, 1]], np.uint32)
    assert oracle.band_ids(sig, 4, 2, 10)[0].tolist() == [2, 3, 8, 1]  # test_lsh.cpp:31-37
    assert oracle.band_ids(sig, 1, 8, 7)[0].tolist() == [(5 + 7 + 100 + 3 + 9 + 9 + 0 + 1) % 7]


def test_threshold(oracle):
    mm, acc = oracle.lib.or_min_matches, oracle.lib.or_accepts
    assert mm(128, 4, 5) == 103 and mm(256, 4, 5) == 205
    assert acc(103, 128, 4, 5) and not acc(102, 128, 4, 5)
    assert not acc(4, 5, 4, 5) and acc(5, 5, 4, 5) and mm(5, 4, 5) == 5
    assert not acc(128, 128, 1, 1) and mm(128, 1, 1) == 129
    assert acc(1, 128, 0, 1) and not acc(0, 128, 0, 1) and mm(128, 0, 1) == 1


def test_components_worked_examples(oracle):
    # test_dedup_graph.cpp:36-47 and :63-70 (dense ids)
    lab = oracle.components(np.array([1, 2, 8]), np.array([2, 3, 9]), 10)
    assert lab[1] == lab[2] == lab[3] == 1 and lab[8] == lab[9] == 8
    assert lab[0] == 0xFFFFFFFF and lab[5] == 0xFFFFFFFF
    lab = oracle.components(np.arange(1000), np.arange(1, 1001), 1001)
    assert (lab == 0).all()


def test_compare_cell_vs_naive(oracle):
    rng = np.random.default_rng(1000)
    for n in (2, 3, 31, 32, 33, 64):
        sigs = rng.integers(0, 3, size=(n, 8)).astype(np.uint32)
        lo, hi, m = oracle.compare_cell(sigs, np.arange(n), 1, 4)
        want = [(i, j, int((sigs[i] == sigs[j]).sum())) for i in range(n) for j in range(i + 1, n)
                if (sigs[i] == sigs[j]).sum() * 4 > 8]
        assert list(zip(lo.tolist(), hi.tolist(), m.tolist())) == want


# ---- against the reference itself ------------------------------------------

def test_family_matches_reference(oracle, ref):
    for seed, H, L in [(5, 128, 5), (5, 256, 5), (42, 16, 5), (7, 32, 3), (11, 8, 9)]:
        assert bytes(oracle.derive_family(seed, H, L)) == bytes(ref.derive_family(seed, H, L))


def test_signatures_and_bands_match_reference(oracle, ref):
    data, offs = ref.generate_synthetic(300, 30, len_min=600, len_max=1200, seed=3)
    want_sig, want_band = ref.signatures(data, offs, K=200, workers=4)
    sig = oracle.signatures(data, offs, oracle.derive_family(5, 128))
    np.testing.assert_array_equal(sig, want_sig)
    np.testing.assert_array_equal(oracle.band_ids(sig, 16, 8, 200), want_band)


def test_compare_and_union_match_reference(oracle, ref):
    rng = np.random.default_rng(5)
    sigs = rng.integers(0, 3, size=(120, 16)).astype(np.uint32)
    cells = [np.sort(rng.choice(120, size=k, replace=False)) for k in (2, 5, 40, 77)]
    offs = np.zeros(len(cells) + 1, np.uint64)
    offs[1:] = np.cumsum([len(c) for c in cells])
    rows = np.concatenate(cells).astype(np.uint32)
    rlo, rhi, rm = ref.compare_cells(sigs, offs, rows, 1, 2)
    mine = set()
    for c in cells:
        lo, hi, m = oracle.compare_cell(sigs, c, 1, 2)
        mine |= set(zip(lo.tolist(), hi.tolist(), m.tolist()))
    assert sorted(mine) == list(zip(rlo.tolist(), rhi.tolist(), rm.tolist()))
    rep, mem = ref.union(rlo, rhi)
    lab = oracle.components(rlo.astype(np.uint32), rhi.astype(np.uint32), 120)
    got = sorted((int(lab[i]), i) for i in range(120) if lab[i] != 0xFFFFFFFF)
    assert got == list(zip(rep.tolist(), mem.tolist()))


# ---- codepoint units (text.cpp:88-113) --------------------------------------
def _rand_utf8(rng, n_units, ill_formed=False):
    """Random text over 1..4-byte scalars (plus, optionally, ill-formed bytes)."""
    pools = [(0x20, 0x7F), (0xA0, 0x800), (0x800, 0xD800), (0xE000, 0x10000), (0x10000, 0x110000)]
    out = bytearray()
    for _ in range(n_units):
        k = rng.integers(0, len(pools) + (2 if ill_formed else 0))
        if k >= len(pools):
            out += bytes(rng.integers(0x80, 0x100, size=int(rng.integers(1, 4)), dtype=np.uint8))
            continue
        lo, hi = pools[k]
        out += chr(int(rng.integers(lo, hi))).encode("utf-8")
    return bytes(out)


def test_decode_codepoints_maximal_subparts(oracle):
    # Unicode 15 ch.3, Table 3-8 (U+FFFD for maximal subparts), which ICU's
    # U8_NEXT (text.cpp:101-113) follows
    b = bytes([0x61, 0xF1, 0x80, 0x80, 0xE1, 0x80, 0xC2, 0x62, 0x80, 0x63, 0x80, 0xBF, 0x64])
    assert oracle.decode_codepoints(b) == [0x61, 0xFFFD, 0xFFFD, 0xFFFD, 0x62, 0xFFFD, 0x63,
                                           0xFFFD, 0xFFFD, 0x64]
    assert oracle.decode_codepoints("é€😀".encode()) == [0xE9, 0x20AC, 0x1F600]
    assert oracle.decode_codepoints(b"\xed\xa0\x80") == [0xFFFD] * 3  # surrogate: ED A0 ill-formed
    assert oracle.decode_codepoints(b"\xf0\x9f\x98") == [0xFFFD]  # truncated 4-byte sequence
    assert oracle.decode_codepoints(b"\xc0\xaf") == [0xFFFD, 0xFFFD]  # overlong lead


def test_decode_codepoints_matches_cpython(oracle):
    # CPython's UTF-8 decoder implements the same maximal-subpart replacement
    rng = np.random.default_rng(3)
    for _ in range(300):
        b = _rand_utf8(rng, int(rng.integers(0, 60)), ill_formed=True)
        want = [ord(c) for c in b.decode("utf-8", errors="replace")]
        assert oracle.decode_codepoints(b) == want, b


def test_codepoint_signatures_oracle_vs_reference(oracle, ref):
    rng = np.random.default_rng(9)
    texts = [_rand_utf8(rng, int(n), ill_formed=bool(i % 3 == 0))
             for i, n in enumerate(rng.integers(5, 400, size=60))]
    offs = np.zeros(len(texts) + 1, np.uint64)
    offs[1:] = np.cumsum([len(t) for t in texts])
    data = np.frombuffer(b"".join(texts), np.uint8).copy()
    for H, L in [(128, 5), (16, 3)]:
        want, _ = ref.signatures(data, offs, seed=5, H=H, L=L, bands=0, rows=0, K=0, unit=1)
        got = oracle.signatures(data, offs, oracle.derive_family(5, H, L), L, unit=1)
        np.testing.assert_array_equal(got, want)


def test_verify_drivers_match_single_thread_oracle(oracle):
    # oracle/verify.c (full-scale parity driver) == or_compare_cell per cell
    import ctypes as C

    from oracle_bind import u32p, u64p

    L = oracle.lib
    L.ov_cells.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint32, u64p, u32p]
    L.ov_compare_cells.argtypes = [u32p, C.c_uint32, u64p, u32p, C.c_uint64, C.c_uint64,
                                   C.c_uint64, C.c_int, C.POINTER(u32p), C.POINTER(u32p),
                                   C.POINTER(u32p), u64p]
    L.ov_compare_cells.restype = C.c_int64
    L.ov_free.argtypes = [C.c_void_p]
    rng = np.random.default_rng(4)
    n, H, B, K = 600, 64, 8, 12
    sig = rng.integers(0, 6, size=(n, H), dtype=np.uint32)  # many near-duplicates
    band = rng.integers(0, K, size=(n, B), dtype=np.uint32)
    off = np.empty(B * K + 1, np.uint64)
    rows = np.empty(n * B, np.uint32)
    assert L.ov_cells(band.ctypes.data_as(u32p), n, B, K, off.ctypes.data_as(u64p),
                      rows.ctypes.data_as(u32p)) == 0
    want, cand = set(), 0
    for c in range(B * K):
        r = rows[int(off[c]):int(off[c + 1])]
        assert (np.diff(r.astype(np.int64)) > 0).all()
        assert (band[r, c // K] == c % K).all()
        cand += len(r) * (len(r) - 1) // 2
        lo, hi, m = oracle.compare_cell(sig, r, 1, 4)
        want |= set(zip(lo.tolist(), hi.tolist(), m.tolist()))
    lo_p, hi_p, m_p, cc = u32p(), u32p(), u32p(), C.c_uint64()
    k = L.ov_compare_cells(sig.ctypes.data_as(u32p), H, off.ctypes.data_as(u64p),
                           rows.ctypes.data_as(u32p), B * K, 1, 4, 3, C.byref(lo_p), C.byref(hi_p),
                           C.byref(m_p), C.byref(cc))
    got = set(zip(np.ctypeslib.as_array(lo_p, (k,)).tolist(), np.ctypeslib.as_array(hi_p, (k,)).tolist(),
                  np.ctypeslib.as_array(m_p, (k,)).tolist()))
    for p in (lo_p, hi_p, m_p):
        L.ov_free(p)
    assert cc.value == cand and got == want and len(want) > 100
