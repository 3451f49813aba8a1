"""Host-side logic of the product library (no GPU): family derivation,
bucket count, threshold, partitions, synthetic corpora, and the C-ABI
surface (every symbol include/neardup_b200.h declares is exported)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2501_01046_b200 import _lib, minhash
from paper_2501_01046_b200._lib import check

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "neardup_b200.h")).read()
    declared = set(re.findall(r"\b(nd_[a-z_0-9]+)\s*\(", hdr))
    lib = _lib.load()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_derive_family_matches_reference(ref):
    for seed, H, L in [(5, 128, 5), (5, 256, 5), (42, 16, 5), (7, 32, 3), (1, 4, 5)]:
        assert bytes(minhash.derive_family(seed, H, L).functions) == bytes(ref.derive_family(seed, H, L))


def test_derive_family_is_pure_and_validates():
    a = minhash.derive_family(42, 16, 5)
    b = minhash.derive_family(42, 16, 5)
    c = minhash.derive_family(43, 16, 5)
    assert bytes(a.functions) == bytes(b.functions) != bytes(c.functions)
    with pytest.raises(_lib.ConfigError):
        minhash.derive_family(1, 0, 5)
    with pytest.raises(_lib.ConfigError):
        minhash.derive_family(1, 4, 0)
    for f in minhash.derive_family(7, 32, 5).functions:
        assert (1 << 21) <= f.modulus < (1 << 23) and 256 < f.base < (1 << 16)
        assert f.base * f.base_inverse % f.modulus == 1
        assert f.base_power == pow(f.base, 4, f.modulus)
        assert f.reduce_factor == (1 << 64) // f.modulus


def test_choose_bucket_count():
    lib = _lib.load()
    out = C.c_uint32()

    def k(n, num, den):
        check(lib.nd_choose_bucket_count(n, num, den, C.byref(out)))
        return out.value

    assert [k(1_000_000, 2, 1), k(30_000_000, 2, 1), k(25, 2, 1), k(4, 3, 2), k(2, 1, 1),
            k(1, 2, 1), k(100, 1, 100), k(0, 2, 1), k(1 << 40, 1, 1)] == [
        2000, 10955, 10, 3, 2, 2, 1, 1, 1 << 20]
    with pytest.raises(_lib.ConfigError):
        k(1 << 62, 1 << 32, 1)
    with pytest.raises(_lib.ConfigError):
        k(10, 0, 1)


def test_min_matches():
    lib = _lib.load()
    assert lib.nd_min_matches(128, 4, 5) == 103
    assert lib.nd_min_matches(256, 4, 5) == 205
    assert lib.nd_min_matches(5, 4, 5) == 5
    assert lib.nd_min_matches(128, 1, 1) == 129
    assert lib.nd_min_matches(128, 0, 1) == 1


def test_partitions():
    lib = _lib.load()
    r = (C.c_uint32 * 8)()
    check(lib.nd_band_partition(2, 4, r))
    assert list(r) == [0, 1, 1, 2, 2, 2, 2, 2]
    check(lib.nd_band_partition(16, 4, r))
    assert list(r) == [0, 4, 4, 8, 8, 12, 12, 16]
    fc = (C.c_uint64 * 9)()
    check(lib.nd_cell_partition(16, 10955, 8, fc))
    cells = 16 * 10955
    assert fc[0] == 0 and fc[8] == cells
    sizes = [fc[i + 1] - fc[i] for i in range(8)]
    assert max(sizes) - min(sizes) <= 1


def _synth(spec):
    lib = _lib.load()
    nb = C.c_uint64()
    check(lib.nd_synth_generate(C.byref(spec), None, None, C.byref(nb)))
    data = np.empty(nb.value, np.uint8)
    offs = np.empty(spec.doc_count + 1, np.uint64)
    check(lib.nd_synth_generate(C.byref(spec), data.ctypes.data_as(_lib.u8p),
                                offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
    return data, offs


def test_synthetic_mode0_is_the_reference_generator(ref):
    spec = _lib.NdSynthSpec(doc_count=2000, group_count=100, group_size_min=2, group_size_max=3,
                            edit_num=1, edit_den=100, len_min=600, len_max=1200, seed=9, mode=0)
    data, offs = _synth(spec)
    rdata, roffs = ref.generate_synthetic(2000, 100, gmin=2, gmax=3, len_min=600, len_max=1200,
                                          seed=9)
    np.testing.assert_array_equal(offs, roffs)
    np.testing.assert_array_equal(data, rdata)


def test_synthetic_mode1_is_deterministic_and_shaped():
    spec = _lib.NdSynthSpec(doc_count=5000, group_count=250, group_size_min=2, group_size_max=5,
                            edit_num=1, edit_den=100, len_min=1600, len_max=2400, seed=4, mode=1,
                            threads=4)
    d1, o1 = _synth(spec)
    spec.threads = 1
    d2, o2 = _synth(spec)
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(d1, d2)
    lens = np.diff(o1)
    assert lens.min() >= 1600 and lens.max() <= 2400
    alphabet = set(b"abcdefghijklmnopqrstuvwxyz0123456789 ")
    assert set(np.unique(d1).tolist()) <= alphabet
    # lognormal law clipped at [200, len_max]
    spec = _lib.NdSynthSpec(doc_count=4000, group_count=0, group_size_min=2, group_size_max=2,
                            edit_num=1, edit_den=100, len_min=2000, len_max=200_000, seed=4,
                            mode=1, len_law=1, sigma_milli=1100)
    _, o = _synth(spec)
    lens = np.diff(o)
    assert lens.min() >= 200 and lens.max() <= 200_000
    assert 1500 < np.median(lens) < 2600


def test_scalar_minhash_primitives():
    # test_minhash.cpp:16-74: modulus 97, base 10; mod_pow / Miller-Rabin
    from paper_2501_01046_b200 import _lib, minhash

    f = _lib.NdHashFn(modulus=97, base=10, base_inverse=68, base_power=pow(10, 2, 97),
                      reduce_factor=(1 << 64) // 97)
    assert minhash.hash_window_direct([1, 2, 3], f) == 30
    assert minhash.roll_next(30, 1, 4, f) == 44
    assert minhash.hash_window_direct([2, 3, 4], f) == 44
    with pytest.raises(_lib.ConfigError):
        minhash.hash_window_direct([], f)
    assert minhash.mod_pow(3, 100, 97) == pow(3, 100, 97)
    assert minhash.mod_pow(5, 0, 1) == 0
    with pytest.raises(_lib.ConfigError):
        minhash.mod_pow(3, 4, 0)
    assert [p for p in range(60) if minhash.is_prime_u32(p)] == [
        2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59]
    assert minhash.is_prime_u32(2147483647) and not minhash.is_prime_u32(25326001)


def test_raw_document_iteration(tmp_path):
    # for_each_raw_document / load_jsonl_file (corpus.cpp:56-91)
    from paper_2501_01046_b200 import corpus

    p = tmp_path / "x.jsonl"
    p.write_bytes(b'{"text": "a"}\n\nnot json\r\n{"text": "b"}\r\n[1]\n{"text": "c"}')
    rejects = []
    docs = corpus.load_jsonl_file(str(p), 7, "text", rejects)
    assert [(d.file_ordinal, d.record_ordinal, d.line, d.text) for d in docs] == [
        (7, 0, 1, b"a"), (7, 1, 4, b"b"), (7, 2, 6, b"c")]
    assert rejects == [(str(p), 3, "invalid_json"), (str(p), 5, "not_an_object")]
