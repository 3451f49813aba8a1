"""Signature store and pair files (host C++ of libneardup_b200, no GPU): the
cases of the reference's tests/unit/test_sigstore.cpp, plus byte identity
with files the reference itself wrote (oracle/_ref run_dedup)."""
import os
import struct

import numpy as np
import pytest

from paper_2501_01046_b200 import _lib, sigstore
from paper_2501_01046_b200.minhash import ShingleUnit
from paper_2501_01046_b200.sigstore import SignatureFileHeader


def _toy(**kw):
    # test_sigstore.cpp:14-26
    h = SignatureFileHeader(hash_count=4, bands=2, rows=2, bucket_count=5, shingle_len=3,
                            unit=ShingleUnit.BYTE, family_seed=7, bucket_scale=(2, 1))
    for k, v in kw.items():
        setattr(h, k, v)
    return h


def _write(path, h, recs):
    ids = [r[0] for r in recs]
    sigstore.write_signature_file(str(path), h, ids, [r[1] for r in recs], [r[2] for r in recs])


RECS = [(0, [1, 2, 3, 4], [1, 3]), (1, [5, 6, 7, 8], [1, 4]), (7, [9, 10, 11, 12], [2, 3])]


def test_header_layout_and_round_trip(tmp_path):
    p = tmp_path / "sigs.feds"
    _write(p, _toy(source_ordinal=9), RECS)
    raw = p.read_bytes()
    # sigstore.cpp:20-36 field order, little-endian
    want = b"FEDS" + struct.pack("<7I", 1, 4, 2, 2, 5, 3, 0) + struct.pack("<5Q", 7, 2, 1, 3, 9)
    assert raw[:72] == want
    assert raw[72:72 + 8 + 16 + 8] == struct.pack("<Q4I2I", 0, 1, 2, 3, 4, 1, 3)
    assert len(raw) == 72 + 3 * (8 + 16 + 8)
    h, ids, v, b = sigstore.read_signature_file(str(p))
    assert (h.record_count, h.source_ordinal, h.family_seed, h.bucket_scale) == (3, 9, 7, (2, 1))
    assert ids.tolist() == [0, 1, 7]
    assert v.tolist() == [r[1] for r in RECS] and b.tolist() == [r[2] for r in RECS]


def test_reader_rejects_corruption(tmp_path):
    # test_sigstore.cpp:124-145
    p = tmp_path / "sigs.feds"
    _write(p, _toy(), RECS[:1])
    good = p.read_bytes()
    cases = {"short.feds": good[:-5], "long.feds": good + b"xyz", "magic.feds": b"X" + good[1:],
             "version.feds": good[:4] + bytes([99]) + good[5:], "trunc.feds": good[:40]}
    bad = bytearray(good)
    bad[72 + 8 + 16] = 9  # bucket id 9 >= bucket_count 5
    cases["bucket.feds"] = bytes(bad)
    for name, data in cases.items():
        (tmp_path / name).write_bytes(data)
        with pytest.raises(_lib.IoError):
            sigstore.read_signature_file(str(tmp_path / name))
    with pytest.raises(_lib.IoError):
        sigstore.read_signature_file(str(tmp_path / "absent.feds"))


def test_run_compatibility_ignores_per_file_fields():
    a = _toy()
    assert a.run_compatible(_toy(record_count=55, source_ordinal=3))
    assert a.run_compatible(_toy(bucket_scale=(4, 2)))  # Ratio normalises
    assert not a.run_compatible(_toy(family_seed=8))
    assert not a.run_compatible(_toy(bucket_count=6))


def test_plan_gather_worked_examples():
    # test_sigstore.cpp:215-258
    p = sigstore.plan_gather(10_000_000_000, 10_000, 16, 4, 16_000_000_000)
    assert p.buckets_per_pass == 4000 and p.passes_per_worker == [3, 3, 3, 3]
    assert sigstore.plan_gather(1000, 50, 16, 1, 1_000_000_000).passes_per_worker == [1]
    f = sigstore.plan_gather(1000, 50, 16, 1, 1_000_000_000, 7)
    assert (f.buckets_per_pass, f.passes_per_worker) == (7, [8])
    assert sigstore.plan_gather(1000, 50, 16, 1, 1_000_000_000, 500).buckets_per_pass == 50
    assert sigstore.plan_gather(0, 50, 16, 1, 1).buckets_per_pass == 50
    for args in [(1_000_000, 10, 16, 1, 5), (1000, 0, 16, 1, 100), (1000, 50, 16, 0, 100),
                 (1000, 50, 16, 1, 0)]:
        with pytest.raises(_lib.ConfigError):
            sigstore.plan_gather(*args)
    with pytest.raises(_lib.ConfigError):
        sigstore.plan_gather(1000, 50, 16, 1, 100, 0)
    # more workers than bands: the band-less worker gets no passes
    assert sigstore.plan_gather(1000, 50, 1, 2, 1_000_000_000).passes_per_worker == [1, 0]


def test_pair_file_format(tmp_path):
    p = str(tmp_path / "x.pairs")
    sigstore.write_pair_file(p, [1, 2], [5, 2**40], [100, 128])
    raw = open(p, "rb").read()
    assert raw == struct.pack("<QQI", 1, 5, 100) + struct.pack("<QQI", 2, 2**40, 128)
    lo, hi, m = sigstore.read_pair_file(p)
    assert lo.tolist() == [1, 2] and hi.tolist() == [5, 2**40] and m.tolist() == [100, 128]
    open(p, "ab").write(b"\0")
    with pytest.raises(_lib.IoError):
        sigstore.read_pair_file(p)
    sigstore.write_pair_file(p, [], [], [])
    assert os.path.getsize(p) == 0 and len(sigstore.read_pair_file(p)[0]) == 0


def test_reference_artifacts_rewrite_byte_identical(ref, oracle, tmp_path):
    # .feds and .pairs files written by the reference's own hash / compare
    # stages parse here and re-serialise to the same bytes
    corpus = str(tmp_path / "c.jsonl")
    ref.generate_synthetic(400, 40, gmin=2, gmax=3, len_min=300, len_max=700, seed=2,
                           corpus_path=corpus, truth_path=str(tmp_path / "t.jsonl"))
    ws = str(tmp_path / "ws")
    os.makedirs(ws)
    ref.run_dedup(corpus, ws, workers=2, memory_budget=150_000)
    feds = sorted(os.listdir(os.path.join(ws, "signatures")))
    assert feds == ["00000_c.feds"]
    src = os.path.join(ws, "signatures", feds[0])
    h, ids, v, b = sigstore.read_signature_file(src)
    assert h.record_count == 400 and h.bucket_count == 40
    out = str(tmp_path / "again.feds")
    sigstore.write_signature_file(out, h, ids, v, b)
    assert open(out, "rb").read() == open(src, "rb").read()
    # the stored signatures are the oracle's
    data, offs = ref.generate_synthetic(400, 40, gmin=2, gmax=3, len_min=300, len_max=700, seed=2)
    np.testing.assert_array_equal(v, oracle.signatures(data, offs, oracle.derive_family(5, 128)))
    pairs = sorted(os.listdir(os.path.join(ws, "pairs")))
    assert len(pairs) > 2  # several gather passes per worker
    for name in pairs:
        src = os.path.join(ws, "pairs", name)
        lo, hi, m = sigstore.read_pair_file(src)
        sigstore.write_pair_file(out, lo, hi, m)
        assert open(out, "rb").read() == open(src, "rb").read()


def test_scan_gather_cases(tmp_path):
    # test_sigstore.cpp:147-212
    from paper_2501_01046_b200.lsh import BandRange, BucketKey

    h = _toy()
    _write(tmp_path / "a.feds", h, RECS[:2] + [(2, [9, 10, 11, 12], [2, 3])])
    _write(tmp_path / "b.feds", _toy(source_ordinal=1), [(3, [13, 14, 15, 16], [1, 3])])
    paths = [str(tmp_path / "a.feds"), str(tmp_path / "b.feds")]
    g = sigstore.scan_gather(paths, h, BandRange(0, 1), 1, 2)
    assert len(g.buckets) == 1 and g.buckets[0].key == BucketKey(0, 1)
    assert list(g.buckets[0].doc_ids) == [0, 1, 3]
    assert list(g.buckets[0].signatures) == [1, 2, 3, 4, 5, 6, 7, 8, 13, 14, 15, 16]
    g = sigstore.scan_gather(paths, h, BandRange(0, 2), 0, 5)
    assert [b.key for b in g.buckets] == [BucketKey(0, 1), BucketKey(1, 3)]
    assert list(g.buckets[1].doc_ids) == [0, 2, 3]
    assert sigstore.scan_gather(paths, h, BandRange(0, 2), 4, 4).buckets == []
    _write(tmp_path / "d.feds", h, [(5, [1, 2, 3, 4], [1, 3]), (3, [5, 6, 7, 8], [1, 3])])
    with pytest.raises(_lib.ConfigError):
        sigstore.scan_gather([str(tmp_path / "d.feds")], h, BandRange(0, 2), 0, 5)
    _write(tmp_path / "o.feds", _toy(family_seed=99), [(0, [1, 2, 3, 4], [1, 3])])
    with pytest.raises(_lib.ConfigError):
        sigstore.scan_gather([str(tmp_path / "o.feds")], h, BandRange(0, 2), 0, 5)
    with pytest.raises(_lib.ConfigError):
        sigstore.scan_gather([], h, BandRange(0, 2), 0, 6)
    with pytest.raises(_lib.ConfigError):
        sigstore.scan_gather([], h, BandRange(0, 3), 0, 5)
