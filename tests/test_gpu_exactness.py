"""Exactness on legal inputs outside the default configuration.

Each case is a shape the reference handles and an earlier GPU path got wrong:
  * H - min_matches + 1 > 510 (H=512 at theta 0 and 1/512; H=1024 at 1/2):
    the joins' 9-bit block tags do not fit, so every cell must go to the
    all-pairs kernel (compare_bucket compares every cell, compare.cpp:24-67);
  * the per-position join (BW = 1, theta < ~1/2) with u32 values spanning
    2^32 (compare_bucket takes arbitrary values, compare.cpp:24-67);
  * hand-built HashFunctionParams outside derive_family's domain
    (minhash.hpp:17-25 is a public struct): exact signatures or ConfigError.
"""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2501_01046_b200 import _lib, compare, lsh, minhash, pipeline
from paper_2501_01046_b200.compare import DuplicatePair, GatheredBucket, GatherResult, SimilarityThreshold

pytestmark = pytest.mark.gpu


def _files(ws):
    return {f: open(os.path.join(ws, f), "rb").read()
            for f in ("groups.jsonl", "removal.txt", "summary.json")}


@pytest.mark.parametrize("thr", [(0, 1), (1, 512)])
def test_run_dedup_h512_low_threshold_byte_identical(ctx, ref, tmp_path, thr):
    # P = 512 - min_matches + 1 = 512 / 511 > 510: no join can take these cells
    corpus = str(tmp_path / "c.jsonl")
    ref.generate_synthetic(1500, 120, gmin=2, gmax=3, edit=(5, 100), len_min=250, len_max=600,
                           seed=29, corpus_path=corpus, truth_path=str(tmp_path / "t.jsonl"))
    ws_ref, ws_gpu = str(tmp_path / "r"), str(tmp_path / "g")
    os.makedirs(ws_ref)
    _, cand = ref.run_dedup(corpus, ws_ref, H=512, bands=64, rows=8, thr=thr,
                            workers=os.cpu_count())
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu, hash_count=512, bands=64, rows=8,
                             threshold=thr)
    rep = pipeline.run_dedup(cfg, ctx=ctx)
    want = _files(ws_ref)
    assert _files(ws_gpu) == want
    assert rep.candidate_pairs == cand
    assert b"members" in want["groups.jsonl"]


def _planted(n, H, rng, lo_bits, hi_bits, flips):
    base = rng.integers(0, 1 << 32, size=H, dtype=np.uint64).astype(np.uint32)
    sig = np.tile(base, (n, 1))
    for r in range(n):
        k = int(rng.integers(0, flips))
        pos = rng.choice(H, size=k, replace=False)
        sig[r, pos] = rng.integers(1 << lo_bits, 1 << hi_bits, size=k, dtype=np.uint64).astype(np.uint32)
    return sig


@pytest.mark.parametrize("H,thr,join_blocks", [(128, (1, 4), None), (128, (4, 5), "0"),
                                                (64, (1, 3), None), (1024, (1, 2), None)])
def test_compare_pass_full_u32_values_vs_reference(ctx, ref, monkeypatch, H, thr, join_blocks):
    # values >= 2^23 everywhere; cells of planted near-copies plus random rows
    if join_blocks is not None:
        monkeypatch.setenv("ND_JOIN_BLOCKS", join_blocks)
    rng = np.random.default_rng(H * 7 + thr[1])
    buckets = []
    for c, n in enumerate([2, 7, 60, 130, 300]):
        sig = _planted(n, H, rng, 23, 32, int(H * 0.9))
        rnd = rng.integers(0, 1 << 32, size=(n // 3 + 1, H), dtype=np.uint64).astype(np.uint32)
        sig = np.concatenate([sig, rnd])
        sig = sig[rng.permutation(len(sig))]
        ids = list(range(c * 10000, c * 10000 + len(sig)))
        buckets.append(GatheredBucket(lsh.BucketKey(c, 0), ids, sig.reshape(-1)))
    t = SimilarityThreshold(thr)
    got = compare.compare_pass(GatherResult(buckets), H, t, ctx=ctx)
    allsig = np.concatenate([b.signatures.reshape(-1, H) for b in buckets])
    ids = np.concatenate([b.doc_ids for b in buckets]).astype(np.uint64)
    offs = np.cumsum([0] + [len(b.doc_ids) for b in buckets]).astype(np.uint64)
    lo, hi, m = ref.compare_cells(allsig, offs, np.arange(len(ids), dtype=np.uint32), *thr,
                                  doc_ids=ids)
    want = [DuplicatePair(int(a), int(b), int(c)) for a, b, c in zip(lo, hi, m)]
    assert got == want
    assert got


def test_per_position_join_value_collisions(ctx, ref, monkeypatch):
    # values that agree in their low 23 bits but differ above them: the old
    # tag << 23 | v key let a value >= 2^23 overwrite a live slot
    monkeypatch.setenv("ND_JOIN_BLOCKS", "0")
    H, n = 64, 200
    rng = np.random.default_rng(3)
    low = rng.integers(0, 1 << 23, size=H, dtype=np.uint64)
    sig = np.empty((n, H), np.uint32)
    for r in range(n):
        hi = rng.integers(0, 4, size=H, dtype=np.uint64) << np.uint64(23)  # 4 variants per position
        sig[r] = (low | hi).astype(np.uint32)
    b = GatheredBucket(lsh.BucketKey(0, 0), list(range(n)), sig.reshape(-1))
    for thr in [(1, 4), (1, 8), (1, 5)]:
        got = compare.compare_bucket(b, H, SimilarityThreshold(thr), ctx=ctx)
        lo, hi_, m = ref.compare_cells(sig, np.array([0, n], np.uint64),
                                       np.arange(n, dtype=np.uint32), *thr)
        assert got == [DuplicatePair(int(a), int(c), int(d)) for a, c, d in zip(lo, hi_, m)]
        assert got


def _colliding_values(tbits, count, lo, hi, rng):
    """`count` distinct values in [lo, hi) whose join-table home slot
    ((v * 0x9E3779B1) >> (32 - tbits), k_compare.cu) is the same."""
    out = set()
    target = None
    while len(out) < count:
        v = rng.integers(lo, hi, size=1 << 16, dtype=np.uint64)
        home = ((v * np.uint64(0x9E3779B1)) & np.uint64(0xFFFFFFFF)) >> np.uint64(32 - tbits)
        if target is None:
            target = int(home[0])
        out.update(int(x) for x in v[home == target])
    return sorted(out)[:count]


def test_per_position_join_mixed_small_and_large_values_one_home_slot(ctx, ref, monkeypatch):
    # Every value at positions < P shares one home slot; half are < 2^23, half
    # >= 2^23.  With the old (tag << 23 | v) key a large value's entry looks
    # stale, a small value takes its slot over, and the next document with
    # the large value starts a second chain: pairs whose FIRST match is that
    # large value were never checked.
    monkeypatch.setenv("ND_JOIN_BLOCKS", "0")
    H, n, thr = 64, 1000, (1, 4)         # min_matches 17, P = 48
    tbits = 11                            # join table of n = 1000 at load 1/2
    rng = np.random.default_rng(12)
    S = np.array(_colliding_values(tbits, 4, 1, 1 << 23, rng)
                 + _colliding_values(tbits, 4, 1 << 23, 1 << 32, rng), np.uint32)
    sig = S[rng.integers(0, len(S), size=(n, H))]
    sig[:, 48:] = rng.integers(0, 1 << 32, size=H - 48, dtype=np.uint64).astype(np.uint32)
    b = GatheredBucket(lsh.BucketKey(0, 0), list(range(n)), sig.reshape(-1))
    got = compare.compare_bucket(b, H, SimilarityThreshold(thr), ctx=ctx)
    lo, hi_, m = ref.compare_cells(sig, np.array([0, n], np.uint64),
                                   np.arange(n, dtype=np.uint32), *thr)
    assert len(got) == len(lo)
    assert got == [DuplicatePair(int(a), int(c), int(d)) for a, c, d in zip(lo, hi_, m)]


# ---------------------------------------------------------------------------
# hand-built hash families


def _fn(p, q, L):
    inv = pow(q, -1, p)
    return _lib.NdHashFn(modulus=p, base=q, base_inverse=inv, base_power=pow(q, L - 1, p),
                         reduce_factor=(1 << 64) // p)


def _family(fns, L=5, unit=minhash.ShingleUnit.BYTE):
    arr = (_lib.NdHashFn * len(fns))(*fns)
    return minhash.HashFamily(len(fns), L, unit, 0, arr)


def _corpus(rng, n=40, lo=5, hi=3000):
    texts = [bytes(rng.integers(0, 256, size=int(k), dtype=np.uint8)) for k in rng.integers(lo, hi, n)]
    texts.append(bytes(rng.integers(0, 256, size=20000, dtype=np.uint8)))  # multi-item document
    offs = np.zeros(len(texts) + 1, np.uint64)
    offs[1:] = np.cumsum([len(t) for t in texts])
    return np.frombuffer(b"".join(texts), np.uint8).copy(), offs


def _oracle_fns(fns):
    from oracle_bind import HashFn

    return (HashFn * len(fns))(*[HashFn(f.modulus, f.base, f.base_inverse, f.base_power,
                                        f.reduce_factor) for f in fns])


@pytest.mark.parametrize("L", [3, 5])
def test_hand_built_families_exact(ctx, oracle, L):
    # p = 257 with q = 65521 (> p), small primes above 255, primes in
    # [2^23, 2^31), and a derive_family function, mixed in one family
    fns = [_fn(257, 65521, L), _fn(263, 3, L), _fn(65537, 40961, L), _fn(1000003, 65519, L),
           _fn(2097143, 65521, L), _fn(8388617, 257, L), _fn(2147483629, 65521, L),
           _fn(2147483647, 1000003, L)]
    fam0 = minhash.derive_family(5, 24, L)
    fns += [fam0.functions[i] for i in range(24)]
    rng = np.random.default_rng(L)
    data, offs = _corpus(rng)
    sig, _ = minhash.signatures_packed(data, offs, _family(fns, L), ctx=ctx, want_bands=False)
    want = oracle.signatures(data, offs, _oracle_fns(fns), L=L)
    assert np.array_equal(sig, want)
    # band sums of values near 2^31 (u64 sums, lsh.cpp:54)
    sig, band = minhash.signatures_packed(data, offs, _family(fns, L), bands=4, rows=8,
                                          bucket_count=977, ctx=ctx)
    assert np.array_equal(band, oracle.band_ids(want, 4, 8, 977))


def test_exact_arithmetic_equals_fast_kernels(ctx, oracle, monkeypatch):
    # the exact (64-bit Barrett) kernel on derive_family's own family agrees
    # with the FP32-quotient kernel and the oracle
    rng = np.random.default_rng(9)
    data, offs = _corpus(rng, n=60, lo=5, hi=5000)
    fam = minhash.derive_family(5, 128, 5)
    fast, _ = minhash.signatures_packed(data, offs, fam, ctx=ctx, want_bands=False)
    monkeypatch.setenv("ND_K1_EXACT", "1")
    ctx._family_key = None  # re-upload: the arithmetic is chosen at upload
    slow, _ = minhash.signatures_packed(data, offs, fam, ctx=ctx, want_bands=False)
    monkeypatch.delenv("ND_K1_EXACT")
    ctx._family_key = None
    assert np.array_equal(fast, slow)
    assert np.array_equal(fast, oracle.signatures(data, offs, oracle.derive_family(5, 128)))


@pytest.mark.parametrize("mutate,msg", [
    (dict(modulus=97, base=10, base_inverse=68, base_power=3, reduce_factor=(1 << 64) // 97), "residues"),
    (dict(base_inverse=5), "base_inverse"),
    (dict(base_power=7), "base_power"),
    (dict(reduce_factor=12345), "reduce_factor"),
])
def test_family_outside_reference_preconditions_is_config_error(ctx, mutate, msg):
    f = _fn(2097143, 65521, 5)
    for k, v in mutate.items():
        setattr(f, k, v)
    rng = np.random.default_rng(0)
    data, offs = _corpus(rng, n=4)
    with pytest.raises(_lib.ConfigError, match=msg):
        minhash.signatures_packed(data, offs, _family([f]), ctx=ctx, want_bands=False)


def test_codepoint_family_needs_moduli_above_max_scalar(ctx):
    f = _fn(1000003, 257, 5)  # fine for bytes, not for code points (> p)
    data = np.frombuffer("héllo wörld ✓ ok".encode(), np.uint8).copy()
    offs = np.array([0, len(data)], np.uint64)
    with pytest.raises(_lib.ConfigError, match="residues"):
        minhash.signatures_packed(data, offs, _family([f], unit=minhash.ShingleUnit.CODEPOINT),
                                  ctx=ctx, want_bands=False)


def test_codepoint_hand_built_family_exact(ctx, oracle):
    fns = [_fn(1114117, 65521, 5), _fn(2147483629, 3, 5), _fn(16777259, 40961, 5)]
    text = "".join(chr(c) for c in np.random.default_rng(1).integers(0x20, 0x10FFFF, 3000)
                   if not 0xD800 <= c < 0xE000)
    data = np.frombuffer(text.encode(), np.uint8).copy()
    offs = np.array([0, len(data)], np.uint64)
    fam = _family(fns, unit=minhash.ShingleUnit.CODEPOINT)
    sig, _ = minhash.signatures_packed(data, offs, fam, ctx=ctx, want_bands=False)
    want = oracle.signatures(data, offs, _oracle_fns(fns), unit=1)
    assert np.array_equal(sig, want)


def test_union_stage_self_loops_and_sparse_ids_vs_reference(ctx, ref, tmp_path):
    # a hand-edited .pairs file: self-loops (no group by themselves,
    # dedup_graph.cpp:70) and ids spread over 2^40 (dense renumbering, no
    # arrays sized by the largest id)
    from paper_2501_01046_b200 import compare as cmp

    corpus = str(tmp_path / "c.jsonl")
    ref.generate_synthetic(600, 40, gmin=2, gmax=3, len_min=300, len_max=600, seed=3,
                           corpus_path=corpus, truth_path=str(tmp_path / "t.jsonl"))
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=str(tmp_path / "g"))
    pipeline.run_dedup(cfg, ctx=ctx)
    stage = __import__("json").load(open(pipeline.compare_stage_path(cfg)))
    path = pipeline.pairs_dir(cfg) + "/" + stage["pair_files"][0]
    pairs = cmp.read_pair_file(path)
    big = 1 << 40
    extra = [DuplicatePair(5, 5, 100), DuplicatePair(big + 9, big + 9, 100),
             DuplicatePair(big + 3, big + 70000, 99), DuplicatePair(big + 70000, big + 123456, 99),
             DuplicatePair(7, big, 101), DuplicatePair(big + 1, big + 1, 100)]
    cmp.write_pair_file(path, pairs + extra)
    rep = pipeline.run_union_stage(cfg, ctx=ctx)
    allp = []
    for f in stage["pair_files"]:
        allp += cmp.read_pair_file(pipeline.pairs_dir(cfg) + "/" + f)
    lo = np.array([p.lo for p in allp], np.uint64)
    hi = np.array([p.hi for p in allp], np.uint64)
    reps, mem = ref.union(lo, hi)
    want = {}
    for r, m in zip(reps.tolist(), mem.tolist()):
        want.setdefault(r, []).append(m)
    assert [(g.representative, g.members) for g in rep.groups] == sorted(want.items())
    assert all(len(g.members) >= 2 for g in rep.groups)
    assert rep.near_duplicates == sorted(mem.tolist())
    assert (big + 9) not in rep.near_duplicates and (big + 3) in rep.near_duplicates
