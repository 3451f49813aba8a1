"""K2-K4 parity: compare, union and full dedup vs the reference itself.

Follows the reference's own tests: test_compare.cpp (tiled == naive over
n in {2,3,31,32,33,64} x thresholds, cross-band repeat suppression),
test_dedup_graph.cpp (transitive closure, order/repeat invariance, long
chains, min representative), and test_pipeline.cpp / acceptance 6 for whole
runs: groups.jsonl, removal.txt and summary.json must be byte-identical with
the reference's run_dedup on the same corpus, and candidate_pairs must match
the reference's compare_stage.json counter.
"""
import json
import os

import numpy as np
import pytest

from paper_2501_01046_b200 import _lib, compare, dedup_graph, lsh, minhash, pipeline
from paper_2501_01046_b200.compare import DuplicatePair, GatheredBucket, GatherResult, SimilarityThreshold

pytestmark = pytest.mark.gpu


def random_bucket(n, H, seed, alphabet=3):
    rng = np.random.default_rng(seed)
    b = GatheredBucket(lsh.BucketKey(0, 0), [i * 3 + 1 for i in range(n)],
                       rng.integers(0, alphabet, size=n * H).astype(np.uint32))
    return b


def naive(bucket, H, thr):
    n = len(bucket.doc_ids)
    sig = bucket.signatures.reshape(n, H)
    out = []
    for i in range(n):
        for j in range(i + 1, n):
            m = int((sig[i] == sig[j]).sum())
            if thr.accepts(m, H):
                out.append(DuplicatePair(bucket.doc_ids[i], bucket.doc_ids[j], m))
    return sorted(out, key=lambda p: (p.lo, p.hi))


@pytest.mark.parametrize("n", [2, 3, 31, 32, 33, 64, 127, 128, 129, 300])
@pytest.mark.parametrize("thr", [(1, 4), (1, 2), (3, 4)])
def test_compare_bucket_equals_naive(ctx, n, thr):
    t = SimilarityThreshold(thr)
    b = random_bucket(n, 8, 1000 + n)
    assert compare.compare_bucket(b, 8, t, ctx=ctx) == naive(b, 8, t)


@pytest.mark.parametrize("H,thr", [(128, (4, 5)), (256, (4, 5)), (64, (1, 2)), (16, (9, 10)),
                                   (128, (0, 1)), (128, (1, 1))])
def test_compare_planted_rows_vs_reference(ctx, ref, H, thr):
    # rows derived from a few bases with controlled mutation rates so match
    # counts straddle the threshold; many cells, sizes across tile boundaries
    rng = np.random.default_rng(H)
    buckets = []
    for c, n in enumerate([2, 5, 40, 129, 260]):
        base = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
        sig = np.tile(base, (n, 1))
        for r in range(n):
            k = int(rng.integers(0, H // 3))
            pos = rng.choice(H, size=k, replace=False)
            sig[r, pos] = rng.integers(0, 1 << 22, size=k)
        buckets.append(GatheredBucket(lsh.BucketKey(c, 0), list(range(c * 1000, c * 1000 + n)),
                                      sig.reshape(-1)))
    t = SimilarityThreshold(thr)
    got = compare.compare_pass(GatherResult(buckets), H, t, ctx=ctx)
    allsig = np.concatenate([b.signatures.reshape(-1, H) for b in buckets])
    ids = np.concatenate([b.doc_ids for b in buckets]).astype(np.uint64)
    offs = np.cumsum([0] + [len(b.doc_ids) for b in buckets]).astype(np.uint64)
    lo, hi, m = ref.compare_cells(allsig, offs, np.arange(len(ids), dtype=np.uint32), *thr,
                                  doc_ids=ids)
    want = [DuplicatePair(int(a), int(b), int(c)) for a, b, c in zip(lo, hi, m)]
    assert got == want
    if thr != (1, 1):
        assert got  # planted rows guarantee accepted pairs


def test_compare_pass_drops_cross_band_repeats(ctx):
    # test_compare.cpp:113-130
    first = GatheredBucket(lsh.BucketKey(0, 1), [10, 20], np.array([1, 2, 3, 4, 1, 2, 3, 9], np.uint32))
    second = GatheredBucket(lsh.BucketKey(1, 4), [10, 20], first.signatures.copy())
    pairs = compare.compare_pass(GatherResult([first, second]), 4, SimilarityThreshold((1, 2)), ctx=ctx)
    assert pairs == [DuplicatePair(10, 20, 3)]


def test_compare_validates(ctx):
    b = random_bucket(4, 8, 2)
    t = SimilarityThreshold((1, 2))
    with pytest.raises(_lib.ConfigError):
        compare.compare_bucket(b, 0, t, ctx=ctx)
    with pytest.raises(_lib.ConfigError):
        compare.compare_bucket(b, 8, t, tile_size=0, ctx=ctx)
    b.signatures = b.signatures[:-1]
    with pytest.raises(_lib.ConfigError):
        compare.compare_bucket(b, 8, t, ctx=ctx)


def groups_of(pairs, ctx):
    return dedup_graph.components(dedup_graph.union_pairs(
        [DuplicatePair(a, b, 9) for a, b in pairs], ctx=ctx))


def test_components_closure_and_representatives(ctx):
    g = groups_of([(1, 2), (2, 3), (8, 9)], ctx)
    assert [(x.representative, x.members) for x in g] == [(1, [1, 2, 3]), (8, [8, 9])]
    g = groups_of([(50, 7), (99, 50), (3, 2)], ctx)
    assert [(x.representative, x.members) for x in g] == [(2, [2, 3]), (7, [7, 50, 99])]
    g = groups_of([(i, i + 1) for i in range(1000)], ctx)
    assert len(g) == 1 and g[0].representative == 0 and len(g[0].members) == 1001
    assert groups_of([], ctx) == []


def test_components_order_and_repeats_invariant(ctx):
    pairs = [(1, 2), (2, 3), (3, 4), (10, 11), (11, 12), (1, 4), (20, 21)]
    want = groups_of(pairs, ctx)
    rng = np.random.default_rng(5)
    for trial in range(10):
        sh = [pairs[i] for i in rng.permutation(len(pairs))]
        if trial % 2:
            sh = sh + pairs
        assert groups_of(sh, ctx) == want


def test_components_random_graphs_vs_reference(ctx, ref):
    rng = np.random.default_rng(9)
    for n_nodes, n_edges in [(50, 40), (2000, 1500), (100000, 60000)]:
        lo = rng.integers(0, n_nodes, size=n_edges)
        hi = rng.integers(0, n_nodes, size=n_edges)
        keep = lo != hi
        lo, hi = np.minimum(lo, hi)[keep] * 7 + 3, np.maximum(lo, hi)[keep] * 7 + 3
        rep, mem = ref.union(lo.astype(np.uint64), hi.astype(np.uint64))
        g = groups_of(list(zip(lo.tolist(), hi.tolist())), ctx)
        got = [(x.representative, m) for x in g for m in x.members]
        assert got == list(zip(rep.tolist(), mem.tolist()))


def test_emit_report(ctx):
    r = dedup_graph.emit_report(groups_of([(1, 2), (5, 6), (6, 7)], ctx), 100, 3)
    assert r.near_duplicates == [1, 2, 5, 6, 7] and r.removals == [2, 6, 7]
    assert r.ratio == pytest.approx(0.05) and r.distinct_pairs == 3
    r = dedup_graph.emit_report([], 42, 0)
    assert r.groups == [] and r.ratio == 0.0


# ---- whole runs vs the reference's run_dedup ---------------------------------

def _files(ws):
    return {f: open(os.path.join(ws, f), "rb").read()
            for f in ("groups.jsonl", "removal.txt", "summary.json")}


def _run_both(ref, tmp_path, corpus_kwargs, cfg_kwargs, ctx):
    corpus = str(tmp_path / "corpus.jsonl")
    truth = str(tmp_path / "truth.jsonl")
    ref.generate_synthetic(corpus_path=corpus, truth_path=truth, **corpus_kwargs)
    ws_ref = str(tmp_path / "ws_ref")
    ws_gpu = str(tmp_path / "ws_gpu")
    os.makedirs(ws_ref)
    H = cfg_kwargs.get("hash_count", 128)
    bands = cfg_kwargs.get("bands", 16)
    rows = cfg_kwargs.get("rows", 8)
    thr = cfg_kwargs.get("threshold", (4, 5))
    ref.run_dedup(corpus, ws_ref, H=H, bands=bands, rows=rows, thr=thr, workers=os.cpu_count())
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu, **cfg_kwargs)
    rep = pipeline.run_dedup(cfg, ctx=ctx)
    stage = json.load(open(os.path.join(ws_ref, "compare_stage.json")))
    return _files(ws_ref), _files(ws_gpu), rep, stage


def test_c1_dedup_byte_identical(ctx, ref, tmp_path):
    # 10k docs, 500 planted pairs, 1600-2400 B, seed 1
    want, got, rep, stage = _run_both(
        ref, tmp_path, dict(doc_count=10000, group_count=500, len_min=1600, len_max=2400, seed=1),
        {}, ctx)
    assert got == want
    assert rep.candidate_pairs == stage["candidate_pairs"] == 4006931
    s = json.loads(want["summary.json"])
    assert s["duplicate_groups"] == 500 and s["near_duplicates"] == 1000
    assert want["groups.jsonl"].startswith(b'{"representative":14,"members":[14,549]}')


def test_dedup_h256_groups_of_five_byte_identical(ctx, ref, tmp_path):
    want, got, rep, stage = _run_both(
        ref, tmp_path, dict(doc_count=4000, group_count=300, gmin=2, gmax=5, edit=(3, 100),
                            len_min=300, len_max=900, seed=7),
        dict(hash_count=256, bands=32, rows=8), ctx)
    assert got == want
    assert rep.candidate_pairs == stage["candidate_pairs"]


@pytest.mark.parametrize("thr", [(1, 2), (9, 10)])
def test_dedup_thresholds_byte_identical(ctx, ref, tmp_path, thr):
    want, got, rep, stage = _run_both(
        ref, tmp_path, dict(doc_count=3000, group_count=200, gmin=2, gmax=4, edit=(8, 100),
                            len_min=250, len_max=700, seed=11),
        dict(threshold=thr), ctx)
    assert got == want
    assert rep.candidate_pairs == stage["candidate_pairs"]


def test_long_document_skew_vs_reference(ctx, ref, tmp_path):
    # lognormal lengths up to 60 KB (multi-item K1 path, skewed big cells)
    spec = _lib.NdSynthSpec(doc_count=1500, group_count=150, group_size_min=2, group_size_max=6,
                            edit_num=1, edit_den=100, len_min=3000, len_max=60000, seed=3,
                            mode=1, len_law=1, sigma_milli=1200)
    import ctypes as C

    lib = _lib.load()
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, None, C.byref(nb)))
    data = np.empty(nb.value, np.uint8)
    offs = np.empty(spec.doc_count + 1, np.uint64)
    _lib.check(lib.nd_synth_generate(C.byref(spec), data.ctypes.data_as(_lib.u8p),
                                     offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
    assert np.diff(offs).max() > 8196  # exercises multi-item documents
    corpus = str(tmp_path / "skew.jsonl")
    with open(corpus, "w") as f:
        for i in range(spec.doc_count):
            f.write(json.dumps({"text": bytes(data[offs[i]:offs[i + 1]]).decode()}) + "\n")
    ws_ref, ws_gpu = str(tmp_path / "r"), str(tmp_path / "g")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref, workers=os.cpu_count())
    rep = pipeline.run_dedup(pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu), ctx=ctx)
    assert _files(ws_gpu) == _files(ws_ref)
    assert rep.candidate_pairs == json.load(open(os.path.join(ws_ref, "compare_stage.json")))["candidate_pairs"]


def test_dedup_pairs_match_reference_pair_files(ctx, ref, tmp_path):
    # distinct pair set (lo, hi, match_count) vs the reference's .pairs files
    corpus = str(tmp_path / "c.jsonl")
    ref.generate_synthetic(2000, 150, gmin=2, gmax=3, len_min=300, len_max=800, seed=5,
                           corpus_path=corpus, truth_path=str(tmp_path / "t.jsonl"))
    ws_ref = str(tmp_path / "r")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref, workers=4)
    want = set()
    for f in os.listdir(os.path.join(ws_ref, "pairs")):
        for p in compare.read_pair_file(os.path.join(ws_ref, "pairs", f)):
            want.add((p.lo, p.hi, p.match_count))
    rep = pipeline.run_dedup(pipeline.RunConfig(inputs=[corpus], workspace=str(tmp_path / "g")),
                             ctx=ctx)
    got = pipeline.dedup_pairs(rep.distinct_pairs, ctx=ctx)
    assert [(p.lo, p.hi, p.match_count) for p in got] == sorted(want)


def test_join_and_all_pairs_paths_agree(ctx, ref, tmp_path, monkeypatch):
    # the same corpus through the hash join (default) and the all-pairs kernel
    corpus = str(tmp_path / "c.jsonl")
    ref.generate_synthetic(3000, 250, gmin=2, gmax=4, edit=(4, 100), len_min=300, len_max=900,
                           seed=23, corpus_path=corpus, truth_path=str(tmp_path / "t.jsonl"))
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ND_JOIN", mode)
        ws = str(tmp_path / f"g{mode}")
        rep = pipeline.run_dedup(pipeline.RunConfig(inputs=[corpus], workspace=ws), ctx=ctx)
        outs[mode] = (_files(ws), pipeline.dedup_pairs(rep.distinct_pairs, ctx=ctx))
    assert outs["1"] == outs["0"]
    assert outs["1"][1]


def test_giant_cells_mix_join_and_all_pairs(ctx, ref, tmp_path):
    # 4500 near-copies of one text put > kJoinMax (4096) documents into cells
    # (all-pairs kernel) while the random documents' cells go through the join
    rng = np.random.default_rng(31)
    alpha = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz0123456789 ", np.uint8)
    base = alpha[rng.integers(0, 37, size=700)]
    docs = []
    for i in range(4500):
        t = base.copy()
        pos = rng.integers(0, 700, size=int(rng.integers(0, 4)))
        t[pos] = alpha[rng.integers(0, 37, size=len(pos))]
        docs.append(t)
    docs += [alpha[rng.integers(0, 37, size=int(n))] for n in rng.integers(300, 900, size=1500)]
    order = rng.permutation(len(docs))
    corpus = str(tmp_path / "g.jsonl")
    with open(corpus, "w") as f:
        for i in order:
            f.write(json.dumps({"text": bytes(docs[i]).decode()}) + "\n")
    ws_ref, ws_gpu = str(tmp_path / "r"), str(tmp_path / "g")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref, workers=os.cpu_count())
    rep = pipeline.run_dedup(pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu), ctx=ctx)
    assert _files(ws_gpu) == _files(ws_ref)
    assert rep.stats is None or rep.candidate_pairs == json.load(
        open(os.path.join(ws_ref, "compare_stage.json")))["candidate_pairs"]


@pytest.mark.parametrize("thr", [(1, 2), (2, 5)])
def test_join_finds_pairs_whose_first_match_is_late(ctx, ref, thr):
    # low thresholds make P = H - min_matches + 1 > 32: pairs whose first
    # equal position lies beyond the 32-position prefix must still be found
    H = 128
    rng = np.random.default_rng(41)
    n = 120
    base = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
    sig = np.tile(base, (n, 1))
    for r in range(n):
        late = int(rng.integers(32, 60))  # positions [0, late) all differ
        sig[r, :late] = rng.integers(0, 1 << 22, size=late)
        k = int(rng.integers(0, 10))
        pos = rng.choice(np.arange(late, H), size=k, replace=False)
        sig[r, pos] = rng.integers(0, 1 << 22, size=k)
    b = GatheredBucket(lsh.BucketKey(0, 0), list(range(n)), sig.reshape(-1))
    t = SimilarityThreshold(thr)
    got = compare.compare_bucket(b, H, t, ctx=ctx)
    lo, hi, m = ref.compare_cells(sig, np.array([0, n], np.uint64), np.arange(n, dtype=np.uint32),
                                  *thr)
    assert got == [DuplicatePair(int(a), int(c), int(d)) for a, c, d in zip(lo, hi, m)]
    assert got


@pytest.mark.parametrize("n", [300, 6000])
def test_all_pairs_dupset_vs_reference(ctx, ref, n):
    # exhaustive oracle (oracle.cpp:53-108) on one cell of every document:
    # n=300 takes the hash join, n=6000 the tiled all-pairs kernel
    from paper_2501_01046_b200 import accuracy

    data, offs = ref.generate_synthetic(n, n // 10, gmin=2, gmax=3, edit=(3, 100), len_min=300,
                                        len_max=700, seed=n)
    sig, _ = ref.signatures(data, offs, K=0, workers=8)
    ids = np.arange(n, dtype=np.uint64) * 3 + 1
    want = ref.all_pairs_dupset(sig, 4, 5, doc_ids=ids)
    got = accuracy.all_pairs_dupset(sig, 128, SimilarityThreshold((4, 5)), ctx=ctx, doc_ids=ids)
    assert got.doc_ids == want.tolist()
    assert got.doc_ids


def test_codepoint_unit_dedup_byte_identical(ctx, ref, tmp_path):
    # --shingle-unit codepoint end to end: NFC-stable multi-byte text (Cyrillic,
    # Greek, CJK, emoji, ASCII), planted near-duplicate pairs
    import unicodedata

    rng = np.random.default_rng(17)
    alphabet = ([chr(c) for c in range(0x430, 0x450)] + [chr(c) for c in range(0x3B1, 0x3CA)]
                + [chr(c) for c in range(0x4E00, 0x4E80)] + [chr(c) for c in range(0x1F600, 0x1F640)]
                + list("abcdefghij    "))
    docs = []
    for _ in range(1200):
        docs.append("".join(rng.choice(alphabet, size=int(rng.integers(250, 900)))))
    for i in range(0, 300, 2):  # 150 near-duplicate pairs
        t = list(docs[i])
        for k in rng.choice(len(t), size=max(1, len(t) // 100), replace=False):
            t[k] = alphabet[int(rng.integers(len(alphabet)))]
        docs[i + 1] = "".join(t)
    order = rng.permutation(len(docs))
    corpus = str(tmp_path / "uni.jsonl")
    with open(corpus, "w", encoding="utf-8") as f:
        for i in order:
            assert unicodedata.is_normalized("NFC", docs[i])
            f.write(json.dumps({"text": docs[i]}, ensure_ascii=bool(i % 2)) + "\n")
    ws_ref, ws_gpu = str(tmp_path / "r"), str(tmp_path / "g")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref, workers=os.cpu_count(), unit=1)
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu, unit=pipeline.ShingleUnit.CODEPOINT)
    rep = pipeline.run_dedup(cfg, ctx=ctx)
    want = _files(ws_ref)
    assert _files(ws_gpu) == want
    assert json.loads(want["summary.json"])["duplicate_groups"] >= 140
    assert rep.candidate_pairs == json.load(open(os.path.join(ws_ref, "compare_stage.json")))["candidate_pairs"]


@pytest.mark.parametrize("H,thr", [(128, (4, 5)), (256, (4, 5)), (128, (9, 10)), (64, (1, 2)),
                                   (128, (0, 1)), (96, (3, 4))])
def test_pigeonhole_join_adversarial(ctx, ref, monkeypatch, H, thr):
    # pairs with close to A = H - min_matches mismatches spread one per block
    # (as few identical blocks as possible), plus low-entropy values so that
    # fingerprints and single positions collide a lot; both join modes and the
    # reference's compare_bucket agree
    rng = np.random.default_rng(H * 7 + thr[0])
    n = 220
    mm = _lib.load().nd_min_matches(H, thr[0], thr[1])
    A = H - mm
    NB = A + 1
    bw = max(w for w in (1, 2, 4, 8) if NB * w <= H) if NB <= H else 1
    base = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
    sig = np.empty((n, H), np.uint32)
    for r in range(n):
        row = base.copy()
        kind = r % 3
        if kind == 0:  # m mismatches, one per block, blocks chosen at random
            m = int(np.clip(A + rng.integers(-2, 3), 0, H))
            blocks = rng.permutation(max(NB, 1))[:m] if bw > 1 else rng.permutation(H)[:m]
            for b in blocks:
                p = int(b) * bw + int(rng.integers(0, bw)) if bw > 1 else int(b)
                row[p] = (row[p] + 1 + rng.integers(0, 3)) % (1 << 22)
            extra = max(0, m - len(blocks))
            row[rng.choice(H, size=extra, replace=False)] ^= 1
        elif kind == 1:  # low-entropy values: many equal positions between rows
            row = rng.integers(0, 6, size=H).astype(np.uint32)
        elif r % 9 == 2:  # copies of the base: pairs with the kind-0 rows near the bound
            pass
        else:  # random row
            row = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
        sig[r] = row
    b = GatheredBucket(lsh.BucketKey(0, 0), list(range(n)), sig.reshape(-1))
    t = SimilarityThreshold(thr)
    lo, hi, m = ref.compare_cells(sig, np.array([0, n], np.uint64), np.arange(n, dtype=np.uint32),
                                  *thr)
    want = [DuplicatePair(int(a), int(c), int(d)) for a, c, d in zip(lo, hi, m)]
    for mode in ("1", "0"):
        monkeypatch.setenv("ND_JOIN_BLOCKS", mode)
        got = compare.compare_bucket(b, H, t, ctx=ctx)
        assert got == want, (mode, len(got), len(want))
    assert want


@pytest.mark.parametrize("n,H", [(700, 128), (2600, 128), (900, 256)])
def test_block_join_handled_pair_set_overflow(ctx, ref, monkeypatch, n, H):
    # one big cluster: every pair is a near-duplicate rediscovered in almost
    # every block, far more pairs than the handled-pair set holds (2^k >=
    # n/2 slots), so the join falls back to checking earlier blocks in HBM;
    # with the set, without it (ND_JOIN_PSET=0) and the reference agree
    rng = np.random.default_rng(n + H)
    base = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
    sig = np.tile(base, (n, 1))
    hit = rng.random((n, H)) < rng.choice([0.02, 0.08, 0.25], size=n)[:, None]
    sig[hit] = rng.integers(0, 1 << 22, size=int(hit.sum())).astype(np.uint32)
    sig[n // 2:] = rng.integers(0, 1 << 22, size=(n - n // 2, H)).astype(np.uint32)
    idx = np.arange(n // 2, n - 1, 7)
    sig[idx] = sig[idx + 1]  # exact pairs in the random half
    b = GatheredBucket(lsh.BucketKey(0, 0), list(range(n)), sig.reshape(-1))
    lo, hi, m = ref.compare_cells(sig, np.array([0, n], np.uint64), np.arange(n, dtype=np.uint32),
                                  4, 5)
    want = [DuplicatePair(int(a), int(c), int(d)) for a, c, d in zip(lo, hi, m)]
    assert len(want) > n
    for mode in ("1", "0"):
        monkeypatch.setenv("ND_JOIN_PSET", mode)
        assert compare.compare_bucket(b, H, SimilarityThreshold((4, 5)), ctx=ctx) == want, mode
    # one barrier per block (double-buffered chain links, the default) and
    # the second barrier after each walk agree on the heaviest walks
    monkeypatch.setenv("ND_JOIN_PSET", "1")
    for mode in ("1", "0"):
        monkeypatch.setenv("ND_JOIN_TWO_BARRIERS", mode)
        assert compare.compare_bucket(b, H, SimilarityThreshold((4, 5)), ctx=ctx) == want, mode


def test_estimator_error_stats(ctx, oracle):
    # oracle.cpp:143-162: per pair exact window Jaccard vs signature estimate
    from paper_2501_01046_b200 import accuracy

    rng = np.random.default_rng(5)
    base = bytes(rng.integers(97, 123, size=800, dtype=np.uint8))
    edit = bytearray(base)
    for i in rng.choice(800, size=20, replace=False):
        edit[i] = 97 + (edit[i] - 96) % 26
    other = bytes(rng.integers(97, 123, size=700, dtype=np.uint8))
    D = minhash.CleanDocument
    pairs = [(D(0, base), D(1, base)), (D(2, base), D(3, bytes(edit))), (D(4, base), D(5, other))]
    fam = minhash.derive_family(5, 128, 5)
    st = accuracy.estimator_error_stats(pairs, fam, ctx=ctx)
    assert st.samples[0].exact_jaccard == 1.0 and st.samples[0].estimated == 1.0
    assert 0.5 < st.samples[1].exact_jaccard < 0.95
    sigs = oracle.signatures(np.frombuffer(base + bytes(edit), np.uint8).copy(),
                             np.array([0, 800, 1600], np.uint64), oracle.derive_family(5, 128))
    assert st.samples[1].estimated == (sigs[0] == sigs[1]).sum() / 128
    assert st.samples[2].exact_jaccard < 0.05
    assert abs(st.mean_abs_error - sum(s.abs_error for s in st.samples) / 3) < 1e-12
    # codepoint windows
    j = accuracy.exact_window_jaccard("ЖЖЖЖЖa", "ЖЖЖЖЖb", 5, minhash.ShingleUnit.CODEPOINT)
    assert (j.intersection, j.union_size) == (1, 3)


@pytest.mark.parametrize("budget", [3_000_000, 400_000])
def test_out_of_core_dedup_byte_identical(ctx, ref, tmp_path, budget):
    # a small HBM budget cuts the buckets into intervals (plan_gather's idea,
    # sigstore.cpp:288-329): pairs, groups and the report must equal the
    # single-pass dedup's and the reference's
    data, offs = ref.generate_synthetic(6000, 500, gmin=2, gmax=4, edit=(3, 100), len_min=300,
                                        len_max=900, seed=19)
    one = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
    assert one.stats["intervals"] == 1
    p1 = pipeline.dedup_pairs(one.distinct_pairs, ctx=ctx)
    d1 = str(tmp_path / "one")
    os.makedirs(d1)
    pipeline.write_report(d1, ctx=ctx)
    sig1 = minhash.signatures_packed(data, offs, minhash.derive_family(5, 128, 5), 16, 8,
                                     one.stats["bucket_count"], ctx=ctx)
    ooc = pipeline.dedup_packed(data, offs, pipeline.RunConfig(hbm_budget=budget), ctx=ctx)
    assert ooc.stats["intervals"] >= 2, ooc.stats
    assert ooc.candidate_pairs == one.candidate_pairs
    assert ooc.stats["emitted_pairs"] >= one.stats["emitted_pairs"]
    assert pipeline.dedup_pairs(ooc.distinct_pairs, ctx=ctx) == p1
    d2 = str(tmp_path / "ooc")
    os.makedirs(d2)
    pipeline.write_report(d2, ctx=ctx)
    assert _files(d2) == _files(d1)
    assert [(g.representative, g.members) for g in ooc.groups] == \
        [(g.representative, g.members) for g in one.groups]
    # rows fetched from host memory equal K1's
    import ctypes as C
    n = len(offs) - 1
    sig = np.empty((n, 128), np.uint32)
    band = np.empty((n, 16), np.uint32)
    ctx.check(ctx.lib.nd_dedup_fetch_signatures(ctx.h, sig.ctypes.data_as(_lib.u32p),
                                                band.ctypes.data_as(_lib.u32p)))
    assert np.array_equal(sig, sig1[0]) and np.array_equal(band, sig1[1])
    # and the reference's run_dedup on the same documents
    corpus = str(tmp_path / "c.jsonl")
    with open(corpus, "w") as f:
        for i in range(n):
            f.write(json.dumps({"text": bytes(data[offs[i]:offs[i + 1]]).decode()}) + "\n")
    ws_ref = str(tmp_path / "r")
    os.makedirs(ws_ref)
    _, cand = ref.run_dedup(corpus, ws_ref, workers=os.cpu_count())
    assert cand == ooc.candidate_pairs
    assert _files(ws_ref)["groups.jsonl"] == _files(d2)["groups.jsonl"]
