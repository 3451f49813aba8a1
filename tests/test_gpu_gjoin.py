"""K3g -- the in-memory dedup's global block join (csrc/k_gjoin.cu) -- against
the per-cell joins (ND_K3=cells) and the reference's compare_pass over the
same cells.

K3g never forms the cells: it joins every block once over all rows and keeps
a pair only if the two rows share a cell (a band with equal bucket ids) and
pass the reference's count (compare.cpp:24-67).  So the shapes that matter are
pairs close to the mismatch bound with as few identical blocks as possible,
near-duplicates that share NO cell (found by the join, must be dropped),
low-entropy rows (fingerprint and table-slot collisions, long chains), every
block width BW in {1, 2, 4, 8}, thresholds whose NB is too large for K3g (the
per-cell path takes them) or zero (no pair possible), and the reference's
counters: candidate pairs (sum n(n-1)/2), non-singleton cells and the
emitted pairs (one per shared cell).
"""
import os

import numpy as np
import pytest

from paper_2501_01046_b200 import _lib, pipeline

pytestmark = pytest.mark.gpu


def _cells(band, K):
    """CSR cells (band-major, bucket order, rows ascending) as scan_gather builds them."""
    n, B = band.shape
    offs, rows = [0], []
    for j in range(B):
        order = np.argsort(band[:, j], kind="stable")
        keys = band[order, j]
        bounds = np.searchsorted(keys, np.arange(K + 1))
        for b in range(K):
            rows.extend(order[bounds[b]:bounds[b + 1]].tolist())
            offs.append(len(rows))
    return np.array(offs, np.uint64), np.array(rows, np.uint32)


def _adversarial(rng, n, H, mm):
    A = H - mm
    NB = A + 1
    bw = max([w for w in (1, 2, 4, 8) if NB * w <= H], default=1)
    base = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
    sig = np.empty((n, H), np.uint32)
    for r in range(n):
        kind = r % 4
        row = base.copy()
        if kind == 0:  # about A mismatches, one per block
            m = int(np.clip(A + rng.integers(-2, 3), 0, H))
            blocks = rng.permutation(max(NB, 1))[:m] if bw > 1 else rng.permutation(H)[:m]
            for b in blocks:
                p = int(b) * bw + int(rng.integers(0, bw)) if bw > 1 else int(b)
                row[p] = (row[p] + 1 + rng.integers(0, 3)) % (1 << 22)
        elif kind == 1:  # low entropy: many equal positions and blocks
            row = rng.integers(0, 4, size=H).astype(np.uint32)
        elif kind == 2:  # a few mismatches from the base
            hit = rng.random(H) < 0.05
            row[hit] = rng.integers(0, 1 << 22, size=int(hit.sum()))
        else:
            row = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
        sig[r] = row
    return sig


def _both(ctx, monkeypatch, sig, band, cfg, K):
    out = {}
    for kind in ("global", "cells"):
        if kind == "cells":
            monkeypatch.setenv("ND_K3", "cells")
        else:
            monkeypatch.delenv("ND_K3", raising=False)
        rep = pipeline.dedup_signatures(sig, band, cfg, bucket_count=K, ctx=ctx)
        st = {k: v for k, v in rep.stats.items() if k != "seconds"}
        out[kind] = (pipeline.dedup_compare_kind(ctx), st,
                     pipeline.dedup_pairs(rep.distinct_pairs, ctx=ctx),
                     [(g.representative, g.members) for g in rep.groups])
    monkeypatch.delenv("ND_K3", raising=False)
    return out


@pytest.mark.parametrize("H,bands,rows,thr,kind", [
    (128, 16, 8, (4, 5), "global"),    # NB 26, BW 4
    (128, 16, 8, (9, 10), "global"),   # NB 13, BW 8
    (64, 8, 8, (1, 2), "global"),      # NB 32, BW 2
    (16, 4, 4, (1, 10), "global"),     # NB 15, BW 1
    (256, 32, 8, (4, 5), "global"),    # NB 52, BW 4
    (96, 12, 8, (3, 4), "global"),     # NB 24, BW 4
    (100, 10, 10, (4, 5), "global"),   # H % 4 != 0 (scalar block loads), NB 20, BW 4
    (128, 16, 8, (1, 4), "cells"),     # NB 96 > 64: the per-cell joins
    (128, 16, 8, (1, 1), "global"),    # min_matches > H: no block, no pair
])
def test_global_join_vs_cells_and_reference(ctx, ref, monkeypatch, H, bands, rows, thr, kind):
    rng = np.random.default_rng(H * 31 + thr[0] * 7 + thr[1])
    n = 900
    mm = _lib.load().nd_min_matches(H, thr[0], thr[1])
    sig = _adversarial(rng, n, H, min(mm, H))
    K = 5  # few buckets: most pairs share cells, ~(4/5)^bands share none
    band = rng.integers(0, K, size=(n, bands)).astype(np.uint32)
    # a few near-duplicate pairs that share no cell at all
    for r in range(0, 60, 2):
        band[r + 1] = (band[r] + 1) % K
    cfg = pipeline.RunConfig(hash_count=H, bands=bands, rows=rows, threshold=thr)
    out = _both(ctx, monkeypatch, sig, band, cfg, K)
    assert out["global"][0] == kind and out["cells"][0] == "cells"
    assert out["global"][1:] == out["cells"][1:]
    offs, crow = _cells(band, K)
    lo, hi, m = ref.compare_cells(sig, offs, crow, *thr)
    want = [(int(a), int(b), int(c)) for a, b, c in zip(lo, hi, m)]
    got = [(p.lo, p.hi, p.match_count) for p in out["global"][2]]
    assert got == want
    timed, _, _ = ref.compare_cells_timed(sig, offs, crow, *thr, workers=os.cpu_count())
    st = out["global"][1]
    assert st["emitted_pairs"] == timed["emitted"]
    sizes = np.diff(offs.astype(np.int64))
    assert st["candidate_pairs"] == int((sizes * (sizes - 1) // 2).sum())
    assert st["nonsingleton_cells"] == int((sizes >= 2).sum())
    assert st["cell_records"] == int(sizes[sizes >= 2].sum())
    if mm <= H and kind == "global":
        assert want  # the shapes do produce pairs


def test_global_join_long_chains_and_doc_ids(ctx, ref, monkeypatch):
    # 40k rows over a 60-value alphabet at BW = 1: every position value is
    # shared by ~700 rows (long chains in every table slot, most chained
    # pairs equal at the block but not near-duplicates), doc ids not 0..n-1
    rng = np.random.default_rng(5)
    n, H, bands, rows = 40000, 16, 4, 4
    sig = rng.integers(0, 60, size=(n, H)).astype(np.uint32)
    sig[1::97] = sig[0::97][: len(sig[1::97])]  # exact copies
    K = 3000
    band = rng.integers(0, K, size=(n, bands)).astype(np.uint32)
    band[1::97] = band[0::97][: len(band[1::97])]
    ids = np.cumsum(rng.integers(1, 5, size=n)).astype(np.uint64)
    cfg = pipeline.RunConfig(hash_count=H, bands=bands, rows=rows, threshold=(1, 4))
    res = {}
    for kind in ("global", "cells"):
        if kind == "cells":
            monkeypatch.setenv("ND_K3", "cells")
        rep = pipeline.dedup_signatures(sig, band, cfg, doc_ids=ids, bucket_count=K, ctx=ctx)
        assert pipeline.dedup_compare_kind(ctx) == kind
        res[kind] = (rep.stats["emitted_pairs"], rep.candidate_pairs,
                     pipeline.dedup_pairs(rep.distinct_pairs, ctx=ctx))
    monkeypatch.delenv("ND_K3", raising=False)
    assert res["global"] == res["cells"]
    offs, crow = _cells(band, K)
    lo, hi, m = ref.compare_cells(sig, offs, crow, 1, 4, doc_ids=ids)
    assert [(p.lo, p.hi, p.match_count) for p in res["global"][2]] == \
        [(int(a), int(b), int(c)) for a, b, c in zip(lo, hi, m)]
    assert len(lo) > 100


def test_dedup_packed_global_vs_cells_vs_reference(ctx, ref, monkeypatch, tmp_path):
    # text through K1 -> K3g -> K4 (nd_dedup) against the per-cell path and the
    # reference's run_dedup report
    data, offs = ref.generate_synthetic(8000, 700, gmin=2, gmax=5, edit=(2, 100), len_min=300,
                                        len_max=1500, seed=29)
    res = {}
    for kind in ("global", "cells"):
        if kind == "cells":
            monkeypatch.setenv("ND_K3", "cells")
        rep = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
        assert pipeline.dedup_compare_kind(ctx) == kind
        d = str(tmp_path / kind)
        os.makedirs(d)
        pipeline.write_report(d, ctx=ctx)
        st = {k: v for k, v in rep.stats.items() if k != "seconds"}
        res[kind] = (st, pipeline.dedup_pairs(rep.distinct_pairs, ctx=ctx),
                     {f: open(os.path.join(d, f), "rb").read()
                      for f in ("groups.jsonl", "removal.txt", "summary.json")})
    monkeypatch.delenv("ND_K3", raising=False)
    assert res["global"] == res["cells"]
    corpus = str(tmp_path / "c.jsonl")
    import json
    with open(corpus, "w") as f:
        for i in range(len(offs) - 1):
            f.write(json.dumps({"text": bytes(data[int(offs[i]):int(offs[i + 1])]).decode()}) + "\n")
    ws = str(tmp_path / "ref")
    os.makedirs(ws)
    _, cand = ref.run_dedup(corpus, ws, workers=os.cpu_count())
    assert open(os.path.join(ws, "groups.jsonl"), "rb").read() == res["global"][2]["groups.jsonl"]
    assert res["global"][0]["candidate_pairs"] == cand


def test_dedup_signatures_validates(ctx):
    sig = np.zeros((4, 128), np.uint32)
    band = np.zeros((4, 16), np.uint32)
    band[2, 3] = 50
    with pytest.raises(_lib.ConfigError, match="bucket count"):
        pipeline.dedup_signatures(sig, band, pipeline.RunConfig(), bucket_count=50, ctx=ctx)
    with pytest.raises(_lib.ConfigError):
        pipeline.dedup_signatures(sig[:, :64], band, pipeline.RunConfig(), bucket_count=50, ctx=ctx)


def test_global_join_identical_rows_and_tiny_batches(ctx, ref, monkeypatch):
    # every row identical (one chain of n rows in every block's slot: the
    # pairs are checked at block 0 and rejected at every later block), then
    # batches of 2 and 3 rows
    H, bands, rows = 128, 16, 8
    rng = np.random.default_rng(3)
    base = rng.integers(0, 1 << 22, size=H).astype(np.uint32)
    cfg = pipeline.RunConfig(hash_count=H, bands=bands, rows=rows)
    for n in (2500, 2, 3):
        sig = np.tile(base, (n, 1))
        if n == 3:
            sig[2] = rng.integers(0, 1 << 22, size=H)
        band = np.tile(rng.integers(0, 7, size=bands).astype(np.uint32), (n, 1))
        out = _both(ctx, monkeypatch, sig, band, cfg, 7)
        assert out["global"][0] == "global"
        assert out["global"][1:] == out["cells"][1:]
        want_pairs = n * (n - 1) // 2 if n != 3 else 1
        assert out["global"][1]["distinct_pairs"] == want_pairs
        assert out["global"][1]["emitted_pairs"] == want_pairs * bands


def test_stage_cell_hist_counts_and_rejects_bad_ids(ctx):
    import ctypes as C

    import torch

    rng = np.random.default_rng(11)
    n, B, K = 5000, 16, 300
    band = rng.integers(0, K, size=(n, B)).astype(np.uint32)
    d_band = torch.from_numpy(band.view(np.int32)).cuda()
    cnt = torch.empty(B * K, dtype=torch.int32, device="cuda")
    ctx.check(ctx.lib.nd_stage_cell_hist(ctx.h, C.c_void_p(d_band.data_ptr()), n, B, K,
                                         C.c_void_p(cnt.data_ptr())))
    want = np.zeros(B * K, np.int64)
    np.add.at(want, (np.arange(B)[None, :] * K + band).ravel(), 1)
    assert np.array_equal(cnt.cpu().numpy(), want)
    band[17, 3] = K
    d_band = torch.from_numpy(band.view(np.int32)).cuda()
    with pytest.raises(_lib.ConfigError, match="bucket count"):
        ctx.check(ctx.lib.nd_stage_cell_hist(ctx.h, C.c_void_p(d_band.data_ptr()), n, B, K,
                                             C.c_void_p(cnt.data_ptr())))
