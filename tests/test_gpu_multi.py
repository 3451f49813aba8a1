"""Multi-GPU behind the C-ABI (nd_ctx_create_multi): the batch is sharded by
document ranges, (cell, row) records go all-to-all over peer copies, every
owner compares its cells reading rows in place, pairs meet on the first device.
On a one-GPU box the shards share the device (the same code path: peer copies
and peer row reads on one device).  Outputs must equal the single-device run
and the reference's run_dedup for any shard count (test_pipeline.cpp:163-179's
worker-count invariance, generalised to GPUs)."""
import json
import os

import numpy as np
import pytest

from paper_2501_01046_b200 import minhash, pipeline
from paper_2501_01046_b200.device import Context

pytestmark = pytest.mark.gpu


def _files(ws):
    return {f: open(os.path.join(ws, f), "rb").read()
            for f in ("groups.jsonl", "removal.txt", "summary.json")}


@pytest.fixture(scope="module")
def corpus(ref, tmp_path_factory):
    d = tmp_path_factory.mktemp("multi")
    path = str(d / "c.jsonl")
    data, offs = ref.generate_synthetic(4000, 300, gmin=2, gmax=4, edit=(3, 100), len_min=300,
                                        len_max=1500, seed=77, corpus_path=path,
                                        truth_path=str(d / "t.jsonl"))
    ws = str(d / "ref")
    os.makedirs(ws)
    _, cand = ref.run_dedup(path, ws, workers=os.cpu_count())
    return data, offs, _files(ws), cand


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_multi_dedup_byte_identical(corpus, tmp_path, shards):
    data, offs, want, cand = corpus
    ctx = Context(devices=[0] * shards)
    assert ctx.shards == shards
    rep = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
    assert rep.candidate_pairs == cand
    assert pipeline.dedup_compare_kind(ctx) == "global"
    ws = str(tmp_path / "g")
    pipeline.write_report(ws, ctx=ctx)
    assert _files(ws) == want
    # the signatures gathered from the shards equal the single-device K1
    n = len(offs) - 1
    import ctypes as C
    from paper_2501_01046_b200 import _lib
    sig = np.empty((n, 128), np.uint32)
    band = np.empty((n, 16), np.uint32)
    ctx.check(ctx.lib.nd_dedup_fetch_signatures(ctx.h, sig.ctypes.data_as(_lib.u32p),
                                                band.ctypes.data_as(_lib.u32p)))
    one = Context(0)
    s1, b1 = minhash.signatures_packed(data, offs, minhash.derive_family(5, 128, 5), 16, 8,
                                       rep.stats["bucket_count"], ctx=one)
    assert np.array_equal(sig, s1) and np.array_equal(band, b1)
    one.close()
    ctx.close()


@pytest.mark.parametrize("shards", [2, 5])
def test_multi_signatures_and_doc_ids(corpus, shards):
    data, offs, _, _ = corpus
    fam = minhash.derive_family(5, 128, 5)
    ctx = Context(devices=[0] * shards)
    one = Context(0)
    s, b = minhash.signatures_packed(data, offs, fam, 16, 8, 200, ctx=ctx)
    s1, b1 = minhash.signatures_packed(data, offs, fam, 16, 8, 200, ctx=one)
    assert np.array_equal(s, s1) and np.array_equal(b, b1)
    ids = np.arange(len(offs) - 1, dtype=np.uint64) * 7 + 3
    r = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), doc_ids=ids, ctx=ctx)
    r1 = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), doc_ids=ids, ctx=one)
    assert [(g.representative, g.members) for g in r.groups] == \
        [(g.representative, g.members) for g in r1.groups]
    assert pipeline.dedup_pairs(r.distinct_pairs, ctx=ctx) == pipeline.dedup_pairs(r1.distinct_pairs, ctx=one)
    one.close()
    ctx.close()


def test_multi_more_shards_than_documents(ref):
    data, offs = ref.generate_synthetic(6, 2, gmin=2, gmax=2, len_min=300, len_max=400, seed=1)
    ctx = Context(devices=[0] * 8)
    one = Context(0)
    r = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
    r1 = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=one)
    assert [g.members for g in r.groups] == [g.members for g in r1.groups]
    one.close()
    ctx.close()


@pytest.mark.parametrize("shards,thr", [(3, (4, 5)), (16, (9, 10))])
def test_multi_global_and_cell_joins_agree(corpus, monkeypatch, shards, thr):
    # K3g on a device group (block k joined by shard k mod G over every
    # shard's rows, read in place; 16 shards > 13 blocks leaves owners idle)
    # against the per-cell joins on the group and K3g on one device: pairs,
    # groups and every counter equal
    data, offs, _, _ = corpus
    cfg = pipeline.RunConfig(threshold=thr)
    res = {}
    for name, devs, env in (("group", [0] * shards, None), ("group_cells", [0] * shards, "cells"),
                            ("one", [0], None)):
        if env:
            monkeypatch.setenv("ND_K3", env)
        else:
            monkeypatch.delenv("ND_K3", raising=False)
        ctx = Context(devices=devs) if len(devs) > 1 else Context(0)
        r = pipeline.dedup_packed(data, offs, cfg, ctx=ctx)
        kind = pipeline.dedup_compare_kind(ctx)
        st = {k: v for k, v in r.stats.items() if k not in ("seconds",)}
        res[name] = (st, pipeline.dedup_pairs(r.distinct_pairs, ctx=ctx),
                     [(g.representative, g.members) for g in r.groups])
        assert kind == ("cells" if env else "global"), (name, kind)
        ctx.close()
    monkeypatch.delenv("ND_K3", raising=False)
    assert res["group"] == res["one"]
    assert res["group"][1:] == res["group_cells"][1:]
    for k in ("candidate_pairs", "emitted_pairs", "nonsingleton_cells", "cell_records",
              "distinct_pairs"):
        assert res["group"][0][k] == res["group_cells"][0][k], k
