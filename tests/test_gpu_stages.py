"""The staged, file-backed workflow on the GPU (hash -> gather-compare -> union)
against the reference's own run_dedup: EVERY artifact of the workspace is
compared byte for byte -- .feds signature files, per-(worker, pass) .pairs
files, run_manifest.json, compare_stage.json, rejects.jsonl and the report
(test_pipeline.cpp's artifact checks, pipeline.cpp:269-532)."""
import json
import os

import pytest

from paper_2501_01046_b200 import _lib, pipeline

pytestmark = pytest.mark.gpu


def _corpus_dir(ref, tmp_path, n=1500, groups=150, seed=4):
    src = str(tmp_path / "all.jsonl")
    ref.generate_synthetic(n, groups, gmin=2, gmax=4, len_min=300, len_max=1200, seed=seed,
                           corpus_path=src, truth_path=str(tmp_path / "truth.jsonl"))
    lines = open(src, encoding="utf-8").read().splitlines(keepends=True)
    d = tmp_path / "corpus"
    d.mkdir()
    half = len(lines) // 2
    bad = ['not json\n', '[1, 2]\n', '{"id": 1}\n', '{"text": 5}\n', '{"text": "too short"}\n', '\n']
    (d / "a.jsonl").write_text("".join(lines[:half] + bad[:3]), encoding="utf-8")
    (d / "b.jsonl").write_text("".join(bad[3:] + lines[half:]), encoding="utf-8")
    (d / "ignored.txt").write_text("not an input\n")
    return str(d)


def _tree(ws):
    out = {}
    for root, _, files in os.walk(ws):
        for f in files:
            if f == "timings.json":
                continue  # wall-clock, not an artifact
            p = os.path.join(root, f)
            out[os.path.relpath(p, ws)] = open(p, "rb").read()
    return out


@pytest.mark.parametrize("workers,budget,hbm", [(1, 1 << 30, 0), (1, 120_000, 0), (3, 300_000, 0),
                                                (20, 1 << 30, 0), (1, 120_000, 250_000),
                                                (3, 300_000, 400_000)])
def test_staged_workspace_byte_identical(ctx, ref, tmp_path, workers, budget, hbm):
    # hbm > 0: a tiny HBM budget forces the out-of-core compare (several
    # bucket intervals, each a union of whole gather passes)
    corpus = _corpus_dir(ref, tmp_path)
    ws_ref, ws_gpu = str(tmp_path / "ref"), str(tmp_path / "gpu")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref, workers=workers, memory_budget=budget)
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu, workers=workers,
                             memory_budget=budget, hbm_budget=hbm)
    if hbm:
        pipeline.run_hash_stage(cfg, ctx=ctx)
        c = pipeline.run_compare_stage(cfg, ctx=ctx)
        assert c.intervals > 2, c.intervals
    rep = pipeline.run_dedup(cfg, ctx=ctx)
    want, got = _tree(ws_ref), _tree(ws_gpu)
    assert sorted(got) == sorted(want)
    assert any(k.startswith("signatures/") for k in want)
    npairs = sum(k.startswith("pairs/") for k in want)
    assert npairs >= workers if workers <= 16 else npairs == 16
    cs_ref = json.loads(want.pop("compare_stage.json"))
    cs_gpu = json.loads(got.pop("compare_stage.json"))
    if workers > 1:  # the reference's gauge peak depends on thread timing
        cs_ref.pop("gather_peak_bytes")
        cs_gpu.pop("gather_peak_bytes")
    else:
        assert (open(os.path.join(ws_gpu, "compare_stage.json"), "rb").read()
                == open(os.path.join(ws_ref, "compare_stage.json"), "rb").read())
    assert cs_gpu == cs_ref
    for k in want:
        assert got[k] == want[k], k
    assert rep.distinct_pairs == json.loads(want["summary.json"])["distinct_pairs"]
    rej = want["rejects.jsonl"].decode().splitlines()
    assert len(rej) == 5 and '"reason":"invalid_json"' in rej[0]


def test_stages_run_separately_and_rerun(ctx, ref, tmp_path):
    corpus = _corpus_dir(ref, tmp_path, n=600, groups=60, seed=9)
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=str(tmp_path / "ws"), workers=2,
                             memory_budget=80_000)
    with pytest.raises(_lib.PrerequisiteError):
        pipeline.run_compare_stage(cfg, ctx=ctx)  # no hash stage yet
    h = pipeline.run_hash_stage(cfg, ctx=ctx)
    assert h.bucket_count == 49 and len(h.signature_files) == 2
    with pytest.raises(_lib.PrerequisiteError):
        pipeline.run_union_stage(cfg, ctx=ctx)  # no compare stage yet
    c = pipeline.run_compare_stage(cfg, ctx=ctx)
    assert c.pass_count == len(c.pair_files) > 2
    r1 = pipeline.run_union_stage(cfg, ctx=ctx)
    before = _tree(cfg.workspace)
    r2 = pipeline.run_union_stage(cfg, ctx=ctx)
    assert _tree(cfg.workspace) == before
    assert [g.members for g in r1.groups] == [g.members for g in r2.groups]
    # artifact-shaping config changed -> the later stages refuse
    cfg.seed = 6
    with pytest.raises(_lib.ConfigError):
        pipeline.run_compare_stage(cfg, ctx=ctx)
    cfg.seed = 5
    # the schedule (workers, budget) does not shape the report
    cfg.workers, cfg.memory_budget = 1, 1 << 30
    pipeline.run_compare_stage(cfg, ctx=ctx)
    pipeline.run_union_stage(cfg, ctx=ctx)
    after = _tree(cfg.workspace)
    for f in ("groups.jsonl", "removal.txt", "summary.json"):
        assert after[f] == before[f]


def test_codepoint_staged_matches_in_memory(ctx, ref, tmp_path):
    corpus = _corpus_dir(ref, tmp_path, n=500, groups=50, seed=12)
    a = pipeline.RunConfig(inputs=[corpus], workspace=str(tmp_path / "a"),
                           unit=pipeline.ShingleUnit.CODEPOINT)
    b = pipeline.RunConfig(inputs=[corpus], workspace=str(tmp_path / "b"),
                           unit=pipeline.ShingleUnit.CODEPOINT)
    pipeline.run_dedup(a, ctx=ctx)
    pipeline.run_dedup_in_memory(b, ctx=ctx)
    ta, tb = _tree(a.workspace), _tree(b.workspace)
    for f in ("groups.jsonl", "removal.txt", "summary.json", "rejects.jsonl"):
        assert ta[f] == tb[f]


def test_eval_accuracy_byte_identical(ctx, ref, tmp_path):
    # run_eval_accuracy (pipeline.cpp:534-585): pipeline LSH dupset vs the
    # exhaustive all-pairs dupset over the same .feds signatures
    from paper_2501_01046_b200 import accuracy

    corpus = _corpus_dir(ref, tmp_path, n=1200, groups=200, seed=21)
    ws_ref, ws_gpu = str(tmp_path / "r"), str(tmp_path / "g")
    os.makedirs(ws_ref)
    ref.eval_accuracy(corpus, ws_ref, workers=4)
    acc = accuracy.run_eval_accuracy(pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu), ctx=ctx)
    want = open(os.path.join(ws_ref, "accuracy.json"), "rb").read()
    assert open(os.path.join(ws_gpu, "accuracy.json"), "rb").read() == want
    assert acc["corpus_size"] == 1200


@pytest.mark.parametrize("H,bands,rows,thr,L", [(100, 20, 5, (4, 5), 5), (60, 12, 5, (3, 4), 4),
                                                (512, 64, 8, (4, 5), 5), (32, 8, 4, (1, 2), 3),
                                                (256, 16, 16, (9, 10), 7)])
def test_unusual_shapes_workspace_byte_identical(ctx, ref, tmp_path, H, bands, rows, thr, L):
    # hash counts that are not a K1 tile size (padded families), one- to
    # 16-row bands, other shingle lengths and thresholds: every artifact equal
    corpus = _corpus_dir(ref, tmp_path, n=900, groups=90, seed=H + L)
    ws_ref, ws_gpu = str(tmp_path / "ref"), str(tmp_path / "gpu")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref, H=H, bands=bands, rows=rows, L=L, thr=thr, workers=2,
                  memory_budget=400_000)
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu, hash_count=H, bands=bands,
                             rows=rows, shingle_len=L, threshold=thr, workers=2,
                             memory_budget=400_000)
    pipeline.run_dedup(cfg, ctx=ctx)
    want, got = _tree(ws_ref), _tree(ws_gpu)
    assert sorted(got) == sorted(want)
    cs_ref, cs_gpu = (json.loads(x.pop("compare_stage.json")) for x in (want, got))
    cs_ref.pop("gather_peak_bytes")
    cs_gpu.pop("gather_peak_bytes")
    assert cs_gpu == cs_ref
    for k in want:
        assert got[k] == want[k], k


def test_run_bench_layout(ctx, ref, tmp_path):
    # run_bench (pipeline.cpp:587-613): sub-workspaces per worker count with
    # identical reports, bench.json rows in the reference's key order
    corpus = _corpus_dir(ref, tmp_path, n=400, groups=40, seed=31)
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=str(tmp_path / "b"))
    rows = pipeline.run_bench(cfg, [1, 3], ctx=ctx)
    assert [r.workers for r in rows] == [1, 3]
    b = json.load(open(os.path.join(cfg.workspace, "bench.json")))
    assert [list(r) for r in b] == [["workers", "hash_seconds", "compare_seconds",
                                     "union_seconds", "total_seconds"]] * 2
    t1, t3 = (_tree(os.path.join(cfg.workspace, f"bench_w{w}")) for w in (1, 3))
    for f in ("groups.jsonl", "removal.txt", "summary.json"):
        assert t1[f] == t3[f]


def test_fsync_files_workspace_byte_identical(ctx, ref, tmp_path, monkeypatch):
    # --fsync (RunConfig::fsync_files): every artifact the reference writes
    # through write_file_bytes(..., fsync) (pipeline.cpp:335,444,487,494,506;
    # SignatureFileWriter sigstore.cpp:117) is fsynced -- Python side files
    # counted here, C++ writers exercised -- and the bytes do not change
    corpus = _corpus_dir(ref, tmp_path)
    ws_ref, ws_gpu = str(tmp_path / "ref"), str(tmp_path / "gpu")
    os.makedirs(ws_ref)
    ref.run_dedup(corpus, ws_ref)
    synced = []
    real = os.fsync
    monkeypatch.setattr(os, "fsync", lambda fd: (synced.append(fd), real(fd))[1])
    cfg = pipeline.RunConfig(inputs=[corpus], workspace=ws_gpu, fsync_files=True)
    pipeline.run_dedup(cfg, ctx=ctx)
    assert len(synced) == 2  # run_manifest.json, compare_stage.json
    assert _tree(ws_gpu) == _tree(ws_ref)
