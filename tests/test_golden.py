"""Committed golden fixtures (tests/golden/, generated from the reference
itself by scripts/make_golden.py): known answers for the oracle and the host
library (CPU), and a whole reference workspace the GPU pipeline must
reproduce byte for byte (-m gpu).  These need neither /root/reference nor the
oracle/_ref build."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle_bind import HashFn
from paper_2501_01046_b200 import lsh, minhash, pipeline
from paper_2501_01046_b200.compare import SimilarityThreshold

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KAT = json.load(open(os.path.join(GOLD, "kat.json")))
FOX = b"the quick brown fox jumps over the lazy dog"


def _fns(fam):
    fns = (HashFn * len(fam["modulus"]))()
    for i in range(len(fns)):
        p, q = fam["modulus"][i], fam["base"][i]
        fns[i].modulus, fns[i].base = p, q
        fns[i].base_inverse, fns[i].base_power = fam["base_inverse"][i], fam["base_power"][i]
        fns[i].reduce_factor = (1 << 64) // p
    return fns


@pytest.mark.parametrize("H", [128, 256])
def test_oracle_and_host_library_vs_golden(oracle, H):
    fam = KAT[f"family_seed5_H{H}"]
    got = minhash.derive_family(5, H, 5)
    assert [f.modulus for f in got.functions] == fam["modulus"]
    assert [f.base for f in got.functions] == fam["base"]
    assert [f.base_inverse for f in got.functions] == fam["base_inverse"]
    assert [f.base_power for f in got.functions] == fam["base_power"]
    data = np.frombuffer(FOX, np.uint8).copy()
    offs = np.array([0, len(FOX)], np.uint64)
    fns = _fns(fam)
    sig = oracle.signatures(data, offs, fns)
    for K in (200, 10955):
        want = KAT[f"fox_H{H}_K{K}"]
        assert sig[0].tolist() == want["signature"]
        assert oracle.band_ids(sig, H // 8, 8, K)[0].tolist() == want["bands"]
    assert oracle.signatures(data, offs, fns, unit=1)[0].tolist() == \
        KAT[f"fox_H{H}_codepoint"]["signature"]


def test_bucket_counts_and_min_matches_vs_golden(oracle):
    for n, K in KAT["bucket_count"].items():
        assert lsh.choose_bucket_count(int(n)) == K
        assert oracle.lib.or_choose_bucket_count(int(n), 2, 1) == K
    for key, mm in KAT["min_matches"].items():
        H, a, b = map(int, key.split("_"))
        assert SimilarityThreshold((a, b)).min_matches(H) == mm
        assert oracle.lib.or_min_matches(H, a, b) == mm


@pytest.mark.gpu
@pytest.mark.parametrize("H", [128, 256])
def test_gpu_signatures_vs_golden(ctx, H):
    data = np.frombuffer(FOX, np.uint8).copy()
    offs = np.array([0, len(FOX)], np.uint64)
    for K in (200, 10955):
        sig, band = minhash.signatures_packed(data, offs, minhash.derive_family(5, H, 5), H // 8, 8,
                                              K, ctx=ctx)
        assert sig[0].tolist() == KAT[f"fox_H{H}_K{K}"]["signature"]
        assert band[0].tolist() == KAT[f"fox_H{H}_K{K}"]["bands"]
    fam = minhash.derive_family(5, H, 5, minhash.ShingleUnit.CODEPOINT)
    sig, _ = minhash.signatures_packed(data, offs, fam, ctx=ctx, want_bands=False)
    assert sig[0].tolist() == KAT[f"fox_H{H}_codepoint"]["signature"]


@pytest.mark.gpu
def test_gpu_workspace_vs_golden(ctx, tmp_path):
    # the reference's run_dedup on corpus_s3.jsonl (2 workers, 200 kB gather
    # budget -> 20 passes): report files, .feds and .pairs digests
    d = json.load(open(os.path.join(GOLD, "ws_s3", "digests.json")))
    cfg = pipeline.RunConfig(inputs=[os.path.join(GOLD, "corpus_s3.jsonl")],
                             workspace=str(tmp_path / "ws"), workers=d["run"]["workers"],
                             memory_budget=d["run"]["memory_budget"])
    pipeline.run_dedup(cfg, ctx=ctx)
    ws = cfg.workspace
    for f in ("groups.jsonl", "removal.txt", "summary.json", "rejects.jsonl"):
        assert open(os.path.join(ws, f), "rb").read() == \
            open(os.path.join(GOLD, "ws_s3", f), "rb").read(), f
    sha = lambda p: hashlib.sha256(open(p, "rb").read()).hexdigest()  # noqa: E731
    assert {f: sha(os.path.join(ws, "signatures", f))
            for f in sorted(os.listdir(os.path.join(ws, "signatures")))} == d["feds"]
    assert {f: sha(os.path.join(ws, "pairs", f))
            for f in sorted(os.listdir(os.path.join(ws, "pairs")))} == d["pairs"]
    stage = json.load(open(os.path.join(ws, "compare_stage.json")))
    stage.pop("gather_peak_bytes")
    assert stage == d["compare_stage"]
