"""Paper-scale configurations (BASELINE.json configs C3/C4/C5) on one B200.

The corpus is generated directly in HBM (nd_synth_text_device, mode 1 --
identical bytes to the host generator), then the in-memory dedup runs on
device-resident text (nd_dedup_device).  Parity evidence at this scale:
  * signatures + band ids of a random sample of documents vs the CPU oracle
    (oracle/oracle.c) on the same bytes;
  * exact match counts of a random sample of the emitted pairs, recomputed by
    the oracle from the documents' text;
  * (--ref-docs N) a full reference run_dedup on the first N documents vs
    nd_dedup on the same N documents (byte-identical report files).

    python scripts/run_configs.py c5 [--docs 2000000] [--ref-docs 100000]
"""
import argparse
import ctypes as C
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2501_01046_b200 import _lib, pipeline  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

CONFIGS = {
    # lognormal, mean ~3.3 KB (median 2.2 KB, sigma 0.9), clipped [200 B, 100 KB],
    # 10% of docs in near-dup groups of 2-5 at edit rate 1/100
    "c3": dict(docs=30_000_000, H=128, bands=16, rows=8, len_min=2200, len_max=100_000,
               sigma=900, group_frac=0.10, gmin=2, gmax=5),
    "c4": dict(docs=30_000_000, H=256, bands=32, rows=8, len_min=2200, len_max=100_000,
               sigma=900, group_frac=0.10, gmin=2, gmax=5),
    # the bench.py workload (BASELINE configs[1]): 1M docs, uniform 1600-2400 B, 10% in
    # near-duplicate pairs -- same generator spec as bench.py
    "c2": dict(docs=1_000_000, H=128, bands=16, rows=8, len_min=1600, len_max=2400,
               sigma=0, group_frac=0.10, gmin=2, gmax=2, law=0, seed=1, K=2000),
    # long-document skew: 2M docs, lognormal median 2 KB up to 200 KB, 30% in clusters of 2-20
    "c5": dict(docs=2_000_000, H=128, bands=16, rows=8, len_min=2000, len_max=200_000,
               sigma=1200, group_frac=0.30, gmin=2, gmax=20),
}


def spec_for(cfg, docs):
    mean_group = (cfg["gmin"] + cfg["gmax"]) / 2
    return _lib.NdSynthSpec(doc_count=docs, group_count=int(docs * cfg["group_frac"] / mean_group),
                            group_size_min=cfg["gmin"], group_size_max=cfg["gmax"], edit_num=1,
                            edit_den=100, len_min=cfg["len_min"], len_max=cfg["len_max"],
                            seed=cfg.get("seed", 3), mode=1, len_law=cfg.get("law", 1),
                            sigma_milli=cfg["sigma"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--docs", type=int, default=None)
    ap.add_argument("--sample", type=int, default=2000)
    ap.add_argument("--ref-docs", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    docs = a.docs or cfg["docs"]
    lib = _lib.load()
    spec = spec_for(cfg, docs)
    t0 = time.time()
    offs = np.empty(docs + 1, np.uint64)
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
    t_len = time.time() - t0
    ctx = Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()),
                                       C.c_void_p(d_text.data_ptr())))
    torch.cuda.synchronize()
    t_gen = time.time() - t0
    rc = pipeline.RunConfig(hash_count=cfg["H"], bands=cfg["bands"], rows=cfg["rows"])
    params = rc.to_params(cfg.get("K", 0))
    stats = _lib.NdDedupStats()
    runs = []
    for it in range(2):  # warm-up + timed
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.check(lib.nd_dedup_device(ctx.h, C.c_void_p(d_text.data_ptr()), C.c_void_p(d_offs.data_ptr()),
                                      None, docs, C.byref(params), C.byref(stats)))
        e1.record(stream)
        torch.cuda.synchronize()
        runs.append(e0.elapsed_time(e1))
    ms = runs[-1]
    lens = np.diff(offs)
    res = {"config": a.config, "docs": docs, "text_bytes": int(nb.value),
           "mean_len": float(lens.mean()), "max_len": int(lens.max()),
           "dedup_ms": ms, "docs_per_s": docs / (ms / 1e3),
           "hwe": float(((lens - 4).astype(np.float64) * cfg["H"]).sum()),
           "stage_seconds": list(stats.seconds), "bucket_count": stats.bucket_count,
           "cells": stats.nonsingleton_cells, "candidate_pairs": stats.candidate_pairs,
           "emitted_pairs": stats.emitted_pairs, "distinct_pairs": stats.distinct_pairs,
           "groups": stats.duplicate_groups, "near_duplicates": stats.near_duplicates,
           "host_lengths_s": t_len, "device_text_s": t_gen - t_len,
           "compare": lib.nd_dedup_compare_kind(ctx.h).decode()}
    res["k1_hwe_per_s"] = res["hwe"] / stats.seconds[0] if stats.seconds[0] else None
    res["candidate_pairs_per_s"] = stats.candidate_pairs / stats.seconds[2] if stats.seconds[2] else None
    print(json.dumps(res), flush=True)

    # ---- parity spot checks -------------------------------------------------------
    from oracle_bind import Oracle

    o = Oracle()
    fam = o.derive_family(5, cfg["H"])
    rng = np.random.default_rng(1)
    sample = np.sort(rng.choice(docs, size=min(a.sample, docs), replace=False))
    text = d_text  # device
    sig_rows = []
    texts = []
    for d in sample:
        b, e = int(offs[d]), int(offs[d + 1])
        texts.append(text[b:e].cpu().numpy())
    so = np.zeros(len(texts) + 1, np.uint64)
    so[1:] = np.cumsum([len(t) for t in texts])
    want = o.signatures(np.concatenate(texts), so, fam)
    # GPU signatures of the sample: rerun K1 on the sample (device entry point)
    from paper_2501_01046_b200 import minhash

    gfam = minhash.derive_family(5, cfg["H"], 5)
    got, _ = minhash.signatures_packed(np.concatenate(texts), so, gfam, ctx=ctx, want_bands=False)
    res["sample_signatures_equal"] = bool(np.array_equal(got, want))
    # pairs: exact recount of a sample of emitted pairs from text
    pairs = pipeline.dedup_pairs(stats.distinct_pairs, ctx=ctx)
    k = min(2000, len(pairs))
    pick = rng.choice(len(pairs), size=k, replace=False) if k else []
    bad = 0
    mm = int(lib.nd_min_matches(cfg["H"], 4, 5))
    for i in pick:
        p = pairs[int(i)]
        ts = [text[int(offs[d]):int(offs[d + 1])].cpu().numpy() for d in (p.lo, p.hi)]
        po = np.array([0, len(ts[0]), len(ts[0]) + len(ts[1])], np.uint64)
        s2 = o.signatures(np.concatenate(ts), po, fam)
        m = int((s2[0] == s2[1]).sum())
        bad += int(m != p.match_count or m < mm)
    res["sample_pairs_checked"] = int(k)
    res["sample_pairs_bad"] = int(bad)
    print(json.dumps({"parity": {k2: res[k2] for k2 in ("sample_signatures_equal", "sample_pairs_checked",
                                                        "sample_pairs_bad")}}), flush=True)

    if a.ref_docs:
        from oracle_bind import Ref

        ref = Ref()
        n = min(a.ref_docs, docs)
        sub = text[:int(offs[n])].cpu().numpy()
        sub_offs = offs[:n + 1].copy()
        with tempfile.TemporaryDirectory() as tmp:
            corpus = os.path.join(tmp, "c.jsonl")
            with open(corpus, "w") as f:
                for i in range(n):
                    f.write('{"text":"' + bytes(sub[int(sub_offs[i]):int(sub_offs[i + 1])]).decode() + '"}\n')
            wr, wg = os.path.join(tmp, "r"), os.path.join(tmp, "g")
            os.makedirs(wr)
            t = time.time()
            ref.run_dedup(corpus, wr, H=cfg["H"], bands=cfg["bands"], rows=cfg["rows"],
                          workers=os.cpu_count(), memory_budget=64 << 30)
            t_ref = time.time() - t
            rep = pipeline.run_dedup(pipeline.RunConfig(inputs=[corpus], workspace=wg, hash_count=cfg["H"],
                                                        bands=cfg["bands"], rows=cfg["rows"]), ctx=ctx)
            same = all(open(os.path.join(wr, f), "rb").read() == open(os.path.join(wg, f), "rb").read()
                       for f in ("groups.jsonl", "removal.txt", "summary.json"))
            stage = json.load(open(os.path.join(wr, "compare_stage.json")))
            res["ref_subset"] = {"docs": n, "report_files_identical": same,
                                 "candidate_pairs_ref": stage["candidate_pairs"],
                                 "candidate_pairs_gpu": rep.candidate_pairs,
                                 "reference_seconds": t_ref, "host_cores": os.cpu_count(),
                                 "groups": len(rep.groups)}
        print(json.dumps({"ref_subset": res["ref_subset"]}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
