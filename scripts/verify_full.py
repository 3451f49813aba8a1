"""Full-scale parity: EVERY signature, band id, distinct duplicate pair and
duplicate group of a paper-scale run checked against the CPU side.

  1. corpus generated in HBM (nd_synth_text_device, the reference generator's
     conventions), full in-memory dedup on the GPU (nd_dedup_device);
  2. every document's signature + band ids recomputed by the REFERENCE ITSELF
     (oracle/_ref: signature_of_document + band_bucket_ids, all host cores),
     chunk by chunk from the same bytes, and compared with the GPU's;
  3. the cells rebuilt on the CPU from those band ids (oracle/verify.c:
     ov_cells), every candidate pair of every cell compared by the C oracle
     (compare_bucket with the reference oracle's exact early exit,
     ov_compare_cells), distinct pairs vs the GPU's (lo, hi, match_count);
  4. components by the oracle's union-find (or_components) vs the GPU's groups.

    python scripts/verify_full.py c3 [--docs N] [--out profiles/r1_c3_full_parity.json]
    python scripts/verify_full.py c4 --rows 0:16000000 --skip-pairs   (split runs)
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from oracle_bind import Ref, u32p, u64p  # noqa: E402
from run_configs import CONFIGS, spec_for  # noqa: E402

from paper_2501_01046_b200 import _lib, pipeline  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402


def log(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--docs", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=500_000)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=None)
    # split runs (one gpurun call is capped at an hour): verify signature rows
    # [a, b) only, and/or skip the pair + group stages
    ap.add_argument("--rows", default=None, help="a:b")
    ap.add_argument("--skip-pairs", action="store_true")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    docs = a.docs or cfg["docs"]
    H, B = cfg["H"], cfg["bands"]
    res = {"config": a.config, "docs": docs, "host_cores": os.cpu_count(), "threads": a.threads}
    lib = _lib.load()
    spec = spec_for(cfg, docs)
    offs = np.empty(docs + 1, np.uint64)
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, offs.ctypes.data_as(u64p), C.byref(nb)))
    ctx = Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()),
                                       C.c_void_p(d_text.data_ptr())))
    params = pipeline.RunConfig(hash_count=H, bands=B, rows=cfg["rows"]).to_params(cfg.get("K", 0))
    stats = _lib.NdDedupStats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.check(lib.nd_dedup_device(ctx.h, C.c_void_p(d_text.data_ptr()), C.c_void_p(d_offs.data_ptr()),
                                  None, docs, C.byref(params), C.byref(stats)))
    e1.record(stream)
    torch.cuda.synchronize()
    K = stats.bucket_count
    res.update(text_bytes=int(nb.value), gpu_dedup_ms=e0.elapsed_time(e1), bucket_count=K,
               candidate_pairs_gpu=stats.candidate_pairs, distinct_pairs_gpu=stats.distinct_pairs,
               groups_gpu=stats.duplicate_groups, near_duplicates_gpu=stats.near_duplicates)
    log(stage="gpu", **res)

    sig = np.empty((docs, H), np.uint32)
    band = np.empty((docs, B), np.uint32)
    ctx.check(lib.nd_dedup_fetch_signatures(ctx.h, sig.ctypes.data_as(u32p), band.ctypes.data_as(u32p)))
    d = stats.distinct_pairs
    plo, phi = np.empty(d, np.uint64), np.empty(d, np.uint64)
    pm = np.empty(d, np.uint32)
    ctx.check(lib.nd_dedup_fetch_pairs(ctx.h, plo.ctypes.data_as(u64p), phi.ctypes.data_as(u64p),
                                       pm.ctypes.data_as(u32p)))
    gmem = np.empty(stats.near_duplicates, np.uint64)
    gst = np.empty(stats.duplicate_groups + 1, np.uint64)
    ctx.check(lib.nd_dedup_fetch_groups(ctx.h, gmem.ctypes.data_as(u64p), gst.ctypes.data_as(u64p)))

    # ---- 2. every signature and band id by the reference itself ----------------
    ref = Ref()
    t = time.time()
    bad_sig = bad_band = 0
    first_bad = None
    r0, r1 = (int(x) for x in a.rows.split(":")) if a.rows else (0, docs)
    r1 = min(r1, docs)
    for c0 in range(r0, r1, a.chunk):
        c1 = min(r1, c0 + a.chunk)
        b0, b1 = int(offs[c0]), int(offs[c1])
        text = d_text[b0:b1].cpu().numpy()
        co = (offs[c0:c1 + 1] - offs[c0]).astype(np.uint64)
        rs, rb = ref.signatures(text, co, H=H, L=5, bands=B, rows=cfg["rows"], K=K,
                                workers=a.threads)
        ds = np.flatnonzero((rs != sig[c0:c1]).any(axis=1))
        db = np.flatnonzero((rb != band[c0:c1]).any(axis=1))
        bad_sig += len(ds)
        bad_band += len(db)
        if first_bad is None and (len(ds) or len(db)):
            first_bad = int(c0 + (ds[0] if len(ds) else db[0]))
        if ((c0 - r0) // a.chunk) % 10 == 0:
            log(stage="signatures", done=c1, bad_sig=bad_sig, bad_band=bad_band,
                seconds=time.time() - t)
    res.update(signatures_checked=r1 - r0, signature_rows=[r0, r1],
               signature_rows_differing=bad_sig,
               band_rows_differing=bad_band, first_bad_doc=first_bad,
               reference_signature_seconds=time.time() - t)
    log(stage="signatures_done", bad_sig=bad_sig, bad_band=bad_band,
        seconds=res["reference_signature_seconds"])

    if a.skip_pairs:
        res["bit_exact_rows"] = bool(bad_sig == 0 and bad_band == 0)
        log(stage="done", **res)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(res, f, indent=1)
        return

    # ---- 3./4. every candidate pair + groups (tests/scale_check.py) ------------
    import scale_check as sc

    pr = sc.check_pairs(sig, band, K, 4, 5, (plo, phi, pm), threads=a.threads)
    key = pr.pop("_keys")
    res.update(pr)
    log(stage="pairs", **pr)
    t = time.time()
    res.update(sc.check_groups(key, docs, (gmem, gst)), oracle_union_seconds=time.time() - t)
    res["bit_exact"] = bool(bad_sig == 0 and bad_band == 0 and res["pairs_identical"]
                            and res["groups_identical"]
                            and res["candidate_pairs_oracle"] == res["candidate_pairs_gpu"])
    log(stage="done", **res)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
