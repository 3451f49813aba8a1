"""Parity at the bench's shape and at paper scale, driver-run (-m gpu).

  * C2 (BASELINE configs[1]): the exact 1M-document shard bench.py times
    (bench.c2_corpus(1M, seed 1), H=128, 16x8 bands, K=2000): EVERY signature
    and band id vs the reference itself (oracle/_ref, all host cores), the
    device entry point bench.py times (nd_signatures_device) vs the dedup's
    K1, then cells, every candidate pair (C oracle) and groups.
  * C3 (BASELINE configs[2]): 30M lognormal documents (98.9 GB of text)
    generated in HBM exactly as bench.py's dedup_c3 leg does; every 30th
    signature row + band ids vs the reference itself, and from the GPU's band
    ids every one of the ~6.6e11 candidate pairs compared by the C oracle
    (threaded) and the union-find groups.  Anchor: the reference's
    candidate_pairs counter (pipeline.cpp:406-411).
"""
import ctypes as C
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(torch):
    from paper_2501_01046_b200 import _lib
    from paper_2501_01046_b200.device import Context

    ctx = Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    return ctx, _lib.load(), _lib


def test_c2_bench_shard_bit_exact():
    import torch

    import bench
    import scale_check as sc
    from paper_2501_01046_b200 import minhash, pipeline

    ctx, lib, _lib = _setup(torch)
    docs = bench.DOCS
    data, offs = bench.c2_corpus(docs, 1)  # rank 0's shard, as bench.py builds it
    d_text = torch.from_numpy(data).cuda()
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    params = pipeline.RunConfig().to_params(bench.K_C2)
    stats, sig, band, pairs, groups = sc.gpu_dedup_device(ctx, lib, _lib, d_text, d_offs, docs,
                                                          params, bench.H, bench.BANDS)
    assert stats.bucket_count == bench.K_C2
    # the bench's timed entry point (value) computes the same rows
    fam = minhash.derive_family(5, bench.H, bench.L)
    d_sig = torch.empty((docs, bench.H), dtype=torch.int32, device="cuda")
    d_band = torch.empty((docs, bench.BANDS), dtype=torch.int32, device="cuda")
    minhash.signatures_device(d_text.data_ptr(), d_offs.data_ptr(), docs, fam, d_sig.data_ptr(),
                              d_band.data_ptr(), bench.BANDS, bench.ROWS, bench.K_C2, ctx=ctx)
    torch.cuda.synchronize()
    assert np.array_equal(d_sig.cpu().numpy().view(np.uint32), sig)
    assert np.array_equal(d_band.cpu().numpy().view(np.uint32), band)
    del d_sig, d_band, d_text, d_offs
    t = time.time()
    checked, bad_sig, bad_band = sc.check_signatures(
        lambda c0, c1: data[int(offs[c0]):int(offs[c1])], offs, sig, band, bench.H, bench.BANDS,
        bench.ROWS, bench.K_C2)
    print(f"C2: {checked} rows vs the reference in {time.time() - t:.0f} s")
    assert checked == docs and bad_sig == 0 and bad_band == 0
    res = sc.check_pairs(sig, band, bench.K_C2, 4, 5, pairs)
    print({k: v for k, v in res.items() if not k.startswith("_")})
    assert res["candidate_pairs_oracle"] == stats.candidate_pairs
    assert res["pairs_identical"] and res["distinct_pairs_oracle"] == stats.distinct_pairs
    g = sc.check_groups(res["_keys"], docs, groups)
    assert g["groups_identical"] and g["groups_oracle"] == stats.duplicate_groups
    assert stats.duplicate_groups > 40_000  # the planted pairs are found
    ctx.close()


def test_c3_paper_scale_parity():
    import torch

    import bench
    import scale_check as sc
    from paper_2501_01046_b200 import pipeline

    ctx, lib, _lib = _setup(torch)
    docs = int(os.environ.get("ND_C3_DOCS", bench.C3["docs"]))
    free, _ = torch.cuda.mem_get_info()
    spec = bench.c3_spec(_lib, docs)
    offs = np.empty(docs + 1, np.uint64)
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, offs.ctypes.data_as(_lib.u64p),
                                     C.byref(nb)))
    assert nb.value + docs * 700 < free, "C3 needs ~120 GB of HBM"
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()),
                                       C.c_void_p(d_text.data_ptr())))
    params = pipeline.RunConfig().to_params(0)
    stats, sig, band, pairs, groups = sc.gpu_dedup_device(ctx, lib, _lib, d_text, d_offs, docs,
                                                          params, bench.H, bench.BANDS)
    K = stats.bucket_count
    if docs == 30_000_000:
        assert K == 10955
    t = time.time()
    checked, bad_sig, bad_band = sc.check_signatures(
        lambda c0, c1: d_text[int(offs[c0]):int(offs[c1])].cpu().numpy(), offs, sig, band,
        bench.H, bench.BANDS, bench.ROWS, K, stride=30)
    print(f"C3: {checked} sampled rows vs the reference in {time.time() - t:.0f} s")
    assert checked >= docs // 30 and bad_sig == 0 and bad_band == 0
    del d_text, d_offs
    torch.cuda.empty_cache()
    res = sc.check_pairs(sig, band, K, 4, 5, pairs)
    print({k: v for k, v in res.items() if not k.startswith("_")})
    assert res["candidate_pairs_oracle"] == stats.candidate_pairs
    assert res["pairs_identical"] and res["distinct_pairs_oracle"] == stats.distinct_pairs
    g = sc.check_groups(res["_keys"], docs, groups)
    assert g["groups_identical"] and g["groups_oracle"] == stats.duplicate_groups
    ctx.close()
