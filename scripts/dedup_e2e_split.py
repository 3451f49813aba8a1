"""Where does a slow host-e2e dedup run spend its time?  The steps of
pipeline.dedup_packed timed one by one (wall clock), GC frozen + disabled."""
import ctypes as C
import gc
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2501_01046_b200 import pipeline  # noqa: E402
from paper_2501_01046_b200._lib import u8p, u64p  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

docs = bench.DOCS
pinned = torch.empty(docs * bench.LEN_MAX, dtype=torch.uint8, pin_memory=True).numpy()
data, offs = bench.c2_corpus(docs, 1, data_out=pinned)
op = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
op[:] = offs
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s.cuda_stream)
cfg = pipeline.RunConfig()
params = cfg.to_params(2000)
for _ in range(2):
    pipeline.dedup_packed(data, op, cfg, bucket_count=2000, ctx=ctx, fetch="arrays")
gc.collect(); gc.freeze(); gc.disable()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    stats = pipeline.NdDedupStats()
    ctx.check(ctx.lib.nd_set_hbm_budget(ctx.h, cfg.hbm_budget))
    t1 = time.perf_counter()
    ctx.check(ctx.lib.nd_dedup(ctx.h, data.ctypes.data_as(u8p), op.ctypes.data_as(u64p), None, docs,
                               C.byref(params), C.byref(stats)))
    t2 = time.perf_counter()
    rep = pipeline._fetch_report(ctx, stats, lists=False)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(json.dumps({"run": i, "total": round((t4 - t0) * 1e3, 2), "budget": round((t1 - t0) * 1e3, 2),
                      "nd_dedup": round((t2 - t1) * 1e3, 2), "fetch": round((t3 - t2) * 1e3, 2),
                      "sync": round((t4 - t3) * 1e3, 2)}), flush=True)
