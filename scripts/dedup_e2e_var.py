"""Run-to-run variance of nd_dedup from pinned host memory on the bench's C2
shard: per run the wall time, the CUDA-event time and the library's stage
seconds (K1, K2, K3, K4a, K4, d2h)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2501_01046_b200 import pipeline  # noqa: E402
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
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 15
if len(sys.argv) > 2 and sys.argv[2] == "nogc":
    import gc
    gc.collect()
    gc.freeze()
    gc.disable()
for i in range(runs):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0.record(s)
    r = pipeline.dedup_packed(data, op, cfg, bucket_count=2000, ctx=ctx, fetch="arrays")
    t_ret = (time.perf_counter() - t) * 1e3
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3
    secs = r.stats.get("seconds") if isinstance(getattr(r, "stats", None), dict) else None
    print(json.dumps({"run": i, "wall_ms": round(wall, 2), "returned_ms": round(t_ret, 2), "event_ms": round(e0.elapsed_time(e1), 2),
                      "stage_ms": [round(x * 1e3, 2) for x in secs] if secs else None}), flush=True)
