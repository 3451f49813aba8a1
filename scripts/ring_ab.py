"""A/B of nd_dedup's host ring (h2d_signatures) in one process: the chunk
gate on/off (ND_K1J_RING_GATE) and one vs three K1j streams, on the C2 shard
and on C3 (30M documents, 99 GB of pinned host text), alternating variants.
    python scripts/ring_ab.py [c2|c3]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_01046_b200 import _lib, pipeline  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s.cuda_stream)
lib = _lib.load()
import ctypes as C  # noqa: E402

if which == "c2":
    docs = bench.DOCS
    pinned = torch.empty(docs * bench.LEN_MAX, dtype=torch.uint8, pin_memory=True).numpy()
    data, offs = bench.c2_corpus(docs, 1, data_out=pinned)
    op = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    op[:] = offs
    K, reps = 2000, 5
else:
    docs = 30_000_000
    spec = bench.c3_spec(_lib, docs)
    op = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, op.ctypes.data_as(_lib.u64p), C.byref(nb)))
    d_offs = torch.from_numpy(op.view(np.int64)).cuda()
    d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()),
                                       C.c_void_p(d_text.data_ptr())))
    host = torch.empty(nb.value, dtype=torch.uint8, pin_memory=True)
    host.copy_(d_text)
    torch.cuda.synchronize()
    del d_text, d_offs
    torch.cuda.empty_cache()
    data = host.numpy()
    K, reps = 0, 2
variants = {"gate3": {"ND_K1J_RING_GATE": "1"}, "nogate3": {}, "one": {"ND_K1J_STREAMS": "1"}}
cfg = pipeline.RunConfig()
res = {k: [] for k in variants}
for rnd in range(reps):
    for name, env in variants.items():
        for k in ("ND_K1J_RING_GATE", "ND_K1J_STREAMS"):
            os.environ.pop(k, None)
        os.environ.update(env)
        if rnd == 0:
            pipeline.dedup_packed(data, op, cfg, bucket_count=K, ctx=ctx, fetch=None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        r = pipeline.dedup_packed(data, op, cfg, bucket_count=K, ctx=ctx, fetch=None)
        e1.record(s)
        torch.cuda.synchronize()
        res[name].append((round(e0.elapsed_time(e1), 2), r.distinct_pairs))
print(json.dumps({"workload": which, "ms": res}))
