"""How much do chunk boundaries cost K1j?  The bench's C2 shard signed from
HBM in one launch vs in the chunk sizes the host pipeline uses (sequential
launches on one stream, no copies)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_01046_b200 import minhash  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

docs = bench.DOCS
data, offs = bench.c2_corpus(docs, 1)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s.cuda_stream)
fam = minhash.derive_family(5, 128, 5)
d = torch.from_numpy(data).cuda()
sig = torch.empty((docs, 128), dtype=torch.int32, device="cuda")
band = torch.empty((docs, 16), dtype=torch.int32, device="cuda")


def run(bounds):
    for a, b in zip(bounds[:-1], bounds[1:]):
        o = torch.from_numpy((offs[a:b + 1] - offs[a]).view(np.int64)).cuda()
        minhash.signatures_device(d.data_ptr() + int(offs[a]), o.data_ptr(), b - a, fam,
                                  sig.data_ptr() + a * 512, band.data_ptr() + a * 64, 16, 8, 2000,
                                  ctx=ctx)


def bounds_for(mbs):
    out, a = [0], 0
    i = 0
    while a < docs:
        cap = mbs[min(i, len(mbs) - 1)] << 20
        b = int(np.searchsorted(offs, offs[a] + cap, side="right")) - 1
        b = max(a + 1, min(b, docs))
        out.append(b)
        a = b
        i += 1
    return out


res = {}
for name, mbs in {"one": [1 << 20], "ramp64_512": [64, 128, 256, 512], "ramp32_512": [32, 64, 128, 256, 512],
                  "fixed512": [512], "fixed256": [256], "ramp64_1024": [64, 128, 256, 512, 1024]}.items():
    b = bounds_for(mbs)
    for _ in range(2):
        run(b)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        run(b)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[name] = {"chunks": len(b) - 1, "ms": round(min(ts), 2)}
print(json.dumps(res))
