"""One traced nd_signatures call on the bench's C2 shard (ND_PIPE_TRACE=1:
per chunk device times of copy in / kernel / copy out on stderr)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_01046_b200 import minhash  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

docs = bench.DOCS
pinned = torch.empty(docs * bench.LEN_MAX, dtype=torch.uint8, pin_memory=True).numpy()
data, offs = bench.c2_corpus(docs, 1, data_out=pinned)
op = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
op[:] = offs
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx = Context(0, stream=s.cuda_stream)
fam = minhash.derive_family(5, 128, 5)
sig = torch.empty((docs, 128), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
band = torch.empty((docs, 16), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
for i in range(4):
    if i == 3:
        os.environ["ND_PIPE_TRACE"] = "1"
        print("traced call:", file=sys.stderr, flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    minhash.signatures_packed(data, op, fam, 16, 8, 2000, ctx=ctx, sig_out=sig, band_out=band)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"call {i}: {e0.elapsed_time(e1):.2f} ms", file=sys.stderr, flush=True)
