"""One K1 launch on the bench's C2 shard (for ncu): python scripts/k1_probe_once.py [docs]"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2501_01046_b200 import minhash
from paper_2501_01046_b200.device import Context
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
data, offs = bench.c2_corpus(n, 1)
ctx = Context(0)
fam = minhash.derive_family(5, 128, 5)
d = torch.from_numpy(data).cuda(); o = torch.from_numpy(offs.view(np.int64)).cuda()
sig = torch.empty((n, 128), dtype=torch.int32, device='cuda'); band = torch.empty((n, 16), dtype=torch.int32, device='cuda')
for _ in range(2):
    minhash.signatures_device(d.data_ptr(), o.data_ptr(), n, fam, sig.data_ptr(), band.data_ptr(), 16, 8, 2000, ctx=ctx)
torch.cuda.synchronize()
print("kernel", ctx.lib.nd_k1_kernel(ctx.h).decode())
