"""One in-memory dedup of the bench workload (C2: 1M docs, device-resident text),
for kernel-level profiling: python scripts/dedup_once.py [docs] [H] [K]
(K: bucket count override; e.g. 1M docs at K=365 gives C3's ~2740-document cells);
python scripts/dedup_once.py c3 [H] [K]: bench.py's C3 corpus, generated in HBM"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_01046_b200 import _lib, pipeline  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

c3 = len(sys.argv) > 1 and sys.argv[1] == "c3"  # bench.py's C3 corpus (30M lognormal docs)
n = 30_000_000 if c3 else int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 128
K = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lib = _lib.load()
if c3:
    import bench
    spec = bench.c3_spec(_lib, n)
else:
    spec = _lib.NdSynthSpec(doc_count=n, group_count=n // 20, group_size_min=2, group_size_max=2,
                            edit_num=1, edit_den=100, len_min=1600, len_max=2400, seed=1, mode=1)
offs = np.empty(n + 1, np.uint64)
nb = C.c_uint64()
_lib.check(lib.nd_synth_generate(C.byref(spec), None, offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
ctx = Context(0)
d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()),
                                   C.c_void_p(d_text.data_ptr())))
params = pipeline.RunConfig(hash_count=H, bands=H // 8, rows=8).to_params(K)
st = _lib.NdDedupStats()
for _ in range(2):
    ctx.check(lib.nd_dedup_device(ctx.h, C.c_void_p(d_text.data_ptr()), C.c_void_p(d_offs.data_ptr()),
                                  None, n, C.byref(params), C.byref(st)))
torch.cuda.synchronize()
print("docs", n, "distinct pairs", st.distinct_pairs, "groups", st.duplicate_groups,
      "seconds", list(st.seconds), "compare", lib.nd_dedup_compare_kind(ctx.h).decode())
