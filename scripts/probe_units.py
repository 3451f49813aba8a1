"""K1 throughput, byte vs codepoint units (fq-cp and wide K1 variants), on the C2 shard (device-resident).
    python scripts/probe_units.py [docs]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_01046_b200 import _lib, minhash  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
lib = _lib.load()
spec = _lib.NdSynthSpec(doc_count=n, group_count=n // 20, group_size_min=2, group_size_max=2,
                        edit_num=1, edit_den=100, len_min=1600, len_max=2400, seed=1, mode=1)
nb = C.c_uint64()
offs = np.empty(n + 1, np.uint64)
_lib.check(lib.nd_synth_generate(C.byref(spec), None, offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
ctx = Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()),
                                   C.c_void_p(d_text.data_ptr())))
d_sig = torch.empty((n, 128), dtype=torch.int32, device="cuda")
d_band = torch.empty((n, 16), dtype=torch.int32, device="cuda")
hwe = float((np.diff(offs).astype(np.float64) - 4).sum() * 128)
import os  # noqa: E402

for unit, cp in ((minhash.ShingleUnit.BYTE, ""), (minhash.ShingleUnit.CODEPOINT, "fq"),
                 (minhash.ShingleUnit.CODEPOINT, "wide")):
    os.environ["ND_K1_CP"] = cp
    fam = minhash.derive_family(5, 128, 5, unit)
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        minhash.signatures_device(d_text.data_ptr(), d_offs.data_ptr(), n, fam, d_sig.data_ptr(),
                                  d_band.data_ptr(), 16, 8, 2000, ctx=ctx)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{unit.name:9s} {cp:4s} {ms:8.2f} ms  {n / ms / 1e3:6.2f} M docs/s  {hwe / ms / 1e9:.3f} T HWE/s")
