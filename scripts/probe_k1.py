"""Quick K1 throughput probe (device-resident input): HWE/s and docs/s."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_01046_b200 import _lib, minhash
from paper_2501_01046_b200.device import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
H = int(sys.argv[2]) if len(sys.argv) > 2 else 128
lib = _lib.load()
spec = _lib.NdSynthSpec(doc_count=n, group_count=n // 20, group_size_min=2, group_size_max=2,
                        edit_num=1, edit_den=100, len_min=1600, len_max=2400, seed=1, mode=1)
nb = C.c_uint64()
t0 = time.time()
_lib.check(lib.nd_synth_generate(C.byref(spec), None, None, C.byref(nb)))
data = np.empty(nb.value, np.uint8)
offs = np.empty(n + 1, np.uint64)
_lib.check(lib.nd_synth_generate(C.byref(spec), data.ctypes.data_as(_lib.u8p),
                                 offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
print(f"gen {n} docs {nb.value/1e9:.2f} GB in {time.time()-t0:.1f}s", flush=True)
ctx = Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
fam = minhash.derive_family(5, H, 5)
d_data = torch.from_numpy(data).cuda()
d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
bands = H // 8
d_sig = torch.empty((n, H), dtype=torch.int32, device="cuda")
d_band = torch.empty((n, bands), dtype=torch.int32, device="cuda")
hwe = float((np.diff(offs).astype(np.float64) - 4).sum() * H)
for it in range(5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    minhash.signatures_device(d_data.data_ptr(), d_offs.data_ptr(), n, fam, d_sig.data_ptr(),
                              d_band.data_ptr(), bands, 8, 2000, ctx=ctx)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"iter {it}: {ms:.2f} ms  {n/ms*1e3/1e6:.2f} M docs/s  {hwe/ms*1e3/1e12:.3f} T HWE/s", flush=True)
# host pipeline (e2e)
pin_d = torch.from_numpy(data).pin_memory().numpy()
pin_o = torch.from_numpy(offs.view(np.int64)).pin_memory().numpy().view(np.uint64)
sig_h = torch.empty((n, H), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
band_h = torch.empty((n, bands), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    minhash.signatures_packed(pin_d, pin_o, fam, bands, 8, 2000, ctx=ctx, sig_out=sig_h, band_out=band_h)
    dt = time.perf_counter() - t
    print(f"host e2e {it}: {dt*1e3:.1f} ms {n/dt/1e6:.2f} M docs/s", flush=True)
ok = np.array_equal(sig_h, d_sig.cpu().numpy().view(np.uint32)) and np.array_equal(band_h, d_band.cpu().numpy().view(np.uint32))
print("host==device:", ok)
