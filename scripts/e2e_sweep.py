"""Host-pipeline chunk sizing probe: C2 signatures e2e (nd_signatures) and C2
dedup e2e (nd_dedup) from pinned host memory, CUDA-event timed (GPU box)."""
import json, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2501_01046_b200 import minhash, pipeline
from paper_2501_01046_b200.device import Context
n = bench.DOCS
pinned = torch.empty(n * bench.LEN_MAX, dtype=torch.uint8, pin_memory=True).numpy()
data, offs = bench.c2_corpus(n, 1, data_out=pinned)
ctx = Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
fam = minhash.derive_family(5, 128, 5)
sig = torch.empty((n, 128), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
band = torch.empty((n, 16), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s); fn(); e1.record(s); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
a = t(lambda: minhash.signatures_packed(data, offs, fam, 16, 8, 2000, ctx=ctx, sig_out=sig, band_out=band))
b = t(lambda: pipeline.dedup_packed(data, offs, pipeline.RunConfig(), bucket_count=2000, ctx=ctx, fetch="arrays"))
print(json.dumps({"first_mb": os.environ.get("ND_H2D_FIRST_MB"), "max_mb": os.environ.get("ND_H2D_MAX_MB"),
                  "sig_e2e_ms": a, "sig_e2e_docs_s": n / a * 1e3, "dedup_e2e_ms": b}))
if os.environ.get("C3"):
    import ctypes as C
    from paper_2501_01046_b200 import _lib
    lib = _lib.load()
    docs = int(os.environ.get("C3"))
    spec = bench.c3_spec(_lib, docs)
    offs3 = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, offs3.ctypes.data_as(_lib.u64p), C.byref(nb)))
    d_offs = torch.from_numpy(offs3.view(np.int64)).cuda()
    d_text = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    ctx.check(lib.nd_synth_text_device(ctx.h, C.byref(spec), C.c_void_p(d_offs.data_ptr()), C.c_void_p(d_text.data_ptr())))
    host = torch.empty(nb.value, dtype=torch.uint8, pin_memory=True); host.copy_(d_text); torch.cuda.synchronize()
    del d_text; torch.cuda.empty_cache()
    h = host.numpy()
    c = t(lambda: pipeline.dedup_packed(h, offs3, pipeline.RunConfig(), ctx=ctx, fetch="arrays"), reps=2)
    print(json.dumps({"c3_docs": docs, "c3_e2e_ms": c, "c3_docs_s": docs / c * 1e3,
                      "streams": os.environ.get("ND_K1J_STREAMS")}))
