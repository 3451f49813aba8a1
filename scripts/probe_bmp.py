"""Codepoint units on BMP text (Cyrillic + CJK, every document has code
points >= 256, all < 2^16): K1j over 16-bit units (default) against K1w
(ND_K1J_U16=0), device-resident, decode (K0) included.
    python scripts/probe_bmp.py [docs] [units_per_doc]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2501_01046_b200 import minhash  # noqa: E402
from paper_2501_01046_b200.device import Context  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 700
rng = np.random.default_rng(3)
pool = np.array([c for c in range(0x430, 0x450)] + [c for c in range(0x4E00, 0x4F00)], np.uint32)
lens = rng.integers(m * 3 // 4, m * 5 // 4, size=n)
cps = pool[rng.integers(0, len(pool), size=int(lens.sum()))]
if os.environ.get("PROBE_MIX") == "1":  # every other document ASCII (byte K1j)
    doc_of = np.repeat(np.arange(n), lens)
    ascii_pool = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz ", np.uint8).astype(np.uint32)
    sel = doc_of % 2 == 0
    cps[sel] = ascii_pool[rng.integers(0, len(ascii_pool), size=int(sel.sum()))]
# UTF-8 of 2- and 3-byte code points, vectorised
nb = np.where(cps < 0x80, 1, np.where(cps < 0x800, 2, 3)).astype(np.uint64)
starts = np.zeros(len(cps) + 1, np.uint64)
starts[1:] = np.cumsum(nb)
buf = np.zeros(int(starts[-1]), np.uint8)
one, two, three = cps < 0x80, (cps >= 0x80) & (cps < 0x800), cps >= 0x800
buf[starts[:-1][one]] = cps[one]
s2, s3 = starts[:-1][two], starts[:-1][three]
c2, c3 = cps[two], cps[three]
buf[s2] = 0xC0 | (c2 >> 6)
buf[s2 + 1] = 0x80 | (c2 & 0x3F)
buf[s3] = 0xE0 | (c3 >> 12)
buf[s3 + 1] = 0x80 | ((c3 >> 6) & 0x3F)
buf[s3 + 2] = 0x80 | (c3 & 0x3F)
doc_cp = np.zeros(n + 1, np.int64)
doc_cp[1:] = np.cumsum(lens)
offs = starts[doc_cp].astype(np.uint64)
d_text = torch.from_numpy(buf).cuda()
d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
H = 128
hwe = float((lens - 4).sum() * H)
d_sig = torch.empty((n, H), dtype=torch.int32, device="cuda")
d_band = torch.empty((n, 16), dtype=torch.int32, device="cuda")
out = {}
# PROBE_SHAPES="name:VAR=v,VAR=v name2:..." (K1j-u16 tuning) instead of u16 on/off
shapes = [("u16", {"ND_K1J_U16": "1"}), ("k1w", {"ND_K1J_U16": "0"})]
if os.environ.get("PROBE_SHAPES"):
    shapes = [(sp.partition(":")[0], dict(x.split("=", 1) for x in sp.partition(":")[2].split(",") if x))
              for sp in os.environ["PROBE_SHAPES"].split()]
knobs = {k for _, e in shapes for k in e}
for variant, env in shapes * 2:
    for k in knobs:
        os.environ.pop(k, None)
    os.environ.update(env)
    ctx = Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    fam = minhash.derive_family(5, H, 5, minhash.ShingleUnit.CODEPOINT)
    ts = []
    for it in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        minhash.signatures_device(d_text.data_ptr(), d_offs.data_ptr(), n, fam, d_sig.data_ptr(),
                                  d_band.data_ptr(), 16, 8, 2000, ctx=ctx)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    chk = int(np.frombuffer(d_sig.cpu().numpy().tobytes(), np.uint64).sum() % (1 << 61))
    kern = ctx.lib.nd_k1_kernel(ctx.h).decode()
    out.setdefault(variant, []).append(ms)
    print(json.dumps({"variant": variant, "kernel": kern, "ms": round(ms, 3), "docs_per_s": n / ms * 1e3,
                      "T_hwe_s": hwe / ms / 1e9, "text_GB": len(buf) / 1e9, "checksum": chk}),
          flush=True)
    ctx.close()
