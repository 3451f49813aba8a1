"""K1 tuning harness: build libneardup_b200 variants that differ only in the
compile-time switches of csrc/k_signature.cu, then (on the GPU box) time K1 on
the bench's C2 shard for each, alternating variants so clock drift hits all.

    python scripts/k1_variants.py build NAME="-DFLAG=1 ..." [...]
    python scripts/k1_variants.py run [--reps 3]            (GPU)
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "variants")


def build(specs):
    from paper_2501_01046_b200 import build as b

    b.build()
    objs = open(os.path.join(b.OBJ, "current.txt")).read().split()
    others = [o for o in objs if "k_signature.cu" not in os.path.basename(o)]
    os.makedirs(OUT, exist_ok=True)
    for spec in specs:
        name, _, flags = spec.partition("=")
        obj = os.path.join(OUT, name + ".o")
        cmd = [b.NVCC] + b.COMMON + b.CUFLAGS + flags.split() + ["-c",
               os.path.join(b.CSRC, "k_signature.cu"), "-o", obj, "-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        spills = [l for l in r.stderr.splitlines() if "spill" in l and " 0 bytes spill stores" not in l]
        lib = os.path.join(OUT, f"lib_{name}.so")
        subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", lib, obj] + others + ["-lpthread"],
                       check=True)
        print(name, flags, "spilling kernels:", len(spills))


PROBE = r"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.environ['ROOT'])
import bench
from paper_2501_01046_b200 import minhash
from paper_2501_01046_b200.device import Context
data, offs = np.load('/tmp/k1v_data.npy', mmap_mode='r'), np.load('/tmp/k1v_offs.npy')
n = len(offs) - 1
ctx = Context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
fam = minhash.derive_family(5, 128, 5)
d = torch.from_numpy(np.ascontiguousarray(data)).cuda(); o = torch.from_numpy(offs.view(np.int64)).cuda()
sig = torch.empty((n, 128), dtype=torch.int32, device='cuda'); band = torch.empty((n, 16), dtype=torch.int32, device='cuda')
hwe = float((np.diff(offs).astype(np.float64) - 4).sum() * 128)
def run():
    minhash.signatures_device(d.data_ptr(), o.data_ptr(), n, fam, sig.data_ptr(), band.data_ptr(), 16, 8, 2000, ctx=ctx)
for _ in range(3): run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s); run(); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
h = int(np.frombuffer(sig.cpu().numpy().tobytes(), np.uint64).sum() % (1 << 61))
print(json.dumps({"ms": min(ts), "ms_med": sorted(ts)[5], "hwe_T": hwe / min(ts) / 1e9, "sum": h,
                  "kernel": ctx.lib.nd_k1_kernel(ctx.h).decode()}))
"""


def run(reps, envs=None):
    """envs: {"name": {"VAR": "value"}} variants by environment (in-tree library)
    instead of the built library variants."""
    import numpy as np

    import bench

    data, offs = bench.c2_corpus(bench.DOCS, 1)
    np.save("/tmp/k1v_data.npy", data)
    np.save("/tmp/k1v_offs.npy", offs)
    if envs:
        cases = {k: v for k, v in envs.items()}
    else:
        cases = {os.path.basename(l)[4:-3]: {"ND_LIB_PATH": l}
                 for l in sorted(glob.glob(os.path.join(OUT, "lib_*.so")))}
    res = {k: [] for k in cases}
    for _ in range(reps):
        for name, extra in cases.items():
            env = dict(os.environ, ROOT=ROOT, **extra)
            r = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
            res[name].append(json.loads(line) if line.startswith("{") else line)
    for k, v in res.items():
        good = [x for x in v if isinstance(x, dict)]
        sums = {x["sum"] for x in good}
        print(json.dumps({"variant": k, "best_ms": min(x["ms"] for x in good) if good else None,
                          "T_hwe_s": max(x["hwe_T"] for x in good) if good else None,
                          "all_ms": [x["ms"] if isinstance(x, dict) else x for x in v],
                          "checksums_agree": len(sums) == 1, "sum": sorted(sums),
                          "kernel": good[0].get("kernel") if good else None}))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
        envs = None
        if "--env" in sys.argv:  # --env name:VAR=val,VAR=val name2:...
            envs = {}
            for spec in sys.argv[sys.argv.index("--env") + 1:]:
                name, _, kv = spec.partition(":")
                envs[name] = dict(x.split("=", 1) for x in kv.split(",") if x)
        run(reps, envs)
