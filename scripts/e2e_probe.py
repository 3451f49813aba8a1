"""Host-pipeline tuning: nd_signatures (pinned host text -> pinned host
signatures + band ids) on the bench's C2 shard, best of N, for environment
variants run in alternating subprocesses:
    python scripts/e2e_probe.py --env s2:ND_H2D_SLOTS=2 s3:ND_H2D_SLOTS=3,ND_H2D_FIRST_MB=32
(PROBE_MODE=dedup: pipeline.dedup_packed -> nd_dedup instead)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import gc, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.environ['ROOT'])
import bench
from paper_2501_01046_b200 import minhash
from paper_2501_01046_b200.device import Context
docs = bench.DOCS
pinned = torch.empty(docs * bench.LEN_MAX, dtype=torch.uint8, pin_memory=True).numpy()
data, offs = bench.c2_corpus(docs, 1, data_out=pinned)
op = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
op[:] = offs
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = Context(0, stream=s.cuda_stream)
fam = minhash.derive_family(5, 128, 5)
sig = torch.empty((docs, 128), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
band = torch.empty((docs, 16), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
from paper_2501_01046_b200 import pipeline
cfg = pipeline.RunConfig()
dedup = os.environ.get("PROBE_MODE") == "dedup"
def run():
    if dedup:
        r = pipeline.dedup_packed(data, op, cfg, bucket_count=2000, ctx=ctx, fetch="arrays")
        sig[0, 0] = r.distinct_pairs
    else:
        minhash.signatures_packed(data, op, fam, 16, 8, 2000, ctx=ctx, sig_out=sig, band_out=band)
for _ in range(3): run()
torch.cuda.synchronize()
gc.collect(); gc.freeze(); gc.disable()  # as bench.py
ts = []
for _ in range(8):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s); run(); e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
h = int(np.frombuffer(sig.tobytes(), np.uint64).sum() % (1 << 61))
print(json.dumps({"ms": min(ts), "ms_med": sorted(ts)[4], "ms_mean": sum(ts) / len(ts),
                  "ms_max": max(ts), "sum": h}))
"""


def main():
    envs = {}
    args = sys.argv[sys.argv.index("--env") + 1:]
    for spec in args:
        name, _, kv = spec.partition(":")
        envs[name] = dict(x.split("=", 1) for x in kv.split(",") if x)
    reps = int(os.environ.get("PROBE_REPS", "2"))
    res = {k: [] for k in envs}
    for _ in range(reps):
        for name, extra in envs.items():
            env = dict(os.environ, ROOT=ROOT, **extra)
            r = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
            res[name].append(json.loads(line) if line.startswith("{") else line)
    for k, v in res.items():
        good = [x for x in v if isinstance(x, dict)]
        print(json.dumps({"variant": k, "env": envs[k], "best_ms": min(x["ms"] for x in good) if good else None,
                          "mean_ms": [round(x["ms_mean"], 2) for x in good],
                          "max_ms": [round(x["ms_max"], 2) for x in good],
                          "all": [x["ms"] if isinstance(x, dict) else x for x in v],
                          "sums": sorted({x["sum"] for x in good})}))


if __name__ == "__main__":
    main()
