"""Regenerates tests/golden/ from the reference itself (oracle/_ref, the
reference's own sources compiled in place).  Run here, where /root/reference
exists; the fixtures are committed so that the parity tests do not need the
reference build.

    python scripts/make_golden.py
"""
import hashlib
import json
import os
import shutil
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_bind import Ref, family_array  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
FOX = b"the quick brown fox jumps over the lazy dog"


def sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def main():
    os.makedirs(GOLD, exist_ok=True)
    ref = Ref()
    kat = {"source": "oracle/_ref (reference sources) via scripts/make_golden.py"}
    for H in (128, 256):
        fam = family_array(ref.derive_family(5, H, 5))
        kat[f"family_seed5_H{H}"] = {"modulus": fam[:, 0].tolist(), "base": fam[:, 1].tolist(),
                                     "base_inverse": fam[:, 2].tolist(),
                                     "base_power": fam[:, 3].tolist()}
        data = np.frombuffer(FOX, np.uint8).copy()
        offs = np.array([0, len(FOX)], np.uint64)
        for K in (200, 10955):
            sig, band = ref.signatures(data, offs, H=H, bands=H // 8, rows=8, K=K)
            kat[f"fox_H{H}_K{K}"] = {"signature": sig[0].tolist(), "bands": band[0].tolist()}
        sig, _ = ref.signatures(data, offs, H=H, bands=0, rows=0, K=0, unit=1)
        kat[f"fox_H{H}_codepoint"] = {"signature": sig[0].tolist()}
    kat["bucket_count"] = {str(n): int(ref.lib.ref_choose_bucket_count(n, 2, 1))
                           for n in (1, 4, 10000, 1000000, 2000000, 30000000)}
    kat["min_matches"] = {f"{H}_{a}_{b}": int(ref.lib.ref_min_matches(H, a, b))
                          for H in (128, 256) for a, b in ((4, 5), (1, 2), (9, 10), (0, 1), (1, 1))}
    with open(os.path.join(GOLD, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    # a small planted corpus and the reference's whole workspace for it
    tmp = tempfile.mkdtemp()
    try:
        corpus = os.path.join(GOLD, "corpus_s3.jsonl")
        ref.generate_synthetic(1500, 120, gmin=2, gmax=4, edit=(2, 100), len_min=250, len_max=600,
                               seed=3, corpus_path=corpus, truth_path=os.path.join(tmp, "t.jsonl"))
        ws = os.path.join(tmp, "ws")
        os.makedirs(ws)
        ref.run_dedup(corpus, ws, workers=2, memory_budget=200_000)
        out = os.path.join(GOLD, "ws_s3")
        shutil.rmtree(out, ignore_errors=True)
        os.makedirs(out)
        for f in ("groups.jsonl", "removal.txt", "summary.json", "rejects.jsonl"):
            shutil.copy(os.path.join(ws, f), out)
        stage = json.load(open(os.path.join(ws, "compare_stage.json")))
        digests = {"compare_stage": {k: v for k, v in stage.items() if k != "gather_peak_bytes"},
                   "feds": {f: sha(os.path.join(ws, "signatures", f))
                            for f in sorted(os.listdir(os.path.join(ws, "signatures")))},
                   "pairs": {f: sha(os.path.join(ws, "pairs", f))
                             for f in sorted(os.listdir(os.path.join(ws, "pairs")))},
                   "run": {"workers": 2, "memory_budget": 200_000}}
        with open(os.path.join(out, "digests.json"), "w") as f:
            json.dump(digests, f, indent=1)
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    print("wrote", GOLD)


if __name__ == "__main__":
    main()
