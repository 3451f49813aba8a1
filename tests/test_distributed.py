"""Multi-rank dedup protocol under gloo (CPU, world sizes 1/2/3): GPU-count
invariance -- identical groups, distinct pairs and candidate_pairs for any
number of ranks -- and equality with the reference's run_dedup.  Per-rank
compute uses the oracle stand-ins of tests/cpu_stages.py; the same protocol
drives the CUDA stages under NCCL (tests/test_gpu_distributed.py)."""
import json
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, data, offs, out_path, cfg_kw):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from cpu_stages import CpuStages
    from paper_2501_01046_b200 import distributed, pipeline

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = len(offs) - 1
    lo, hi = n * rank // world, n * (rank + 1) // world
    sub = offs[lo:hi + 1] - offs[lo]
    shard = data[offs[lo]:offs[hi]]
    res = distributed.dedup_sharded(shard, sub, pipeline.RunConfig(**cfg_kw), CpuStages())
    if rank == 0:
        r = res.report
        with open(out_path, "w") as f:
            json.dump({"groups": [[g.representative, g.members] for g in r.groups],
                       "distinct": res.distinct_pairs, "cand": res.candidate_pairs,
                       "K": res.bucket_count, "N": res.documents}, f)
    dist.destroy_process_group()


def _run(world, data, offs, tmp_path, cfg_kw):
    out = str(tmp_path / f"w{world}.json")
    mp.spawn(_worker, args=(world, _free_port(), data, offs, out, cfg_kw), nprocs=world, join=True)
    return json.load(open(out))


@pytest.fixture(scope="module")
def corpus(ref):
    return ref.generate_synthetic(900, 60, gmin=2, gmax=4, edit=(2, 100), len_min=250,
                                  len_max=600, seed=13)


@pytest.mark.parametrize("cfg_kw", [{}, {"hash_count": 64, "bands": 8, "rows": 8,
                                          "threshold": (3, 4)}])
def test_rank_count_invariance(corpus, tmp_path, cfg_kw):
    data, offs = corpus
    res = [_run(w, data, offs, tmp_path, cfg_kw) for w in (1, 2, 3)]
    assert res[0]["groups"], "planted corpus must produce groups"
    assert res[0] == res[1] == res[2]


def test_sharded_matches_reference_run_dedup(corpus, ref, tmp_path):
    data, offs = corpus
    got = _run(2, data, offs, tmp_path, {})
    corpus_path = str(tmp_path / "c.jsonl")
    with open(corpus_path, "w") as f:
        for i in range(len(offs) - 1):
            f.write(json.dumps({"text": bytes(data[offs[i]:offs[i + 1]]).decode()}) + "\n")
    ws = str(tmp_path / "ws")
    os.makedirs(ws)
    ref.run_dedup(corpus_path, ws, workers=4)
    want = [json.loads(l) for l in open(os.path.join(ws, "groups.jsonl"))]
    assert got["groups"] == [[g["representative"], g["members"]] for g in want]
    summary = json.load(open(os.path.join(ws, "summary.json")))
    stage = json.load(open(os.path.join(ws, "compare_stage.json")))
    assert got["distinct"] == summary["distinct_pairs"]
    assert got["cand"] == stage["candidate_pairs"]
