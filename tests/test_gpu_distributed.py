"""The multi-GPU dedup protocol on the CUDA stages (NCCL, world size 1 on the
single-GPU box): identical to the single-GPU in-memory path and to the
reference.  Multi-rank invariance of the same protocol is covered under gloo
by tests/test_distributed.py."""
import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_nccl_world1_equals_single_gpu(ctx, ref):
    import torch
    import torch.distributed as dist

    from paper_2501_01046_b200 import distributed, pipeline

    data, offs = ref.generate_synthetic(3000, 200, gmin=2, gmax=3, edit=(2, 100), len_min=300,
                                        len_max=900, seed=17)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        res = distributed.dedup_sharded(data, offs, pipeline.RunConfig(),
                                        distributed.GpuStages(ctx, torch.device("cuda", 0)))
    finally:
        dist.destroy_process_group()
    single = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
    got = [(g.representative, g.members) for g in res.report.groups]
    assert got == [(g.representative, g.members) for g in single.groups]
    assert got, "planted corpus must produce groups"
    assert res.distinct_pairs == single.distinct_pairs
    assert res.candidate_pairs == single.candidate_pairs


def _gpu_worker(rank, world, port, data, offs, out_path):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2501_01046_b200 import distributed, pipeline
    from paper_2501_01046_b200.device import Context

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = len(offs) - 1
    lo, hi = n * rank // world, n * (rank + 1) // world
    sub = offs[lo:hi + 1] - offs[lo]
    shard = data[offs[lo]:offs[hi]]
    ctx = Context(0)
    res = distributed.dedup_sharded(shard, sub, pipeline.RunConfig(),
                                    distributed.GpuStages(ctx, torch.device("cuda", 0)))
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"groups": [[g.representative, g.members] for g in res.report.groups],
                       "distinct": res.distinct_pairs, "cand": res.candidate_pairs,
                       "emitted": res.emitted_pairs}, f)
    dist.destroy_process_group()
    ctx.close()


@pytest.mark.parametrize("world,peer,k3", [(2, "1", ""), (3, "1", ""), (2, "0", ""), (2, "1", "cells")])
def test_sharded_cuda_stages_several_ranks(ctx, ref, tmp_path, monkeypatch, world, peer, k3):
    # the multi-rank protocol over the REAL device stages: `world` processes
    # share the one GPU (gloo moves the collective buffers through the host;
    # NCCL refuses two ranks on one device) -- owner split, all-to-all of cell
    # records, all-gathers and the union all run on K1..K4.  peer="1": K3 reads
    # the other ranks' signature rows through CUDA IPC mappings (nd_peer.cu);
    # "0": the rows are all-gathered
    import torch.multiprocessing as mp

    monkeypatch.setenv("ND_PEER_SIGS", peer)
    if k3:
        monkeypatch.setenv("ND_K3", k3)
    else:
        monkeypatch.delenv("ND_K3", raising=False)
    from paper_2501_01046_b200 import pipeline

    data, offs = ref.generate_synthetic(2500, 200, gmin=2, gmax=4, edit=(2, 100), len_min=300,
                                        len_max=900, seed=29)
    out = str(tmp_path / "r.json")
    mp.spawn(_gpu_worker, args=(world, _free_port(), data, offs, out), nprocs=world, join=True)
    got = json.load(open(out))
    single = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
    assert got["groups"] == [[g.representative, g.members] for g in single.groups]
    assert got["groups"]
    assert got["distinct"] == single.distinct_pairs
    assert got["cand"] == single.candidate_pairs
    if peer == "1" and not k3:
        # K3g over IPC peer memory: each rank joins its blocks over all rows;
        # the emitted-pairs counter (one per shared cell) equals one device's
        monkeypatch.delenv("ND_K3", raising=False)
        one = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), ctx=ctx)
        assert got["emitted"] == one.stats["emitted_pairs"]


def test_bench_two_ranks_harness(tmp_path):
    # bench.py's multi-rank path (barriers, max over ranks, sharded dedup,
    # one JSON line on rank 0) with two ranks sharing the GPU through gloo
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ND_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--docs", "100000", "--no-cpu",
           "--no-staged"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["dedup"]["documents"] == 200000 and d["gpu_launches"] > 0
