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
