"""Multi-GPU dedup: one process per GPU, documents sharded by contiguous ranges
(SURVEY 8e).  The reference partitions bands over worker threads
(band_partition, lsh.cpp:62-72; paper: "process j is in charge of
N_band/N_GPU bands"); here cells (band*K + bucket) are owned by
contiguous ranges so that any number of GPUs is balanced (nd_cell_partition).

  1. N = all-reduce(n_r); K = choose_bucket_count(N); doc_base = exclusive
     prefix of n_r (global row = doc_base + local row, ascending doc order).
  2. K1 on the local shard (rank-local, no collective).
  3. (cell, row) records of the shard, stably sorted by cell on the device;
     split by owner range -> all-to-all (counts, then records).  Records
     arrive grouped by source rank = ascending rows, so a stable regroup keeps
     each cell's rows ascending, like the reference's file scan.
  4. Every owner must read any row: by default each rank exports its rows as
     a CUDA IPC handle, the handles are all-gathered and K3 reads the other
     ranks' rows in peer memory over NVLink (nd_peer.cu); ND_PEER_SIGS=0 (and
     the CPU protocol tests) all-gather the rows instead.
  5. K2+K3 on the owned cells -> distinct pairs (global rows).
  6. All-gather of the pairs; K4 (distinct + components) on every rank
     (cheap, identical everywhere); rank 0 writes / returns the report.
Outputs are identical for any number of ranks (tests/test_distributed.py).

The per-rank compute steps go through a "stages" object; GpuStages (the
product) calls the C-ABI on device tensors.  torch.distributed is plumbing:
NCCL over NVLink on GPUs, gloo on CPU for the protocol tests.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import NdDedupStats
from .lsh import cell_partition, choose_bucket_count, _ratio


@dataclass
class ShardResult:
    report: object | None  # DedupReport on rank 0 (fetch="lists"/"arrays"), else None
    candidate_pairs: int
    emitted_pairs: int
    distinct_pairs: int
    bucket_count: int
    documents: int


class GpuStages:
    """Per-rank device stages over torch CUDA tensors (C-ABI entry points)."""

    def __init__(self, ctx, device):
        import torch

        self.torch = torch
        self.ctx = ctx
        self.device = device

    def tensor(self, shape, dtype):
        return self.torch.empty(shape, dtype=dtype, device=self.device)

    def signatures(self, data, offsets, family, bands, rows, K):
        """Pinned host text -> device signatures/band keys (pipelined H2D + K1)."""
        t = self.torch
        n = len(offsets) - 1
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        sig = self.tensor((n, family.hash_count), t.int32)
        band = self.tensor((n, bands), t.int32)
        self.ctx.upload_family(family)
        self.ctx.check(self.ctx.lib.nd_signatures_h2d(
            self.ctx.h, data.ctypes.data_as(_lib.u8p), offsets.ctypes.data_as(_lib.u64p), n, bands,
            rows, K, C.c_void_p(sig.data_ptr()), C.c_void_p(band.data_ptr())))
        return sig, band

    def ctx_sync(self):
        self.torch.cuda.synchronize(self.device)

    def cell_records(self, band, bands, K, doc_base):
        t = self.torch
        n = band.shape[0]
        keys = self.tensor((n * bands,), t.int32)
        vals = self.tensor((n * bands,), t.int32)
        self.ctx.check(self.ctx.lib.nd_stage_cell_records(
            self.ctx.h, C.c_void_p(band.data_ptr()), n, bands, K, doc_base,
            C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr())))
        self.ctx_sync()
        return keys, vals

    def compare(self, sig_all, keys, vals, key_limit, H, threshold):
        """K2 + K3 + distinct pairs of the owned cells; returns (lo, hi, m, candidates)."""
        t = self.torch
        num, den = threshold
        npairs, cand = C.c_uint64(), C.c_uint64()
        self.ctx.check(self.ctx.lib.nd_stage_compare(
            self.ctx.h, C.c_void_p(sig_all.data_ptr()), sig_all.shape[0], H,
            C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()), keys.shape[0], key_limit,
            num, den, C.byref(npairs), C.byref(cand)))
        k = npairs.value
        lo, hi, m = (self.tensor((max(k, 1),), t.int32) for _ in range(3))
        self.ctx.check(self.ctx.lib.nd_stage_pairs_copy(
            self.ctx.h, C.c_void_p(lo.data_ptr()), C.c_void_p(hi.data_ptr()),
            C.c_void_p(m.data_ptr())))
        self.ctx_sync()
        return lo[:k], hi[:k], m[:k], cand.value

    # ---- compare over peer memory (nd_peer.cu): the other ranks' rows are read
    # in place through CUDA IPC mappings instead of being all-gathered
    peer_capable = True

    def export_rows(self, sig) -> bytes:
        h = (C.c_uint8 * 64)()
        self.ctx.check(self.ctx.lib.nd_peer_export(self.ctx.h, C.c_void_p(sig.data_ptr()),
                                                   sig.shape[0], sig.shape[1], h))
        return bytes(h)

    def open_peers(self, handles: bytes, row_base, world: int, rank: int) -> None:
        hb = (C.c_uint8 * len(handles)).from_buffer_copy(handles)
        rb = np.ascontiguousarray(row_base, np.uint64)
        self.ctx.check(self.ctx.lib.nd_peer_open(self.ctx.h, hb, rb.ctypes.data_as(_lib.u64p),
                                                 world, rank))

    # ---- packed records: one u64 per (cell, row), sorted by cell, with the owner
    # splits found on the device (one all-to-all instead of two)
    packed_capable = True

    def records_packed(self, band, bands, K, doc_base, world):
        t = self.torch
        n = band.shape[0]
        rec = self.tensor((max(n * bands, 1),), t.int64)
        split = np.zeros(world + 1, np.uint64)
        self.ctx.check(self.ctx.lib.nd_stage_records_packed(
            self.ctx.h, C.c_void_p(band.data_ptr()), n, bands, K, doc_base, world,
            C.c_void_p(rec.data_ptr()), split.ctypes.data_as(_lib.u64p)))
        return rec[: n * bands], [int(x) for x in split]

    def compare_peer_packed(self, rec, key_limit, threshold):
        t = self.torch
        num, den = threshold
        npairs, cand = C.c_uint64(), C.c_uint64()
        self.ctx.check(self.ctx.lib.nd_stage_compare_peer_packed(
            self.ctx.h, C.c_void_p(rec.data_ptr()), rec.shape[0], key_limit, num, den,
            C.byref(npairs), C.byref(cand)))
        k = npairs.value
        lo, hi, m = (self.tensor((max(k, 1),), t.int32) for _ in range(3))
        self.ctx.check(self.ctx.lib.nd_stage_pairs_copy(
            self.ctx.h, C.c_void_p(lo.data_ptr()), C.c_void_p(hi.data_ptr()),
            C.c_void_p(m.data_ptr())))
        self.ctx_sync()
        return lo[:k], hi[:k], m[:k], cand.value

    def compare_peer(self, keys, vals, key_limit, threshold):
        t = self.torch
        num, den = threshold
        npairs, cand = C.c_uint64(), C.c_uint64()
        self.ctx.check(self.ctx.lib.nd_stage_compare_peer(
            self.ctx.h, C.c_void_p(keys.data_ptr()), C.c_void_p(vals.data_ptr()), keys.shape[0],
            key_limit, num, den, C.byref(npairs), C.byref(cand)))
        k = npairs.value
        lo, hi, m = (self.tensor((max(k, 1),), t.int32) for _ in range(3))
        self.ctx.check(self.ctx.lib.nd_stage_pairs_copy(
            self.ctx.h, C.c_void_p(lo.data_ptr()), C.c_void_p(hi.data_ptr()),
            C.c_void_p(m.data_ptr())))
        self.ctx_sync()
        return lo[:k], hi[:k], m[:k], cand.value

    def close_peers(self) -> None:
        self.ctx.check(self.ctx.lib.nd_peer_close(self.ctx.h))

    # ---- K3g over peer memory: every rank's rows, band ids and block
    # fingerprints mapped in place; rank r joins the blocks k = r (mod world)
    gjoin_capable = True

    def cell_hist(self, band, bands, K):
        cnt = self.tensor((bands * K,), self.torch.int32)
        self.ctx.check(self.ctx.lib.nd_stage_cell_hist(
            self.ctx.h, C.c_void_p(band.data_ptr()), band.shape[0], bands, K,
            C.c_void_p(cnt.data_ptr())))
        return cnt

    def export_gjoin(self, sig, band, threshold) -> bytes:
        h = (C.c_uint8 * 64)()
        num, den = threshold
        self.ctx.check(self.ctx.lib.nd_peer_export_gjoin(
            self.ctx.h, C.c_void_p(sig.data_ptr()), C.c_void_p(band.data_ptr()), sig.shape[0],
            sig.shape[1], band.shape[1], num, den, h))
        return bytes(h)

    def gjoin_peer(self, rank: int):
        t = self.torch
        npairs, emitted = C.c_uint64(), C.c_uint64()
        self.ctx.check(self.ctx.lib.nd_stage_gjoin_peer(self.ctx.h, rank, C.byref(npairs),
                                                        C.byref(emitted)))
        k = npairs.value
        lo, hi, m = (self.tensor((max(k, 1),), t.int32) for _ in range(3))
        self.ctx.check(self.ctx.lib.nd_stage_pairs_copy(
            self.ctx.h, C.c_void_p(lo.data_ptr()), C.c_void_p(hi.data_ptr()),
            C.c_void_p(m.data_ptr())))
        self.ctx_sync()
        return lo[:k], hi[:k], m[:k], emitted.value

    def union(self, lo, hi, m, nnodes):
        st = NdDedupStats()
        ptr = (lambda x: C.c_void_p(x.data_ptr()) if x.numel() else None)
        self.ctx.check(self.ctx.lib.nd_stage_union(self.ctx.h, ptr(lo), ptr(hi), ptr(m),
                                                   lo.numel(), nnodes, C.byref(st)))
        return st

    def report(self, stats, fetch):
        from .pipeline import _fetch_report

        return _fetch_report(self.ctx, stats, lists=(fetch != "arrays"))


def _all_gather_var(dist, t, group, torch):
    """all_gather of a 1-D/2-D tensor whose first dimension differs per rank."""
    world = dist.get_world_size(group)
    dev = t.device
    if _host_collectives(dist, group, dev):  # gloo: collectives on host copies
        out, sizes = _all_gather_var(dist, t.cpu(), group, torch)
        return out.to(dev), sizes
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)]), sizes


def _all_gather_v(dist, t, group, torch):
    """all_gather of tensors whose first dimension differs per rank without
    padding: every rank sends its whole tensor to every rank through one
    all-to-all (NCCL's all-gather-v); gloo groups fall back to the padded form."""
    world = dist.get_world_size(group)
    if world == 1:
        return t, [t.shape[0]]
    if _host_collectives(dist, group, t.device):
        return _all_gather_var(dist, t, group, torch)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    flat = t.reshape(t.shape[0], -1)
    out = torch.empty((sum(sizes), flat.shape[1]), dtype=t.dtype, device=t.device)
    send = flat.repeat(world, 1) if t.shape[0] else flat
    dist.all_to_all_single(out, send, [s for s in sizes], [t.shape[0]] * world, group=group)
    return out.reshape((sum(sizes),) + tuple(t.shape[1:])), sizes


def _events(torch, dev, timings):
    if timings is None or dev.type != "cuda":
        return None
    return [torch.cuda.Event(enable_timing=True) for _ in range(4)]


def _host_collectives(dist, group, device) -> bool:
    """NCCL runs the collectives on device tensors; a gloo group (CPU protocol
    tests, or several ranks sharing one GPU in the GPU tests) gets host copies."""
    return device.type == "cuda" and dist.get_backend(group) == "gloo"


def dedup_sharded(data, offsets, config, stages, group=None, fetch="lists",
                  timings: dict | None = None) -> ShardResult:
    """Distributed in-memory dedup of this rank's shard (see module doc).
    `timings` (optional) receives this rank's device times of the cell-record
    all-to-all and the edge all-gather (CUDA events on the current stream,
    which waits for the collective) and the bytes it sent / received."""
    import torch
    import torch.distributed as dist

    from .minhash import derive_family

    config.validate()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = stages.device
    host = _host_collectives(dist, group, dev)
    cdev = torch.device("cpu") if host else dev  # where collective buffers live
    n_local = len(offsets) - 1
    # 1. global N, K, doc_base
    cnt = torch.tensor([n_local], dtype=torch.int64, device=cdev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    N = sum(counts)
    doc_base = sum(counts[:rank])
    if N == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                               "no documents survive preprocessing; nothing to deduplicate")
    if N >= 2**32:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "more than 2^32 documents")
    K = choose_bucket_count(N, config.bucket_scale)
    b = config.bands
    fam = derive_family(config.seed, config.hash_count, config.shingle_len, config.unit)
    # 2. K1 on the shard
    sig, band = stages.signatures(data, offsets, fam, b, config.rows, K)
    thr = _ratio(config.threshold)
    ev = _events(torch, dev, timings)
    mm = _lib.load().nd_min_matches(config.hash_count, thr[0], thr[1])
    nblocks = config.hash_count - mm + 1 if mm <= config.hash_count else 0
    if (getattr(stages, "gjoin_capable", False) and os.environ.get("ND_K3", "") != "cells"
            and os.environ.get("ND_PEER_SIGS", "1") != "0" and nblocks <= 64):
        return _dedup_gjoin(stages, sig, band, counts, N, K, b, thr, rank, world, group, dev,
                            cdev, ev, timings, fetch, dist, torch)
    # 3. records -> owners
    packed = getattr(stages, "packed_capable", False) and os.environ.get("ND_PEER_SIGS", "1") != "0"
    if packed:
        # one u64 per (cell, row), sorted by cell, owner splits from the device
        rec, split = stages.records_packed(band, b, K, doc_base, world)
        send = [split[i + 1] - split[i] for i in range(world)]
    else:
        keys, vals = stages.cell_records(band, b, K, doc_base)
        first = cell_partition(b, K, world)
        bounds = torch.tensor(first[1:-1], dtype=torch.int64, device=dev)
        splits = torch.searchsorted(keys.to(torch.int64), bounds) if world > 1 else \
            torch.zeros(0, dtype=torch.int64, device=dev)
        edges = [0] + [int(x) for x in splits.tolist()] + [keys.shape[0]]
        send = [edges[i + 1] - edges[i] for i in range(world)]
    send_t = torch.tensor(send, dtype=torch.int64, device=cdev)
    recv_t = torch.empty_like(send_t)
    dist.all_to_all_single(recv_t, send_t, group=group)
    recv = [int(x) for x in recv_t.tolist()]
    if ev:
        ev[0].record()
    if packed:
        rrec = torch.empty(sum(recv), dtype=torch.int64, device=cdev)
        dist.all_to_all_single(rrec, rec.to(cdev), recv, send, group=group)
        rec_bytes = 8
    else:
        rkeys = torch.empty(sum(recv), dtype=keys.dtype, device=cdev)
        rvals = torch.empty(sum(recv), dtype=vals.dtype, device=cdev)
        dist.all_to_all_single(rkeys, keys.to(cdev), recv, send, group=group)
        dist.all_to_all_single(rvals, vals.to(cdev), recv, send, group=group)
        rec_bytes = keys.element_size() + vals.element_size()
    if ev:
        ev[1].record()
    if packed:
        h = torch.tensor(list(stages.export_rows(sig)), dtype=torch.uint8, device=cdev)
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h, group=group)
        handles = b"".join(bytes(x.cpu().tolist()) for x in hs)
        row_base = [sum(counts[:r]) for r in range(world + 1)]
        stages.open_peers(handles, row_base, world, rank)
        lo, hi, m, cand_local = stages.compare_peer_packed(rrec.to(dev), b * K, thr)
        dist.barrier(group=group)
        stages.close_peers()
    elif getattr(stages, "peer_capable", False) and os.environ.get("ND_PEER_SIGS", "1") != "0":
        rkeys, rvals = rkeys.to(dev), rvals.to(dev)
        # 4+5. compare the owned cells reading every rank's rows in peer memory:
        # exchange IPC handles, map, compare, and keep the rows alive until
        # every rank is done (barrier)
        h = torch.tensor(list(stages.export_rows(sig)), dtype=torch.uint8, device=cdev)
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h, group=group)
        handles = b"".join(bytes(x.cpu().tolist()) for x in hs)
        row_base = [sum(counts[:r]) for r in range(world + 1)]
        stages.open_peers(handles, row_base, world, rank)
        lo, hi, m, cand_local = stages.compare_peer(rkeys, rvals, b * K, thr)
        dist.barrier(group=group)
        stages.close_peers()
    else:
        rkeys, rvals = rkeys.to(dev), rvals.to(dev)
        # 4. all signature rows on every rank
        sig_all, _ = _all_gather_var(dist, sig, group, torch)
        # 5. compare the owned cells
        lo, hi, m, cand_local = stages.compare(sig_all, rkeys, rvals, b * K, config.hash_count, thr)
    emitted = torch.tensor([lo.shape[0]], dtype=torch.int64, device=cdev)
    # candidate pairs of the owned cells (sum n(n-1)/2, pipeline.cpp:406-411)
    cand = torch.tensor([cand_local], dtype=torch.int64, device=cdev)
    dist.all_reduce(cand, group=group)
    dist.all_reduce(emitted, group=group)
    # 6. edges everywhere, union stage
    trip = torch.stack([lo, hi, m], dim=1) if lo.numel() else torch.zeros((0, 3), dtype=lo.dtype, device=dev)
    if ev:
        ev[2].record()
    all_trip, _ = _all_gather_v(dist, trip, group, torch)
    if ev:
        ev[3].record()
        torch.cuda.synchronize(dev)
        timings.update(
            exchange_ms=ev[0].elapsed_time(ev[1]),
            exchange_sent_bytes=(sum(send) - send[rank]) * rec_bytes,
            exchange_recv_bytes=(sum(recv) - recv[rank]) * rec_bytes,
            edges_ms=ev[2].elapsed_time(ev[3]),
            edges_bytes=int(all_trip.numel()) * all_trip.element_size())
    st = stages.union(all_trip[:, 0].contiguous(), all_trip[:, 1].contiguous(),
                      all_trip[:, 2].contiguous(), N)
    rep = stages.report(st, fetch) if (rank == 0 and fetch) else None
    if rep is not None:
        rep.candidate_pairs = int(cand.item())
    return ShardResult(rep, int(cand.item()), int(emitted.item()), st.distinct_pairs, K, N)


def _dedup_gjoin(stages, sig, band, counts, N, K, b, thr, rank, world, group, dev, cdev, ev,
                 timings, fetch, dist, torch) -> ShardResult:
    """K3g across ranks (nd_stage_gjoin_peer): no record exchange -- the cell
    histograms are all-reduced for the reference's counters, and each rank
    joins its blocks over every rank's rows, band ids and fingerprints read in
    place through CUDA IPC mappings (NVLink peer memory)."""
    cnt = stages.cell_hist(band, b, K)
    if ev:
        ev[0].record()
    c = cnt.to(cdev)
    dist.all_reduce(c, group=group)
    if ev:
        ev[1].record()
    c = c.to(torch.int64)
    cand_total = int((c * (c - 1) // 2).sum().item())
    h = torch.tensor(list(stages.export_gjoin(sig, band, thr)), dtype=torch.uint8, device=cdev)
    hs = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(hs, h, group=group)
    handles = b"".join(bytes(x.cpu().tolist()) for x in hs)
    row_base = [sum(counts[:r]) for r in range(world + 1)]
    stages.open_peers(handles, row_base, world, rank)
    lo, hi, m, emitted_local = stages.gjoin_peer(rank)
    dist.barrier(group=group)
    stages.close_peers()
    emitted = torch.tensor([emitted_local], dtype=torch.int64, device=cdev)
    dist.all_reduce(emitted, group=group)
    trip = torch.stack([lo, hi, m], dim=1) if lo.numel() else torch.zeros((0, 3), dtype=lo.dtype, device=dev)
    if ev:
        ev[2].record()
    all_trip, _ = _all_gather_v(dist, trip, group, torch)
    if ev:
        ev[3].record()
        torch.cuda.synchronize(dev)
        timings.update(
            exchange_ms=ev[0].elapsed_time(ev[1]),
            exchange_sent_bytes=int(c.numel()) * 4,
            exchange_recv_bytes=int(c.numel()) * 4,
            edges_ms=ev[2].elapsed_time(ev[3]),
            edges_bytes=int(all_trip.numel()) * all_trip.element_size(),
            compare="global")
    st = stages.union(all_trip[:, 0].contiguous(), all_trip[:, 1].contiguous(),
                      all_trip[:, 2].contiguous(), N)
    rep = stages.report(st, fetch) if (rank == 0 and fetch) else None
    if rep is not None:
        rep.candidate_pairs = cand_total
    return ShardResult(rep, cand_total, int(emitted.item()), st.distinct_pairs, K, N)
