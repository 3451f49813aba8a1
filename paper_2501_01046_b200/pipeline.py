"""Stage orchestration -- mirror of the reference's pipeline.hpp.

  RunConfig            pipeline.hpp:21-48 (same fields, validate, config_hash)
  run_dedup            pipeline.hpp:100   (JSONL inputs -> workspace report)
  dedup_packed         in-memory run_dedup over a packed batch (the hot path)
The reference persists every stage to disk (.feds, .pairs); here the three
stages run back to back on the GPU with intermediates resident in HBM
(nd_dedup), and only the report is written, with the reference's writers'
byte format (groups.jsonl, removal.txt, summary.json).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import NdDedupStats, NdParams, u8p, u64p
from .corpus import CorpusManifest, build_manifest, surviving_documents  # noqa: F401
from .dedup_graph import DedupReport, DuplicateGroup
from .device import Context, default_context
from .lsh import _ratio
from .minhash import ShingleUnit, pack_documents


@dataclass
class RunConfig:
    inputs: list[str] = field(default_factory=list)
    workspace: str = ""
    text_field: str = "text"
    hash_count: int = 128
    bands: int = 16
    rows: int = 8
    shingle_len: int = 5
    unit: ShingleUnit = ShingleUnit.BYTE
    threshold: tuple[int, int] = (4, 5)
    bucket_scale: tuple[int, int] = (2, 1)
    min_chars: int = 200
    seed: int = 5
    workers: int = 1
    memory_budget: int = 1 << 30
    buckets_per_pass: int | None = None
    tile_size: int = 32
    fsync_files: bool = False
    oracle_override: bool = False

    def validate(self, need_workspace: bool = False) -> None:
        """pipeline.cpp:20-33."""
        err = _lib.ConfigError
        if need_workspace and not self.workspace:
            raise err(_lib.ND_ERR_CONFIG, "workspace directory is required")
        if self.bands == 0 or self.rows == 0:
            raise err(_lib.ND_ERR_CONFIG, "bands and rows must be positive")
        if self.hash_count != self.bands * self.rows:
            raise err(_lib.ND_ERR_CONFIG, f"hash count {self.hash_count} must equal bands*rows = "
                                          f"{self.bands}*{self.rows}")
        if self.shingle_len == 0:
            raise err(_lib.ND_ERR_CONFIG, "shingle length must be positive")
        tn, td = _ratio(self.threshold)
        if tn > td:
            raise err(_lib.ND_ERR_CONFIG, "threshold must be at most 1")
        if _ratio(self.bucket_scale)[0] == 0:
            raise err(_lib.ND_ERR_CONFIG, "bucket scale must be positive")
        if self.workers == 0:
            raise err(_lib.ND_ERR_CONFIG, "worker count must be positive")
        if self.memory_budget == 0:
            raise err(_lib.ND_ERR_CONFIG, "memory budget must be positive")
        if self.tile_size == 0:
            raise err(_lib.ND_ERR_CONFIG, "tile size must be positive")

    def config_hash(self) -> int:
        """pipeline.cpp:35-54: FNV-1a over the artifact-shaping fields."""
        def rstr(r):
            from math import gcd

            n, d = _ratio(r)
            g = gcd(n, d) or 1
            n, d = n // g, d // g
            if n == 0:
                d = 1
            return str(n) if d == 1 else f"{n}/{d}"

        blob = "neardup-config-v1"
        for k, v in [("text_field", self.text_field), ("hash_count", str(self.hash_count)),
                     ("bands", str(self.bands)), ("rows", str(self.rows)),
                     ("shingle_len", str(self.shingle_len)),
                     ("unit", "byte" if self.unit == ShingleUnit.BYTE else "codepoint"),
                     ("threshold", rstr(self.threshold)),
                     ("bucket_scale", rstr(self.bucket_scale)),
                     ("min_chars", str(self.min_chars)), ("seed", str(self.seed))]:
            blob += f"|{k}={v}"
        h = 14695981039346656037
        for c in blob.encode():
            h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h

    def to_params(self, bucket_count: int = 0) -> NdParams:
        tn, td = _ratio(self.threshold)
        sn, sd = _ratio(self.bucket_scale)
        return NdParams(hash_count=self.hash_count, bands=self.bands, rows=self.rows,
                        shingle_len=self.shingle_len, unit=int(self.unit),
                        bucket_count=bucket_count, threshold_num=tn, threshold_den=td,
                        scale_num=sn, scale_den=sd, seed=self.seed)


def _fetch_report(ctx: Context, stats: NdDedupStats, lists: bool = True) -> DedupReport:
    mem = np.empty(stats.near_duplicates, np.uint64)
    gs = np.empty(stats.duplicate_groups + 1, np.uint64)
    ctx.check(ctx.lib.nd_dedup_fetch_groups(ctx.h, mem.ctypes.data_as(u64p), gs.ctypes.data_as(u64p)))
    if not lists:  # arrays only: members in group order + group offsets
        rep = DedupReport(total_documents=stats.documents, distinct_pairs=stats.distinct_pairs)
        rep.candidate_pairs = stats.candidate_pairs
        rep.group_members, rep.group_start = mem, gs
        rep.stats = {k: getattr(stats, k) for k, _ in NdDedupStats._fields_ if k != "seconds"}
        rep.stats["seconds"] = list(stats.seconds)
        return rep
    groups = []
    for g in range(stats.duplicate_groups):
        m = mem[int(gs[g]):int(gs[g + 1])].tolist()
        groups.append(DuplicateGroup(m[0], m))
    near = sorted(mem.tolist())
    removals = sorted(int(x) for g in groups for x in g.members[1:])
    total = stats.documents
    rep = DedupReport(groups, near, removals, total, stats.distinct_pairs,
                      len(near) / total if total else 0.0)
    rep.candidate_pairs = stats.candidate_pairs
    rep.stats = {k: getattr(stats, k) for k, _ in NdDedupStats._fields_ if k != "seconds"}
    rep.stats["seconds"] = list(stats.seconds)
    return rep


def dedup_packed(data: np.ndarray, offsets: np.ndarray, config: RunConfig | None = None,
                 doc_ids: np.ndarray | None = None, bucket_count: int = 0,
                 ctx: Context | None = None, fetch="lists") -> DedupReport:
    """In-memory run_dedup over a packed batch of surviving documents (host buffers).

    doc_ids (ascending) default to 0..n-1.  bucket_count 0 = choose_bucket_count(n).
    fetch: "lists" (DuplicateGroup objects), "arrays" (numpy members + offsets),
    or None (statistics only; results stay on the device)."""
    config = config or RunConfig()
    config.validate()
    ctx = ctx or default_context()
    data = np.ascontiguousarray(data, np.uint8)
    offsets = np.ascontiguousarray(offsets, np.uint64)
    n = len(offsets) - 1
    ids = None if doc_ids is None else np.ascontiguousarray(doc_ids, np.uint64)
    stats = NdDedupStats()
    params = config.to_params(bucket_count)
    dp = data.ctypes.data_as(u8p) if data.size else C.cast(C.c_char_p(b"\0"), u8p)
    ctx.check(ctx.lib.nd_dedup(ctx.h, dp, offsets.ctypes.data_as(u64p),
                               ids.ctypes.data_as(u64p) if ids is not None else None, n,
                               C.byref(params), C.byref(stats)))
    if not fetch:
        rep = DedupReport(total_documents=stats.documents, distinct_pairs=stats.distinct_pairs)
        rep.candidate_pairs = stats.candidate_pairs
        return rep
    return _fetch_report(ctx, stats, lists=(fetch != "arrays"))


def dedup_pairs(distinct_pairs: int, ctx: Context | None = None):
    """Sorted distinct duplicate pairs (doc ids) of the last dedup on ctx."""
    from .compare import DuplicatePair

    ctx = ctx or default_context()
    lo = np.empty(distinct_pairs, np.uint64)
    hi = np.empty(distinct_pairs, np.uint64)
    m = np.empty(distinct_pairs, np.uint32)
    ctx.check(ctx.lib.nd_dedup_fetch_pairs(ctx.h, lo.ctypes.data_as(u64p), hi.ctypes.data_as(u64p),
                                           m.ctypes.data_as(_lib.u32p)))
    return [DuplicatePair(int(a), int(b), int(c)) for a, b, c in zip(lo, hi, m)]


def write_report(workspace: str, ctx: Context | None = None, total_records: int = 0) -> None:
    ctx = ctx or default_context()
    os.makedirs(workspace, exist_ok=True)
    ctx.check(ctx.lib.nd_dedup_write_report(ctx.h, workspace.encode(), total_records))


def run_dedup(config: RunConfig, ctx: Context | None = None) -> DedupReport:
    """pipeline.cpp:510-532 on the GPU: load + filter the JSONL inputs, dedup in
    memory, write groups.jsonl / removal.txt / summary.json (+ rejects.jsonl)."""
    config.validate(need_workspace=True)
    os.makedirs(config.workspace, exist_ok=True)
    manifest, rejects = build_manifest(config.inputs, config)
    if manifest.total_surviving == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                               "no documents survive preprocessing; nothing to deduplicate")
    docs = []
    for i in range(len(manifest.files)):
        docs.extend(surviving_documents(manifest, i, config))
    data, offsets = pack_documents(docs)
    ids = np.array([d.doc_id for d in docs], np.uint64)
    ctx = ctx or default_context()
    rep = dedup_packed(data, offsets, config, ids, ctx=ctx)
    write_report(config.workspace, ctx, manifest.total_records)
    with open(os.path.join(config.workspace, "rejects.jsonl"), "w") as f:
        for e in rejects:
            f.write(json.dumps({"file": e[0], "line": e[1], "reason": e[2]},
                               separators=(",", ":")) + "\n")
    return rep
