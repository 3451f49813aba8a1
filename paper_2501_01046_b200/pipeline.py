"""Stage orchestration -- mirror of the reference's pipeline.hpp.

  RunConfig            pipeline.hpp:21-48 (same fields, validate, config_hash)
  run_hash_stage       pipeline.cpp:269-339  JSONL -> K1 on the GPU -> one .feds file per input
  run_compare_stage    pipeline.cpp:382-432  .feds -> HBM -> K2/K3 -> one .pairs file per
                                             (worker, gather pass) + compare_stage.json
  run_union_stage      pipeline.cpp:434-508  .pairs -> K4 -> groups.jsonl, removal.txt, summary.json
  run_dedup            pipeline.cpp:510-532  the three stages + timings.json
  run_dedup_in_memory  the same report with every intermediate resident in HBM (nd_dedup)
  dedup_packed         in-memory dedup of a packed host batch (the bench's hot path)
Every artifact is written with the reference's byte format, so a workspace
produced here is byte-identical with the reference's (tests/test_gpu_stages.py).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import NdDedupStats, NdParams, u8p, u64p
from .corpus import (CorpusManifest, build_manifest, build_manifest_cached,  # noqa: F401
                     default_text_cache_bytes, surviving_documents, surviving_packed)
from .dedup_graph import DedupReport, DuplicateGroup
from .device import Context, default_context
from .lsh import _ratio
from .minhash import ShingleUnit, pack_documents  # noqa: F401  (re-exported: the reference API)


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
    # schedule only (not artifact-shaping): HBM the compare stage may fill per
    # bucket interval; 0 = 70 % of free device memory (nd_set_hbm_budget)
    hbm_budget: int = 0

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
    # HBM budget of the in-memory dedup (0 = 70% of free device memory):
    # above it, bucket intervals run out of core over host-resident rows
    ctx.check(ctx.lib.nd_set_hbm_budget(ctx.h, config.hbm_budget))
    ctx.check(ctx.lib.nd_dedup(ctx.h, dp, offsets.ctypes.data_as(u64p),
                               ids.ctypes.data_as(u64p) if ids is not None else None, n,
                               C.byref(params), C.byref(stats)))
    if not fetch:
        rep = DedupReport(total_documents=stats.documents, distinct_pairs=stats.distinct_pairs)
        rep.candidate_pairs = stats.candidate_pairs
        return rep
    return _fetch_report(ctx, stats, lists=(fetch != "arrays"))


def dedup_signatures(sig: np.ndarray, band: np.ndarray, config: RunConfig | None = None,
                     doc_ids: np.ndarray | None = None, bucket_count: int = 0,
                     ctx: Context | None = None, fetch="lists") -> DedupReport:
    """In-memory compare + union over signature rows already computed (n x H
    sig, n x bands band ids, e.g. from read_sig_file): the compare and union
    stages of run_dedup (pipeline.cpp:347-476) without their files."""
    config = config or RunConfig()
    config.validate()
    ctx = ctx or default_context()
    sig = np.ascontiguousarray(sig, np.uint32)
    band = np.ascontiguousarray(band, np.uint32)
    n = sig.shape[0]
    if sig.shape != (n, config.hash_count) or band.shape != (n, config.bands):
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "signature / band id shapes do not match the config")
    ids = None if doc_ids is None else np.ascontiguousarray(doc_ids, np.uint64)
    stats = NdDedupStats()
    params = config.to_params(bucket_count)
    ctx.check(ctx.lib.nd_dedup_signatures(ctx.h, sig.ctypes.data_as(_lib.u32p),
                                          band.ctypes.data_as(_lib.u32p),
                                          ids.ctypes.data_as(u64p) if ids is not None else None, n,
                                          C.byref(params), C.byref(stats)))
    if not fetch:
        rep = DedupReport(total_documents=stats.documents, distinct_pairs=stats.distinct_pairs)
        rep.candidate_pairs = stats.candidate_pairs
        return rep
    return _fetch_report(ctx, stats, lists=(fetch != "arrays"))


def dedup_compare_kind(ctx: Context | None = None) -> str:
    """How the last in-memory dedup on ctx compared: "global" or "cells"."""
    ctx = ctx or default_context()
    return ctx.lib.nd_dedup_compare_kind(ctx.h).decode()


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


def run_dedup_in_memory(config: RunConfig, ctx: Context | None = None) -> DedupReport:
    """pipeline.cpp:510-532 with every intermediate kept in HBM: load + filter the
    JSONL inputs, dedup in memory (nd_dedup), write groups.jsonl / removal.txt /
    summary.json (+ rejects.jsonl).  Same report bytes as run_dedup, no .feds or
    .pairs artifacts."""
    config.validate(need_workspace=True)
    os.makedirs(config.workspace, exist_ok=True)
    manifest, rejects, cache = build_manifest_cached(config.inputs, config,
                                                     default_text_cache_bytes())
    if manifest.total_surviving == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                               "no documents survive preprocessing; nothing to deduplicate")
    parts = [cache.pop(i, None) or surviving_packed(manifest, i, config)
             for i in range(len(manifest.files))]
    data = np.concatenate([p[0] for p in parts])
    offsets = np.zeros(manifest.total_surviving + 1, np.uint64)
    np.cumsum(np.concatenate([np.diff(p[1]) for p in parts]), out=offsets[1:])
    ids = np.concatenate([p[2] for p in parts])
    ctx = ctx or default_context()
    rep = dedup_packed(data, offsets, config, ids, ctx=ctx)
    write_report(config.workspace, ctx, manifest.total_records)
    _write_rejects(rejects_path(config), rejects)
    return rep


# ---- the staged, file-backed workflow (pipeline.hpp:50-96) ---------------------
def run_manifest_path(c: RunConfig) -> str:
    return c.workspace + "/run_manifest.json"


def rejects_path(c: RunConfig) -> str:
    return c.workspace + "/rejects.jsonl"


def compare_stage_path(c: RunConfig) -> str:
    return c.workspace + "/compare_stage.json"


def groups_path(c: RunConfig) -> str:
    return c.workspace + "/groups.jsonl"


def removal_path(c: RunConfig) -> str:
    return c.workspace + "/removal.txt"


def summary_path(c: RunConfig) -> str:
    return c.workspace + "/summary.json"


def timings_path(c: RunConfig) -> str:
    return c.workspace + "/timings.json"


def accuracy_path(c: RunConfig) -> str:
    return c.workspace + "/accuracy.json"


def run_eval_accuracy(config: RunConfig, ctx: Context | None = None) -> dict:
    """pipeline.cpp:534-585 (implemented in accuracy.py)."""
    from .accuracy import run_eval_accuracy as _run

    return _run(config, ctx=ctx)


def signatures_dir(c: RunConfig) -> str:
    return c.workspace + "/signatures"


def pairs_dir(c: RunConfig) -> str:
    return c.workspace + "/pairs"


def _dump2(obj) -> str:
    """nlohmann ordered_json::dump(2) + newline (UTF-8 kept, same escapes)."""
    return json.dumps(obj, indent=2, ensure_ascii=False) + "\n"


def _write_text(path: str, text: str, fsync: bool = False) -> None:
    """write_file_bytes (util.cpp:132-140): write, flush, optional fsync."""
    with open(path, "w", encoding="utf-8", newline="") as f:
        f.write(text)
        if fsync:
            f.flush()
            os.fsync(f.fileno())


def _write_rejects(path: str, rejects) -> None:
    """RejectLog::write_jsonl (corpus.cpp:18-29)."""
    _write_text(path, "".join(json.dumps({"file": e[0], "line": e[1], "reason": e[2]},
                                         separators=(",", ":"), ensure_ascii=False) + "\n"
                              for e in rejects))


def _ratio_str(r) -> str:
    from math import gcd

    n, d = _ratio(r)
    g = gcd(n, d) or 1
    n, d = n // g, d // g
    if n == 0:
        d = 1
    return str(n) if d == 1 else f"{n}/{d}"


def _parameters(c: RunConfig) -> dict:
    """config_parameters_json (pipeline.cpp:252-265)."""
    return {"text_field": c.text_field, "hash_count": c.hash_count, "bands": c.bands,
            "rows": c.rows, "shingle_len": c.shingle_len,
            "unit": "byte" if c.unit == ShingleUnit.BYTE else "codepoint",
            "threshold": _ratio_str(c.threshold), "bucket_scale": _ratio_str(c.bucket_scale),
            "min_chars": c.min_chars, "seed": c.seed}


def signature_file_name(ordinal: int, source_path: str) -> str:
    """pipeline.cpp:101-105: %05llu_<stem>.feds."""
    return f"{ordinal:05d}_{os.path.splitext(os.path.basename(source_path))[0]}.feds"


def header_template(c: RunConfig, bucket_count: int):
    """pipeline.cpp:107-118."""
    from .sigstore import SignatureFileHeader

    return SignatureFileHeader(c.hash_count, c.bands, c.rows, bucket_count, c.shingle_len,
                               c.unit, c.seed, _ratio(c.bucket_scale))


@dataclass
class HashStageOutput:
    manifest: CorpusManifest
    bucket_count: int = 0
    signature_files: list[str] = field(default_factory=list)
    total_signature_bytes: int = 0


@dataclass
class CompareStageOutput:
    buckets_per_pass: int = 0
    pass_count: int = 0
    candidate_pairs: int = 0
    emitted_pairs: int = 0
    gather_peak_bytes: int = 0
    pair_files: list[str] = field(default_factory=list)
    seconds: list[float] = field(default_factory=list)
    intervals: int = 1


def run_hash_stage(config: RunConfig, ctx: Context | None = None) -> HashStageOutput:
    """pipeline.cpp:269-339: ingest, sign every input file on the GPU (K1) into
    one .feds file each, write rejects.jsonl and run_manifest.json."""
    from .lsh import choose_bucket_count

    config.validate(need_workspace=True)
    os.makedirs(signatures_dir(config), exist_ok=True)
    os.makedirs(pairs_dir(config), exist_ok=True)
    manifest, rejects, cache = build_manifest_cached(config.inputs, config,
                                                     default_text_cache_bytes())
    if manifest.total_surviving == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG,
                               "no documents survive preprocessing; nothing to deduplicate")
    ctx = ctx or default_context()
    out = HashStageOutput(manifest)
    out.bucket_count = choose_bucket_count(manifest.total_surviving, config.bucket_scale)
    base = header_template(config, out.bucket_count)
    for i, fs in enumerate(manifest.files):
        path = signatures_dir(config) + "/" + signature_file_name(i, fs.path)
        packed = cache.pop(i, None)
        data, offsets, ids, _ = packed if packed is not None else surviving_packed(manifest, i,
                                                                                  config)
        if len(ids) != fs.surviving:
            raise _lib.PrerequisiteError(_lib.ND_ERR_PREREQ,
                                         f"'{fs.path}' yielded {len(ids)} documents, manifest "
                                         f"says {fs.surviving}")
        h = base.to_c()
        h.source_ordinal = i
        dp = data.ctypes.data_as(u8p) if data.size else C.cast(C.c_char_p(b"\0"), u8p)
        ctx.check(ctx.lib.nd_hash_file(ctx.h, dp, offsets.ctypes.data_as(u64p),
                                       ids.ctypes.data_as(u64p), len(ids), C.byref(h),
                                       path.encode(), int(config.fsync_files)))
        out.signature_files.append(path)
        out.total_signature_bytes += os.path.getsize(path)
    _write_rejects(rejects_path(config), rejects)
    doc = {"format_version": 1, "config_hash": config.config_hash(),
           "parameters": _parameters(config), "bucket_count": out.bucket_count,
           "totals": {"records": manifest.total_records, "surviving": manifest.total_surviving,
                      "signature_bytes": out.total_signature_bytes},
           "files": [{"path": f.path, "records": f.records, "surviving": f.surviving,
                      "record_offset": f.record_offset,
                      "signature_file": os.path.basename(out.signature_files[i])}
                     for i, f in enumerate(manifest.files)]}
    _write_text(run_manifest_path(config), _dump2(doc), config.fsync_files)  # pipeline.cpp:335
    return out


def _load_json_artifact(path: str, stage_hint: str) -> dict:
    """pipeline.cpp:267-277."""
    if not os.path.exists(path):
        raise _lib.PrerequisiteError(_lib.ND_ERR_PREREQ,
                                     f"'{path}' is missing; run the {stage_hint} stage first")
    try:
        with open(path, "rb") as f:
            j = json.loads(f.read())
    except ValueError:
        j = None
    if not isinstance(j, dict):
        raise _lib.IoError(_lib.ND_ERR_IO, f"'{path}' is not valid JSON")
    return j


def _check_config_hash(artifact: dict, config: RunConfig, path: str) -> None:
    if artifact.get("config_hash", 0) != config.config_hash():
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, f"configuration changed since '{path}' was "
                                                   "written; rerun the earlier stages")


def _load_run_manifest(config: RunConfig) -> dict:
    """load_run_manifest (pipeline.cpp:356-378)."""
    path = run_manifest_path(config)
    doc = _load_json_artifact(path, "hash")
    _check_config_hash(doc, config, path)
    try:
        return {"bucket_count": int(doc["bucket_count"]),
                "total_records": int(doc["totals"]["records"]),
                "total_surviving": int(doc["totals"]["surviving"]),
                "total_signature_bytes": int(doc["totals"]["signature_bytes"]),
                "source_paths": [e["path"] for e in doc["files"]],
                "signature_files": [signatures_dir(config) + "/" + e["signature_file"]
                                    for e in doc["files"]]}
    except (KeyError, TypeError, ValueError):
        raise _lib.IoError(_lib.ND_ERR_IO, f"'{path}' is missing required fields")


def run_compare_stage(config: RunConfig, ctx: Context | None = None) -> CompareStageOutput:
    """pipeline.cpp:382-432: plans the gather passes, compares every cell on the
    GPU with all signature records resident in HBM, writes one pair file per
    worker and pass plus compare_stage.json."""
    from .corpus import expand_inputs
    from .sigstore import plan_gather

    config.validate(need_workspace=True)
    m = _load_run_manifest(config)
    if config.inputs:
        if sorted(expand_inputs(config.inputs)) != m["source_paths"]:
            raise _lib.PrerequisiteError(_lib.ND_ERR_PREREQ, "input files differ from the hashed "
                                                             "manifest; rerun the hash stage")
    if config.buckets_per_pass is not None and config.buckets_per_pass < 1:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "buckets-per-pass override must be at least 1")
    ctx = ctx or default_context()
    plan = plan_gather(m["total_signature_bytes"], m["bucket_count"], config.bands,
                       config.workers, config.memory_budget, config.buckets_per_pass)
    expected = header_template(config, m["bucket_count"]).to_c()
    paths = (C.c_char_p * max(1, len(m["signature_files"])))(
        *[p.encode() for p in m["signature_files"]])
    st = _lib.NdCompareStageStats()
    tn, td = _ratio(config.threshold)
    os.makedirs(pairs_dir(config), exist_ok=True)
    ctx.check(ctx.lib.nd_set_hbm_budget(ctx.h, config.hbm_budget))
    ctx.check(ctx.lib.nd_compare_stage(ctx.h, paths, len(m["signature_files"]), C.byref(expected),
                                       m["total_signature_bytes"], config.workers,
                                       config.memory_budget, config.buckets_per_pass or 0, tn, td,
                                       pairs_dir(config).encode(), int(config.fsync_files),
                                       C.byref(st)))
    names = sorted(pairs_dir(config) + f"/w{w}_p{p}.pairs"
                   for w, np_ in enumerate(plan.passes_per_worker) for p in range(np_))
    out = CompareStageOutput(st.buckets_per_pass, st.pass_count, st.candidate_pairs,
                             st.emitted_pairs, st.gather_peak_bytes, names, list(st.seconds),
                             st.intervals)
    doc = {"config_hash": config.config_hash(), "bucket_count": m["bucket_count"],
           "buckets_per_pass": out.buckets_per_pass, "pass_count": out.pass_count,
           "workers": config.workers, "memory_budget": config.memory_budget,
           "candidate_pairs": out.candidate_pairs, "emitted_pairs": out.emitted_pairs,
           "gather_peak_bytes": out.gather_peak_bytes,
           "pair_files": [os.path.basename(f) for f in names]}
    _write_text(compare_stage_path(config), _dump2(doc), config.fsync_files)  # pipeline.cpp:444
    return out


def run_union_stage(config: RunConfig, ctx: Context | None = None) -> DedupReport:
    """pipeline.cpp:434-508: merge the pair files (sort + distinct), union +
    components on the GPU, write groups.jsonl, removal.txt, summary.json."""
    config.validate(need_workspace=True)
    m = _load_run_manifest(config)
    spath = compare_stage_path(config)
    stage = _load_json_artifact(spath, "gather-compare")
    _check_config_hash(stage, config, spath)
    try:
        files = [pairs_dir(config) + "/" + str(n) for n in stage["pair_files"]]
    except (KeyError, TypeError):
        raise _lib.IoError(_lib.ND_ERR_IO, f"'{spath}' is missing required fields")
    ctx = ctx or default_context()
    paths = (C.c_char_p * max(1, len(files)))(*[p.encode() for p in files])
    stats = NdDedupStats()
    ctx.check(ctx.lib.nd_union_stage(ctx.h, paths, len(files), m["total_surviving"],
                                     m["total_records"], config.workspace.encode(),
                                     int(config.fsync_files), C.byref(stats)))
    return _fetch_report(ctx, stats)


def run_dedup(config: RunConfig, ctx: Context | None = None, timings: dict | None = None) -> DedupReport:
    """pipeline.cpp:510-532: hash -> gather-compare -> union, every artifact on
    disk exactly as the reference writes it; wall-clock per stage in
    timings.json."""
    import time

    t0 = time.perf_counter()
    run_hash_stage(config, ctx)
    t1 = time.perf_counter()
    cmp = run_compare_stage(config, ctx)
    t2 = time.perf_counter()
    rep = run_union_stage(config, ctx)
    t3 = time.perf_counter()
    rep.candidate_pairs = cmp.candidate_pairs
    rep.stats["candidate_pairs"] = cmp.candidate_pairs
    rep.stats["emitted_pairs"] = cmp.emitted_pairs
    t = {"workers": config.workers, "hash_seconds": t1 - t0, "compare_seconds": t2 - t1,
         "union_seconds": t3 - t2, "total_seconds": t3 - t0}
    _write_text(timings_path(config), _dump2(t))
    if timings is not None:
        timings.update(t)
    return rep


@dataclass
class BenchRow:
    workers: int
    timings: dict


def run_bench(config: RunConfig, worker_counts, ctx: Context | None = None) -> list[BenchRow]:
    """pipeline.cpp:587-613: one full run_dedup per worker count, each in its own
    sub-workspace (bench_w<N>), and bench.json with the stage times.  On the GPU
    the worker count only shapes the gather-pass plan (and so the pair files),
    never the report."""
    from dataclasses import replace

    if not worker_counts:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "bench needs at least one worker count")
    rows = []
    for w in worker_counts:
        sub = replace(config, workers=w or 1,
                      workspace=config.workspace + f"/bench_w{w or 1}")
        os.makedirs(sub.workspace, exist_ok=True)
        t = {}
        run_dedup(sub, ctx, timings=t)
        rows.append(BenchRow(sub.workers, t))
    os.makedirs(config.workspace, exist_ok=True)
    _write_text(config.workspace + "/bench.json",
                _dump2([{"workers": r.workers, "hash_seconds": r.timings["hash_seconds"],
                         "compare_seconds": r.timings["compare_seconds"],
                         "union_seconds": r.timings["union_seconds"],
                         "total_seconds": r.timings["total_seconds"]} for r in rows]))
    return rows
