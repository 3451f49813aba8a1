"""Clustering -- mirror of the reference's dedup_graph.hpp.

  UnionFind / union_pairs  dedup_graph.hpp:15-34 -> K4 connected components (GPU)
  DuplicateGroup           dedup_graph.hpp:36-39
  components               dedup_graph.hpp:43   (groups by representative = min member)
  DedupReport / emit_report dedup_graph.hpp:45-55
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import u32p, u64p
from .device import Context, default_context


@dataclass
class DuplicateGroup:
    representative: int
    members: list[int]


@dataclass
class DedupReport:
    groups: list[DuplicateGroup] = field(default_factory=list)
    near_duplicates: list[int] = field(default_factory=list)
    removals: list[int] = field(default_factory=list)
    total_documents: int = 0
    distinct_pairs: int = 0
    ratio: float = 0.0
    candidate_pairs: int | None = None
    stats: dict | None = None


class UnionFind:
    """Result of union_pairs: the connected components of the pair graph,
    computed on the device; doc ids are densely renumbered in ascending order
    (the reference renumbers in first-seen order, dedup_graph.cpp:9-20; the
    components are the same)."""

    def __init__(self, ids: np.ndarray, members: np.ndarray, group_start: np.ndarray):
        self._ids = ids
        self._members = members
        self._group_start = group_start

    def size(self) -> int:
        return int(len(self._ids))

    def index_of(self, doc_id: int):
        i = int(np.searchsorted(self._ids, doc_id))
        return i if i < len(self._ids) and int(self._ids[i]) == doc_id else None

    def doc_at(self, index: int) -> int:
        return int(self._ids[index])


def union_pairs(pairs, ctx: Context | None = None) -> UnionFind:
    """Connectivity = transitive closure of the pairs; order/repeats irrelevant."""
    ctx = ctx or default_context()
    lo = np.array([p.lo for p in pairs], np.uint64)
    hi = np.array([p.hi for p in pairs], np.uint64)
    ids = np.unique(np.concatenate([lo, hi])) if len(pairs) else np.zeros(0, np.uint64)
    if len(ids) >= 2**32:
        raise ValueError("too many distinct documents in pairs for the dense index")
    rl = np.searchsorted(ids, lo).astype(np.uint32)
    rh = np.searchsorted(ids, hi).astype(np.uint32)
    nm, ng = C.c_uint64(), C.c_uint64()
    ctx.check(ctx.lib.nd_union(ctx.h, rl.ctypes.data_as(u32p), rh.ctypes.data_as(u32p), len(rl),
                               len(ids), C.byref(nm), C.byref(ng)))
    members = np.empty(nm.value, np.uint32)
    gstart = np.empty(ng.value + 1, np.uint64)
    ctx.check(ctx.lib.nd_groups_fetch(ctx.h, members.ctypes.data_as(u32p),
                                      gstart.ctypes.data_as(u64p)))
    return UnionFind(ids, members, gstart)


def components(uf: UnionFind) -> list[DuplicateGroup]:
    """Groups with >= 2 members, rep = min member, members sorted, sorted by rep."""
    out = []
    ids, mem, gs = uf._ids, uf._members, uf._group_start
    for g in range(len(gs) - 1):
        m = [int(x) for x in ids[mem[int(gs[g]):int(gs[g + 1])]]]
        if len(m) >= 2:
            out.append(DuplicateGroup(m[0], m))
    return out


def emit_report(groups, total_documents: int, distinct_pairs: int) -> DedupReport:
    """dedup_graph.cpp:83-102."""
    near = sorted(d for g in groups for d in g.members)
    removals = sorted(d for g in groups for d in g.members if d != g.representative)
    ratio = len(near) / total_documents if total_documents > 0 else 0.0
    return DedupReport(list(groups), near, removals, total_documents, distinct_pairs, ratio)
