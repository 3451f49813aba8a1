"""CPU stand-ins for the per-rank device stages of
paper_2501_01046_b200.distributed (TEST INFRASTRUCTURE ONLY).

They let the multi-GPU protocol (all-gather of counts, owner split,
all-to-all of cell records, all-gather of signatures and edges, union) run
under the gloo backend on CPU.  Every compute step is the oracle
(oracle/oracle.c), so these tests check the exchange logic, not the kernels
(the kernels are checked against the same oracle by the -m gpu tests).
"""
from types import SimpleNamespace

import numpy as np
import torch

from oracle_bind import HashFn, Oracle
from paper_2501_01046_b200.dedup_graph import DedupReport, DuplicateGroup


class CpuStages:
    def __init__(self):
        self.device = torch.device("cpu")
        self.o = Oracle()

    def signatures(self, data, offsets, family, bands, rows, K):
        fns = (HashFn * family.hash_count).from_buffer_copy(bytes(family.functions))
        sig = self.o.signatures(np.ascontiguousarray(data, np.uint8),
                                np.ascontiguousarray(offsets, np.uint64), fns, family.shingle_len)
        band = self.o.band_ids(sig, bands, rows, K)
        return torch.from_numpy(sig.view(np.int32)), torch.from_numpy(band.view(np.int32))

    def cell_records(self, band, bands, K, doc_base):
        b = band.numpy().view(np.uint32)
        n = b.shape[0]
        keys = (np.arange(bands, dtype=np.uint64)[None, :] * K + b).reshape(-1)
        vals = np.repeat(np.arange(n, dtype=np.uint64) + doc_base, bands)
        order = np.argsort(keys, kind="stable")
        return (torch.from_numpy(keys[order].astype(np.int32)),
                torch.from_numpy(vals[order].astype(np.int32)))

    def compare(self, sig_all, keys, vals, key_limit, H, threshold):
        sig = sig_all.numpy().view(np.uint32)
        k = keys.numpy()
        v = vals.numpy().view(np.uint32)
        order = np.argsort(k, kind="stable")
        k, v = k[order], v[order]
        found, cand = set(), 0
        starts = np.flatnonzero(np.r_[True, k[1:] != k[:-1]])
        ends = np.r_[starts[1:], len(k)]
        for s, e in zip(starts, ends):
            n = e - s
            if n < 2:
                continue
            cand += n * (n - 1) // 2
            lo, hi, m = self.o.compare_cell(sig, v[s:e], threshold[0], threshold[1])
            found |= set(zip(lo.tolist(), hi.tolist(), m.tolist()))
        trip = sorted(found)
        t = lambda i: torch.tensor([x[i] for x in trip], dtype=torch.int32)
        return t(0), t(1), t(2), cand

    def union(self, lo, hi, m, nnodes):
        pairs = sorted(set(zip(lo.tolist(), hi.tolist())))
        lab = self.o.components(np.array([p[0] for p in pairs], np.uint32),
                                np.array([p[1] for p in pairs], np.uint32), nnodes)
        groups = {}
        for i, l in enumerate(lab.tolist()):
            if l != 0xFFFFFFFF:
                groups.setdefault(l, []).append(i)
        return SimpleNamespace(distinct_pairs=len(pairs), groups=groups, nnodes=nnodes)

    def report(self, st, fetch):
        groups = [DuplicateGroup(r, sorted(ms)) for r, ms in sorted(st.groups.items())]
        near = sorted(x for g in groups for x in g.members)
        rem = sorted(x for g in groups for x in g.members[1:])
        return DedupReport(groups, near, rem, st.nnodes, st.distinct_pairs,
                           len(near) / st.nnodes if st.nnodes else 0.0)
