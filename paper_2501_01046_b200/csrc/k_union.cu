// K4: distinct pairs and connected components.
//
// Distinct pairs: the packed (lo << nb | hi) keys are radix-sorted and the
// first of every run kept -- compare_pass's sort + unique (compare.cpp:77-84)
// and the union stage's merge (pipeline.cpp:466-473) in one pass.
//
// Components: replaces UnionFind/union_pairs/components
// (dedup_graph.cpp:9-81).  Hook-and-compress over the edge list:
//   hook:      for every edge, r_u = find(u), r_v = find(v); if different,
//              atomicMin(parent[max(r_u, r_v)], min(r_u, r_v))
//   compress:  parent[i] = find(i) for every node
// until no hook changes anything.  Hooks only ever point a root at a smaller
// root of the same component, so the surviving root is the component's
// minimum node -- the reference's representative (the minimum member,
// dedup_graph.cpp:62-66).  Members are then ordered by (root, node) with one
// radix sort, which is exactly "groups sorted by representative, members
// ascending" (dedup_graph.cpp:74-81).
#include "nd_internal.cuh"

namespace ndb {
namespace {

inline unsigned blocks_for(uint64_t n, unsigned tb) { return static_cast<unsigned>((n + tb - 1) / tb); }

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = static_cast<uint32_t>(i);
}

__global__ void k_first_of_run(const uint64_t* __restrict__ keys, uint64_t m,
                               uint32_t* __restrict__ flag) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < m) flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void k_compact_pairs(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                const uint32_t* __restrict__ flag, const uint64_t* __restrict__ idx,
                                uint64_t m, int nb, uint32_t* __restrict__ lo,
                                uint32_t* __restrict__ hi, uint32_t* __restrict__ mc) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= m || !flag[i]) return;
  uint64_t o = idx[i];
  const uint64_t mask = (nb >= 64) ? ~0ull : ((1ull << nb) - 1);
  lo[o] = static_cast<uint32_t>(keys[i] >> nb);
  hi[o] = static_cast<uint32_t>(keys[i] & mask);
  mc[o] = vals[i];
}

__device__ __forceinline__ uint32_t find_root(uint32_t* parent, uint32_t x) {
  uint32_t p = parent[x];
  while (p != x) {  // path halving; races only ever shorten paths
    uint32_t g = parent[p];
    if (g != p) parent[x] = g;
    x = p;
    p = g;
  }
  return x;
}

__global__ void k_hook(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi, uint64_t e,
                       uint32_t* parent, uint32_t* __restrict__ changed) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= e) return;
  uint32_t a = find_root(parent, lo[i]);
  uint32_t b = find_root(parent, hi[i]);
  if (a == b) return;
  uint32_t big = max(a, b), small = min(a, b);
  uint32_t old = atomicMin(&parent[big], small);
  if (old != small) *changed = 1u;
}

__global__ void k_compress(uint32_t* parent, uint64_t n) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) parent[i] = find_root(parent, static_cast<uint32_t>(i));
}

__global__ void k_mark(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi, uint64_t e,
                       uint32_t* __restrict__ in_edge) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= e) return;
  // a self-loop record (possible in a hand-written .pairs file) makes no
  // group by itself: components() keeps groups of 2+ (dedup_graph.cpp:70)
  if (lo[i] == hi[i]) return;
  in_edge[lo[i]] = 1u;
  in_edge[hi[i]] = 1u;
}

__global__ void k_member_keys(const uint32_t* __restrict__ in_edge, const uint64_t* __restrict__ idx,
                              const uint32_t* __restrict__ parent, uint64_t n, int nb,
                              uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                              uint32_t* __restrict__ removal_flag) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !in_edge[i]) return;
  uint64_t o = idx[i];
  keys[o] = (static_cast<uint64_t>(parent[i]) << nb) | i;
  vals[o] = static_cast<uint32_t>(i);
  removal_flag[o] = parent[i] != i ? 1u : 0u;
}

__global__ void k_group_heads(const uint64_t* __restrict__ keys, uint64_t m, int nb,
                              uint32_t* __restrict__ flag) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < m) flag[i] = (i == 0 || (keys[i] >> nb) != (keys[i - 1] >> nb)) ? 1u : 0u;
}

__global__ void k_group_starts(const uint32_t* __restrict__ flag, const uint64_t* __restrict__ idx,
                               uint64_t m, uint64_t* __restrict__ start) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  if (flag[i]) start[idx[i]] = i;
  if (i == 0) start[idx[m]] = m;
}

__global__ void k_compact_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ flag,
                              const uint64_t* __restrict__ idx, uint64_t m, uint32_t* __restrict__ dst) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < m && flag[i]) dst[idx[i]] = src[i];
}

__global__ void k_pack_pairs(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi,
                             const uint32_t* __restrict__ m, uint64_t count, int nb,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  uint32_t a = min(lo[i], hi[i]), b = max(lo[i], hi[i]);
  keys[i] = (static_cast<uint64_t>(a) << nb) | b;
  vals[i] = m ? m[i] : 0u;
}

}  // namespace

void pack_pairs(PairSet& ps, const uint32_t* lo, const uint32_t* hi, const uint32_t* m,
                uint64_t count, cudaStream_t s) {
  ps.cap = count ? count : 1;
  ps.keys = ps.dkeys.as<uint64_t>(ps.cap);
  ps.vals = ps.dvals.as<uint32_t>(ps.cap);
  ps.count = count;
  if (count) {
    k_pack_pairs<<<blocks_for(count, 256), 256, 0, s>>>(lo, hi, m, count, ps.nb, ps.keys, ps.vals);
    ND_CHECK_LAUNCH();
  }
}

uint64_t unique_pairs(PairSet& ps, cudaStream_t s) {
  const unsigned tb = 256;
  const uint64_t m = ps.count;
  ps.distinct = 0;
  if (m == 0) return 0;
  radix_sort_u64(ps.keys, ps.vals, m, 2 * ps.nb, ps.sort, s);
  uint32_t* flag = ps.flag.as<uint32_t>(m);
  uint64_t* idx = ps.idx.as<uint64_t>(m + 1);
  k_first_of_run<<<blocks_for(m, tb), tb, 0, s>>>(ps.keys, m, flag);
  ND_CHECK_LAUNCH();
  scan_u32_to_u64(flag, idx, m, ps.scan, s);
  uint64_t d = 0;
  ND_CUDA(cudaMemcpyAsync(&d, idx + m, sizeof d, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  ps.lo = ps.dlo.as<uint32_t>(d);
  ps.hi = ps.dhi.as<uint32_t>(d);
  ps.mc = ps.dmc.as<uint32_t>(d);
  k_compact_pairs<<<blocks_for(m, tb), tb, 0, s>>>(ps.keys, ps.vals, flag, idx, m, ps.nb, ps.lo,
                                                   ps.hi, ps.mc);
  ND_CHECK_LAUNCH();
  ps.distinct = d;
  return d;
}

void components(GroupSet& gs, const uint32_t* lo, const uint32_t* hi, uint64_t e, uint64_t n,
                cudaStream_t s) {
  const unsigned tb = 256;
  gs.members = 0;
  gs.groups = 0;
  gs.removals = 0;
  if (e == 0 || n == 0) return;
  uint32_t* parent = gs.parent.as<uint32_t>(n);
  uint32_t* changed = gs.flagbuf.as<uint32_t>(1);
  k_iota<<<blocks_for(n, tb), tb, 0, s>>>(parent, n);
  ND_CHECK_LAUNCH();
  for (int it = 0; it < 4096; ++it) {
    uint32_t h = 0;
    ND_CUDA(cudaMemsetAsync(changed, 0, sizeof(uint32_t), s));
    k_hook<<<blocks_for(e, tb), tb, 0, s>>>(lo, hi, e, parent, changed);
    ND_CHECK_LAUNCH();
    k_compress<<<blocks_for(n, tb), tb, 0, s>>>(parent, n);
    ND_CHECK_LAUNCH();
    ND_CUDA(cudaMemcpyAsync(&h, changed, sizeof h, cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
    if (!h) break;
    if (it == 4095) fail(ND_ERR_INTERNAL, "connected components did not converge");
  }
  // members: nodes that appear in any pair (UnionFind only holds those,
  // dedup_graph.cpp:9-20), ordered by (root, node)
  uint32_t* in_edge = gs.in_edge.as<uint32_t>(n);
  ND_CUDA(cudaMemsetAsync(in_edge, 0, n * sizeof(uint32_t), s));
  k_mark<<<blocks_for(e, tb), tb, 0, s>>>(lo, hi, e, in_edge);
  ND_CHECK_LAUNCH();
  uint64_t* idx = gs.idx.as<uint64_t>(n + 1);
  scan_u32_to_u64(in_edge, idx, n, gs.scan, s);
  uint64_t mcount = 0;
  ND_CUDA(cudaMemcpyAsync(&mcount, idx + n, sizeof mcount, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  const int nb = bits_for(n - 1) ? bits_for(n - 1) : 1;
  uint64_t* keys = gs.keys.as<uint64_t>(mcount);
  uint32_t* vals = gs.vals.as<uint32_t>(mcount);
  uint32_t* rflag = gs.rflag.as<uint32_t>(mcount);
  k_member_keys<<<blocks_for(n, tb), tb, 0, s>>>(in_edge, idx, parent, n, nb, keys, vals, rflag);
  ND_CHECK_LAUNCH();
  // near_duplicates (dedup_graph.cpp:89-95) are the members in node order,
  // which is the order k_member_keys wrote them in; keep a copy before sorting
  gs.near = gs.dnear.as<uint32_t>(mcount);
  ND_CUDA(cudaMemcpyAsync(gs.near, vals, mcount * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  // removals = members that are not their component's representative, node order
  uint64_t* ridx = gs.ridx.as<uint64_t>(mcount + 1);
  scan_u32_to_u64(rflag, ridx, mcount, gs.scan, s);
  radix_sort_u64(keys, vals, mcount, 2 * nb, gs.sort, s);
  uint32_t* gflag = gs.gflag.as<uint32_t>(mcount);
  uint64_t* gidx = gs.gidx.as<uint64_t>(mcount + 1);
  k_group_heads<<<blocks_for(mcount, tb), tb, 0, s>>>(keys, mcount, nb, gflag);
  ND_CHECK_LAUNCH();
  scan_u32_to_u64(gflag, gidx, mcount, gs.scan, s);
  uint64_t tail[2];
  ND_CUDA(cudaMemcpyAsync(&tail[0], gidx + mcount, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaMemcpyAsync(&tail[1], ridx + mcount, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  gs.groups = tail[0];
  gs.removals = tail[1];
  gs.group_start = gs.gstart.as<uint64_t>(gs.groups + 1);
  k_group_starts<<<blocks_for(mcount, tb), tb, 0, s>>>(gflag, gidx, mcount, gs.group_start);
  ND_CHECK_LAUNCH();
  gs.removal = gs.drem.as<uint32_t>(gs.removals);
  k_compact_u32<<<blocks_for(mcount, tb), tb, 0, s>>>(gs.near, rflag, ridx, mcount, gs.removal);
  ND_CHECK_LAUNCH();
  gs.member_rows = vals;
  gs.members = mcount;
}

}  // namespace ndb
