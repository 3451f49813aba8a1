// K3g: the in-memory dedup's compare as one global block join.
//
// The reference compares every pair inside every LSH cell and keeps the pairs
// with m >= min_matches (compare_bucket, compare.cpp:24-67), then sorts and
// uniques them over all cells (compare_pass, compare.cpp:69-85).  Its output
// is therefore the set
//
//     { (a, b) : a and b share a cell (band j with bucket_a[j] == bucket_b[j])
//                and matches(a, b) >= min_matches }
//
// with each pair emitted once per shared cell (the emitted-pairs counter).
// The per-cell join (k_join_blocks) finds this set cell by cell, so every
// document's blocks are joined once per band.  K3g joins each block once for
// the whole corpus:
//
//  * pigeonhole: with A = H - min_matches allowed mismatches, NB = A + 1
//    disjoint blocks of BW positions; an accepted pair has a block with no
//    mismatch (the same argument as the per-cell join);
//  * block k, all n rows at once: a 32-bit fingerprint per (row, block)
//    (k_gj_fps, block-major), rows chained per table slot of the fingerprint
//    (k_gj_insert: one atomicExch per row into a table of >= n slots), and
//    each row walks the rows chained before it (k_gj_walk);
//  * a chained pair with equal fingerprints is checked at its FIRST
//    identical block only (block k identical, no block j < k identical), so
//    every pair is checked once; the check then requires a shared cell (the
//    band ids) and the reference's count with its early exit (oracle.cpp:81-92),
//    and adds the number of shared cells to the emitted-pairs counter.
//
// The cells themselves are only needed for the reference's counters
// (candidate pairs = sum n(n-1)/2, non-singleton cells, their records,
// pipeline.cpp:406-411): one histogram over band * K + bucket (k_cell_hist).
#include <algorithm>
#include <mutex>
#include <cstdlib>
#include <string>

#include "nd_internal.cuh"
#include "k_compare_util.cuh"

namespace ndb {
namespace {

constexpr uint32_t kNoRow = 0xFFFFFFFFu;

template <int BW>
__device__ __forceinline__ uint32_t gj_fp(const uint32_t (&v)[BW]) {
  // bijective per step (xor, odd multiply, xorshift): for BW = 1 equal
  // fingerprints mean equal values
  uint32_t h = 0x9E3779B9u;
#pragma unroll
  for (int t = 0; t < BW; ++t) {
    h = (h ^ v[t]) * 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
  }
  return h;
}

// fps[k * n + row] for k < NB: one thread per row, the row read once
template <int BW>
__global__ void k_gj_fps(const uint32_t* __restrict__ sig, uint64_t n, uint32_t H, uint32_t NB,
                         uint32_t* __restrict__ fps) {
  const bool vec = (H & 3) == 0;
  for (uint64_t row = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; row < n;
       row += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t* r = sig + row * H;
    for (uint32_t k = 0; k < NB; ++k) {
      uint32_t v[BW];
      load_block<BW>(r + static_cast<uint64_t>(k) * BW, vec, v);
      fps[static_cast<uint64_t>(k) * n + row] = gj_fp<BW>(v);
    }
  }
}

// chain row i into the slot of its fingerprint: table entries and links are
// (fingerprint << 32 | row) of the row chained before (kNoRow: end)
__global__ void k_gj_insert(const FpCol fc, uint64_t n, unsigned long long* __restrict__ table,
                            int tbits, unsigned long long* __restrict__ link) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t f = fc.get(i);
  const uint32_t slot = (f * 0x9E3779B1u) >> (32 - tbits);
  link[i] = atomicExch(&table[slot], (static_cast<unsigned long long>(f) << 32) | i);
}

template <int BW>
__device__ __noinline__ void gj_check(const SigView& sv, const SigView& bv, uint32_t d,
                                      uint32_t e, uint32_t k, uint32_t min_match, int nb,
                                      uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_m,
                                      unsigned long long* __restrict__ count, uint64_t cap,
                                      unsigned long long* __restrict__ emitted) {
  const uint32_t H = sv.H, B = bv.H;
  const bool vec = (H & 3) == 0;
  const uint32_t* a = sv.row(d);
  const uint32_t* b = sv.row(e);
  if (!same_block<BW>(a + k * BW, b + k * BW, vec)) return;  // fingerprint collision
  for (uint32_t j = 0; j < k; ++j)
    if (same_block<BW>(a + j * BW, b + j * BW, vec)) return;  // checked at block j
  const uint32_t* ba = bv.row(d);
  const uint32_t* bb = bv.row(e);
  uint32_t shared = 0;
  for (uint32_t j = 0; j < B; ++j) shared += __ldg(ba + j) == __ldg(bb + j);
  if (shared == 0) return;  // no common cell: the reference never compares them
  bool alive;
  const uint32_t m = full_matches(a, b, H, H - min_match, alive);
  if (!alive || m < min_match) return;
  emit(d, e, m, nb, out_key, out_m, count, cap);
  atomicAdd(emitted, static_cast<unsigned long long>(shared));
}

template <int BW>
__global__ void k_gj_walk(const FpCol fc, uint64_t n, const unsigned long long* __restrict__ link,
                          const SigView sv, const SigView bv, uint32_t k, uint32_t min_match,
                          int nb, uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_m,
                          unsigned long long* __restrict__ count, uint64_t cap,
                          unsigned long long* __restrict__ emitted) {
  const uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (d >= n) return;
  const uint32_t f = fc.get(d);
  unsigned long long c = link[d];
  while (static_cast<uint32_t>(c) != kNoRow) {
    const uint32_t e = static_cast<uint32_t>(c);
    if (static_cast<uint32_t>(c >> 32) == f)
      gj_check<BW>(sv, bv, static_cast<uint32_t>(d), e, k, min_match, nb, out_key, out_m, count,
                   cap, emitted);
    c = __ldg(link + e);
  }
}

// (a band id >= K is not counted; bad != nullptr counts them)
__global__ void k_cell_hist(const uint32_t* __restrict__ band, uint64_t n, uint32_t B, uint32_t K,
                            uint32_t* __restrict__ cnt, unsigned int* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n * B;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t b = band[i];
    if (b < K) atomicAdd(&cnt[static_cast<uint64_t>(i % B) * K + b], 1u);
    else if (bad) atomicAdd(bad, 1u);
  }
}

// out[0] = sum n(n-1)/2, out[1] = cells with n >= 2, out[2] = their records;
// n = the sum over `parts` histograms (one per shard of a device group)
__global__ void k_cell_stats(const uint32_t* __restrict__ cnt0, const uint32_t* const* __restrict__ cnts,
                             uint32_t parts, uint64_t cells, unsigned long long* __restrict__ out) {
  unsigned long long p = 0, c = 0, r = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < cells;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long v = 0;
    if (cnt0) v = cnt0[i];
    else
      for (uint32_t q = 0; q < parts; ++q) v += cnts[q][i];
    if (v >= 2) {
      p += v * (v - 1) / 2;
      c += 1;
      r += v;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    p += __shfl_down_sync(0xFFFFFFFFu, p, o);
    c += __shfl_down_sync(0xFFFFFFFFu, c, o);
    r += __shfl_down_sync(0xFFFFFFFFu, r, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, p);
    atomicAdd(out + 1, c);
    atomicAdd(out + 2, r);
  }
}

template <int BW>
void gj_blocks(GJoin& g, const FpCols& fc, const SigView& sv, const SigView& bv, uint64_t n,
               const std::vector<uint32_t>& blocks, uint32_t mm, int nb, uint64_t* out_key,
               uint32_t* out_m, unsigned long long* count, uint64_t cap,
               unsigned long long* emitted, cudaStream_t s) {
  const unsigned tb = 256;
  const unsigned grid = static_cast<unsigned>((n + tb - 1) / tb);
  for (uint32_t k : blocks) {
    FpCol col;
    col.base = fc.base0 ? fc.base0 + static_cast<uint64_t>(k) * n : nullptr;
    col.bases = fc.bases;
    col.row_base = fc.row_base;
    col.world = fc.world;
    col.k = k;
    ND_CUDA(cudaMemsetAsync(g.table, 0xFF, (uint64_t{1} << g.tbits) * 8, s));
    k_gj_insert<<<grid, tb, 0, s>>>(col, n, g.table, g.tbits, g.link);
    ND_CHECK_LAUNCH();
    k_gj_walk<BW><<<grid, tb, 0, s>>>(col, n, g.link, sv, bv, k, mm, nb, out_key, out_m, count,
                                      cap, emitted);
    ND_CHECK_LAUNCH();
  }
}

template <int BW>
void gj_fps_launch(const uint32_t* sig, uint64_t n, uint32_t H, uint32_t NB, uint32_t* fps,
                   cudaStream_t s) {
  const unsigned tb = 256;
  const uint64_t blocks = (n + tb - 1) / tb;
  k_gj_fps<BW><<<static_cast<unsigned>(std::min<uint64_t>(blocks, 64ull * sm_count())), tb, 0,
                 s>>>(sig, n, H, NB, fps);
  ND_CHECK_LAUNCH();
}

}  // namespace

// Free device memory for the budget decisions.  cudaMemGetInfo measured
// 0.1-125 ms per call on B200 (profiles/r2_dedup_e2e_variance.txt), so the
// value is cached per device and re-queried only when a decision is within a
// factor of `margin` of the cached limit (a decision far from the limit does
// not depend on the exact figure; nd_set_hbm_budget overrides the budget).
uint64_t device_free_bytes(uint64_t need, uint64_t num, uint64_t den) {
  static std::mutex mu;
  static uint64_t cached[64] = {};
  int dev = 0;
  ND_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  uint64_t& c = cached[dev & 63];
  // usable = c * num / den; re-query unless need < usable / 2
  if (c == 0 || need >= c / den * num / 2) {
    size_t free_b = 0, total_b = 0;
    ND_CUDA(cudaMemGetInfo(&free_b, &total_b));
    c = free_b;
  }
  return c;
}

bool global_join_eligible(uint64_t n, uint32_t H, uint32_t B, uint32_t K, uint32_t mm) {
  const char* e = getenv("ND_K3");  // "cells": the per-cell join for every dedup
  if (e && std::string(e) == "cells") return false;
  if (n >= kNoRow || static_cast<uint64_t>(B) * K > (uint64_t{1} << 30)) return false;
  uint32_t NB = 0;
  int BW = 1;
  if (mm <= H) join_block_shape(H, mm, &NB, &BW);
  if (NB > kGJoinMaxBlocks) return false;
  // fingerprints + links + table must fit next to what is already resident
  const uint64_t need = n * (4ull * NB + 8) + (uint64_t{8} << std::max(10, bits_for(n))) +
                        4ull * B * K;
  return need < device_free_bytes(need, 8, 10) / 10 * 8;
}

void gj_cell_hist(GJoin& g, const uint32_t* band, uint64_t n, uint32_t B, uint32_t K,
                  cudaStream_t s, unsigned int* bad) {
  const uint64_t cells = static_cast<uint64_t>(B) * K;
  uint32_t* cnt = g.cnt.as<uint32_t>(cells + 1);
  ND_CUDA(cudaMemsetAsync(cnt, 0, cells * 4, s));
  if (n) {
    k_cell_hist<<<8 * sm_count(), 256, 0, s>>>(band, n, B, K, cnt, bad);
    ND_CHECK_LAUNCH();
  }
}

void gj_reset(GJoin& g, cudaStream_t s) {
  g.acc_d = reinterpret_cast<unsigned long long*>(g.acc.as<uint64_t>(4));
  ND_CUDA(cudaMemsetAsync(g.acc_d, 0, 4 * sizeof(uint64_t), s));
}

void gj_cell_stats(GJoin& g, const uint32_t* const* d_cnts, uint32_t parts, uint64_t cells,
                   cudaStream_t s) {
  k_cell_stats<<<8 * sm_count(), 256, 0, s>>>(nullptr, d_cnts, parts, cells, g.acc_d);
  ND_CHECK_LAUNCH();
}

void gj_cell_counts(GJoin& g, const uint32_t* band, uint64_t n, uint32_t B, uint32_t K,
                    cudaStream_t s) {
  gj_reset(g, s);
  gj_cell_hist(g, band, n, B, K, s);
  k_cell_stats<<<8 * sm_count(), 256, 0, s>>>(static_cast<const uint32_t*>(g.cnt.ptr), nullptr, 1,
                                              static_cast<uint64_t>(B) * K, g.acc_d);
  ND_CHECK_LAUNCH();
}

void gj_fps(const uint32_t* sig, uint64_t n, uint32_t H, uint32_t mm, uint32_t* fps,
            cudaStream_t s) {
  uint32_t NB = 0;
  int BW = 1;
  if (mm <= H) join_block_shape(H, mm, &NB, &BW);
  if (!n || !NB) return;
  switch (BW) {
    case 8: gj_fps_launch<8>(sig, n, H, NB, fps, s); break;
    case 4: gj_fps_launch<4>(sig, n, H, NB, fps, s); break;
    case 2: gj_fps_launch<2>(sig, n, H, NB, fps, s); break;
    default: gj_fps_launch<1>(sig, n, H, NB, fps, s);
  }
}

void gj_join(GJoin& g, const FpCols& fc, const SigView& sv, const SigView& bv, uint64_t n,
             uint32_t mm, const std::vector<uint32_t>& blocks, int nb, uint64_t* out_key,
             uint32_t* out_m, unsigned long long* count, uint64_t cap, cudaStream_t s) {
  const uint32_t H = sv.H;
  uint32_t NB = 0;
  int BW = 1;
  if (mm <= H) join_block_shape(H, mm, &NB, &BW);
  ND_CUDA(cudaMemsetAsync(g.acc_d + 3, 0, sizeof(uint64_t), s));
  if (n < 2 || NB == 0 || blocks.empty()) return;
  g.tbits = std::max(10, bits_for(n - 1));
  g.table = reinterpret_cast<unsigned long long*>(g.table_buf.as<uint64_t>(uint64_t{1} << g.tbits));
  g.link = reinterpret_cast<unsigned long long*>(g.link_buf.as<uint64_t>(n));
  unsigned long long* emitted = g.acc_d + 3;
  switch (BW) {
    case 8: gj_blocks<8>(g, fc, sv, bv, n, blocks, mm, nb, out_key, out_m, count, cap, emitted, s); break;
    case 4: gj_blocks<4>(g, fc, sv, bv, n, blocks, mm, nb, out_key, out_m, count, cap, emitted, s); break;
    case 2: gj_blocks<2>(g, fc, sv, bv, n, blocks, mm, nb, out_key, out_m, count, cap, emitted, s); break;
    default: gj_blocks<1>(g, fc, sv, bv, n, blocks, mm, nb, out_key, out_m, count, cap, emitted, s);
  }
}

void gj_pairs(GJoin& g, const uint32_t* sig, const uint32_t* band, uint64_t n, uint32_t H,
              uint32_t B, uint32_t mm, int nb, uint64_t* out_key, uint32_t* out_m,
              unsigned long long* count, uint64_t cap, cudaStream_t s) {
  uint32_t NB = 0;
  int BW = 1;
  if (mm <= H) join_block_shape(H, mm, &NB, &BW);
  if (n < 2 || NB == 0) {
    ND_CUDA(cudaMemsetAsync(g.acc_d + 3, 0, sizeof(uint64_t), s));
    return;
  }
  g.fps = g.fps_buf.as<uint32_t>(n * NB);
  gj_fps(sig, n, H, mm, g.fps, s);
  FpCols fc;
  fc.base0 = g.fps;
  std::vector<uint32_t> blocks(NB);
  for (uint32_t k = 0; k < NB; ++k) blocks[k] = k;
  gj_join(g, fc, SigView(sig, H), SigView(band, B), n, mm, blocks, nb, out_key, out_m, count, cap,
          s);
}

GJoinCounts gj_read(GJoin& g, cudaStream_t s) {
  uint64_t h[4];
  ND_CUDA(cudaMemcpyAsync(h, g.acc_d, sizeof h, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  return GJoinCounts{h[0], h[1], h[2], h[3]};
}

}  // namespace ndb
