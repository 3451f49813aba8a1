// Device helpers shared by the in-cell compare (k_compare.cu) and the global
// block join (k_gjoin.cu): the exact early-exit match count, pair emission,
// and block loads/equality.
#pragma once
#include "nd_internal.cuh"

namespace ndb {
namespace {

__device__ __forceinline__ uint32_t full_matches(const uint32_t* __restrict__ a,
                                                 const uint32_t* __restrict__ b, uint32_t H,
                                                 uint32_t allowed, bool& alive) {
  uint32_t matches = 0;
  alive = true;
  for (uint32_t h0 = 0; h0 < H; h0 += 32) {
    const uint32_t hi = min(H, h0 + 32);
    for (uint32_t h = h0; h < hi; ++h) matches += __ldg(a + h) == __ldg(b + h);
    if (hi - matches > allowed) {  // accepting count unreachable (oracle.cpp:81-92)
      alive = false;
      return matches;
    }
  }
  return matches;
}

__device__ __forceinline__ void emit(uint32_t ra, uint32_t rb, uint32_t m, int nb,
                                     uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_m,
                                     unsigned long long* __restrict__ count, uint64_t cap) {
  const uint32_t lo = min(ra, rb), hi = max(ra, rb);
  unsigned long long slot = atomicAdd(count, 1ull);
  if (slot < cap) {
    out_key[slot] = (static_cast<uint64_t>(lo) << nb) | hi;
    out_m[slot] = m;
  }
}

template <int BW>
__device__ __forceinline__ void load_block(const uint32_t* __restrict__ p, bool vec, uint32_t (&v)[BW]) {
  if constexpr (BW % 4 == 0) {
    if (vec) {
#pragma unroll
      for (int q = 0; q < BW / 4; ++q) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(p) + q);
        v[4 * q] = x.x;
        v[4 * q + 1] = x.y;
        v[4 * q + 2] = x.z;
        v[4 * q + 3] = x.w;
      }
      return;
    }
  }
#pragma unroll
  for (int t = 0; t < BW; ++t) v[t] = __ldg(p + t);
}

template <int BW>
__device__ __forceinline__ bool same_block(const uint32_t* __restrict__ a,
                                           const uint32_t* __restrict__ b, bool vec) {
  uint32_t x[BW], y[BW];
  load_block<BW>(a, vec, x);
  load_block<BW>(b, vec, y);
  bool eq = true;
#pragma unroll
  for (int t = 0; t < BW; ++t) eq &= x[t] == y[t];
  return eq;
}

}  // namespace
}  // namespace ndb
