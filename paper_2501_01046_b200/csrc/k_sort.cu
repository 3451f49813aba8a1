// Stable LSD radix sort of (key, value) pairs on the device, 8-bit digits.
//
// Used for (1) grouping (cell, doc) records into LSH cells -- the GPU form of
// scan_gather (sigstore.cpp:228-286), stability keeps each cell's documents
// in ascending doc order exactly like the reference's file scan --, (2) the
// sort + unique of duplicate pairs (compare.cpp:77-84, pipeline.cpp:466-473)
// and (3) ordering component members into groups (dedup_graph.cpp:56-81).
//
// Per pass: k_upsweep (per-tile digit histogram) -> exclusive scan of the
// digit-major [256 x tiles] histogram -> k_downsweep (warp-level stable
// ranking with __match_any_sync, the tile staged in shared memory in digit
// order, then each digit's run written contiguously).  HBM-bound: 2 reads + 1 write of
// the records per pass.
#include "nd_internal.cuh"

namespace ndb {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;                         // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
constexpr int kRadix = 256;

template <class K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return static_cast<uint32_t>(k >> shift) & 0xFFu;
}

template <class K>
__global__ void __launch_bounds__(kSortThreads)
    k_upsweep(const K* __restrict__ keys, uint64_t n, int shift, uint32_t* __restrict__ hist,
              uint32_t tiles) {
  __shared__ uint32_t h[kRadix];
  for (int i = threadIdx.x; i < kRadix; i += kSortThreads) h[i] = 0;
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile;
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    uint64_t idx = base + static_cast<uint64_t>(r) * kSortThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[digit_of(keys[idx], shift)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
    hist[static_cast<uint64_t>(d) * tiles + blockIdx.x] = h[d];
}

// Tile layout for stability: warp w owns keys [base + w*256, base + w*256 + 256),
// consumed in 8 rounds of 32 consecutive keys.
template <class K, class V>
__global__ void __launch_bounds__(kSortThreads)
    k_downsweep(const K* __restrict__ keys_in, const V* __restrict__ vals_in, K* __restrict__ keys_out,
                V* __restrict__ vals_out, uint64_t n, int shift,
                const uint64_t* __restrict__ offsets, uint32_t tiles) {
  constexpr int kWarpsPerBlock = kSortThreads / 32;
  __shared__ uint32_t whist[kWarpsPerBlock][kRadix];
  __shared__ uint64_t base_off[kRadix];
  __shared__ uint32_t tile_cnt[kRadix], tile_start[kRadix];
  __shared__ K sk[kSortTile];
  __shared__ V sv[kSortTile];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kWarpsPerBlock * kRadix; i += kSortThreads)
    (&whist[0][0])[i] = 0;
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
    base_off[d] = offsets[static_cast<uint64_t>(d) * tiles + blockIdx.x];
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortTile + warp * (32 * kSortItems);
  const unsigned lt = (1u << lane) - 1u;
  K k[kSortItems];
  V v[kSortItems];
  uint32_t dg[kSortItems], rk[kSortItems];
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    uint64_t idx = base + r * 32 + lane;
    bool valid = idx < n;
    k[r] = valid ? keys_in[idx] : K(0);
    v[r] = valid ? vals_in[idx] : V(0);
    uint32_t d = valid ? digit_of(k[r], shift) : 0xFFFFFFFFu;  // invalid lanes form their own group
    dg[r] = d;
    unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    uint32_t before = valid ? whist[warp][d] : 0;
    rk[r] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && (peers & lt) == 0) whist[warp][d] = before + __popc(peers);  // group leader
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan across warps, per digit; tile digit totals
  for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < kWarpsPerBlock; ++w) {
      uint32_t c = whist[w][d];
      whist[w][d] = acc;
      acc += c;
    }
    tile_cnt[d] = acc;
  }
  __syncthreads();
  // exclusive scan of the tile's digit totals (one warp, 8 digits per lane)
  if (warp == 0) {
    uint32_t c[kRadix / 32], sum = 0;
#pragma unroll
    for (int q = 0; q < kRadix / 32; ++q) {
      c[q] = tile_cnt[lane * (kRadix / 32) + q];
      sum += c[q];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += t;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int q = 0; q < kRadix / 32; ++q) {
      tile_start[lane * (kRadix / 32) + q] = run;
      run += c[q];
    }
  }
  __syncthreads();
  // stage the tile in digit order, then write each digit's run contiguously
  // (consecutive threads -> consecutive addresses: coalesced stores)
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
    if (dg[r] == 0xFFFFFFFFu) continue;
    const uint32_t lp = tile_start[dg[r]] + whist[warp][dg[r]] + rk[r];
    sk[lp] = k[r];
    sv[lp] = v[r];
  }
  __syncthreads();
  const uint64_t tbase = static_cast<uint64_t>(blockIdx.x) * kSortTile;
  const uint32_t tn = n - tbase < kSortTile ? static_cast<uint32_t>(n - tbase) : kSortTile;
  for (uint32_t i = threadIdx.x; i < tn; i += kSortThreads) {
    const K key = sk[i];
    const uint32_t d = digit_of(key, shift);
    const uint64_t dst = base_off[d] + (i - tile_start[d]);
    keys_out[dst] = key;
    vals_out[dst] = sv[i];
  }
}

template <class K, class V>
void radix_sort_impl(K* keys, V* vals, uint64_t n, int key_bits, SortScratch& sc,
                     cudaStream_t s) {
  if (n <= 1 || key_bits <= 0) return;
  const uint32_t tiles = static_cast<uint32_t>((n + kSortTile - 1) / kSortTile);
  K* k_alt = sc.keys_alt.as<K>(n);
  V* v_alt = sc.vals_alt.as<V>(n);
  uint32_t* hist = sc.hist.as<uint32_t>(static_cast<uint64_t>(kRadix) * tiles);
  uint64_t* offs = sc.offs.as<uint64_t>(static_cast<uint64_t>(kRadix) * tiles + 1);
  K* src_k = keys;
  V* src_v = vals;
  K* dst_k = k_alt;
  V* dst_v = v_alt;
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
    k_upsweep<K><<<tiles, kSortThreads, 0, s>>>(src_k, n, shift, hist, tiles);
    ND_CHECK_LAUNCH();
    scan_u32_to_u64(hist, offs, static_cast<uint64_t>(kRadix) * tiles, sc.scan, s);
    k_downsweep<K, V><<<tiles, kSortThreads, 0, s>>>(src_k, src_v, dst_k, dst_v, n, shift, offs,
                                                     tiles);
    ND_CHECK_LAUNCH();
    std::swap(src_k, dst_k);
    std::swap(src_v, dst_v);
  }
  if (passes & 1) {  // result sits in the alternate buffers
    ND_CUDA(cudaMemcpyAsync(keys, src_k, n * sizeof(K), cudaMemcpyDeviceToDevice, s));
    ND_CUDA(cudaMemcpyAsync(vals, src_v, n * sizeof(V), cudaMemcpyDeviceToDevice, s));
  }
}

}  // namespace

void radix_sort_u32(uint32_t* keys, uint32_t* vals, uint64_t n, int key_bits, SortScratch& sc,
                    cudaStream_t s) {
  radix_sort_impl<uint32_t, uint32_t>(keys, vals, n, key_bits, sc, s);
}

void radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t n, int key_bits, SortScratch& sc,
                    cudaStream_t s) {
  radix_sort_impl<uint64_t, uint32_t>(keys, vals, n, key_bits, sc, s);
}

}  // namespace ndb
