// Exclusive prefix sums (reduce-then-scan, 3 launches), used to turn per-doc
// segment counts and per-cell histograms into offsets.  HBM-bound and small
// next to the hot kernels; tiles of 2048 elements per 256-thread block.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "nd_internal.cuh"

namespace ndb {
namespace {

constexpr int kThreads = 256;
constexpr int kPer = 8;
constexpr int kTile = kThreads * kPer;

template <class In>
__global__ void __launch_bounds__(kThreads) k_tile_sums(const In* __restrict__ in, uint64_t n,
                                                        uint64_t* __restrict__ sums) {
  uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  uint64_t acc = 0;
  for (int i = 0; i < kPer; ++i) {
    uint64_t idx = base + static_cast<uint64_t>(i) * kThreads + threadIdx.x;
    if (idx < n) acc += static_cast<uint64_t>(in[idx]);
  }
  using R = cub::BlockReduce<uint64_t, kThreads>;
  __shared__ typename R::TempStorage tmp;
  uint64_t total = R(tmp).Sum(acc);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// in-place exclusive scan of up to kTile entries by one block; writes total
template <class In>
__global__ void __launch_bounds__(kThreads) k_tile_scan(const In* __restrict__ in, uint64_t n,
                                                        const uint64_t* __restrict__ tile_prefix,
                                                        uint64_t* __restrict__ out) {
  uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  uint64_t v[kPer];
  // blocked arrangement: thread t owns [base + t*kPer, base + t*kPer + kPer)
  for (int i = 0; i < kPer; ++i) {
    uint64_t idx = base + static_cast<uint64_t>(threadIdx.x) * kPer + i;
    v[i] = idx < n ? static_cast<uint64_t>(in[idx]) : 0;
  }
  using S = cub::BlockScan<uint64_t, kThreads>;
  __shared__ typename S::TempStorage tmp;
  uint64_t block_total;
  S(tmp).ExclusiveSum(v, v, block_total);
  uint64_t pre = tile_prefix ? tile_prefix[blockIdx.x] : 0;
  for (int i = 0; i < kPer; ++i) {
    uint64_t idx = base + static_cast<uint64_t>(threadIdx.x) * kPer + i;
    if (idx < n) out[idx] = v[i] + pre;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = pre + block_total;
}

template <class In>
void scan_impl(const In* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp, cudaStream_t s) {
  if (n == 0) {
    ND_CUDA(cudaMemsetAsync(d_out, 0, sizeof(uint64_t), s));
    return;
  }
  // level sizes: n_0 = n, n_{i+1} = ceil(n_i / kTile) until a single tile
  std::vector<uint64_t> ns{n};
  while (ns.back() > static_cast<uint64_t>(kTile)) ns.push_back((ns.back() + kTile - 1) / kTile);
  const size_t levels = ns.size() - 1;  // number of tile-sum levels
  size_t words = 0;
  for (size_t i = 1; i < ns.size(); ++i) words += 2 * ns[i] + 1;
  uint64_t* pool = tmp.as<uint64_t>(words + 1);
  std::vector<uint64_t*> sums(levels), prefix(levels);
  for (size_t i = 0; i < levels; ++i) {
    sums[i] = pool;
    pool += ns[i + 1];
    prefix[i] = pool;
    pool += ns[i + 1] + 1;
  }
  // reduce down
  for (size_t i = 0; i < levels; ++i) {
    unsigned tiles = static_cast<unsigned>(ns[i + 1]);
    if (i == 0)
      k_tile_sums<In><<<tiles, kThreads, 0, s>>>(d_in, ns[0], sums[0]);
    else
      k_tile_sums<uint64_t><<<tiles, kThreads, 0, s>>>(sums[i - 1], ns[i], sums[i]);
    ND_CHECK_LAUNCH();
  }
  if (levels == 0) {
    k_tile_scan<In><<<1, kThreads, 0, s>>>(d_in, n, nullptr, d_out);
    ND_CHECK_LAUNCH();
    return;
  }
  // top level fits one tile
  k_tile_scan<uint64_t><<<1, kThreads, 0, s>>>(sums[levels - 1], ns[levels], nullptr,
                                                prefix[levels - 1]);
  ND_CHECK_LAUNCH();
  // scan up
  for (size_t i = levels; i-- > 0;) {
    unsigned tiles = static_cast<unsigned>(ns[i + 1]);
    if (i == 0)
      k_tile_scan<In><<<tiles, kThreads, 0, s>>>(d_in, ns[0], prefix[0], d_out);
    else
      k_tile_scan<uint64_t><<<tiles, kThreads, 0, s>>>(sums[i - 1], ns[i], prefix[i], prefix[i - 1]);
    ND_CHECK_LAUNCH();
  }
}

}  // namespace

void scan_u64(const uint64_t* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp, cudaStream_t s) {
  scan_impl<uint64_t>(d_in, d_out, n, tmp, s);
}

void scan_u32_to_u64(const uint32_t* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp,
                     cudaStream_t s) {
  scan_impl<uint32_t>(d_in, d_out, n, tmp, s);
}

}  // namespace ndb
