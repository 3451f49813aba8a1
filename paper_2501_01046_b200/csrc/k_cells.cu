// K2: LSH cell grouping -- the GPU form of scan_gather (sigstore.cpp:228-286).
//
// Every (document, band) pair becomes a record (cell = band*K + bucket, row).
// Records are emitted document-major, so a STABLE sort by cell leaves each
// cell's rows in ascending document order, exactly the order the reference's
// sequential scan produces (and enforces, sigstore.cpp:259-262).  Runs of
// equal cells are then compacted, singleton cells dropped
// (sigstore.cpp:271-284), and the work list for K3 is built: one item per
// (cell, tile of kCmpRows rows).  candidate_pairs = sum n(n-1)/2 is the
// reference's own counter (pipeline.cpp:406-411).
#include <cstdlib>

#include "nd_internal.cuh"

namespace ndb {
namespace {

__global__ void k_records(const uint32_t* __restrict__ band, uint64_t n, uint32_t bands,
                          uint32_t K, uint32_t doc_base, uint32_t* __restrict__ keys,
                          uint32_t* __restrict__ vals) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n * bands) return;
  uint32_t j = static_cast<uint32_t>(i % bands);
  keys[i] = j * K + band[i];
  vals[i] = doc_base + static_cast<uint32_t>(i / bands);
}

__global__ void k_heads(const uint32_t* __restrict__ keys, uint64_t m, uint32_t* __restrict__ flag) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void k_run_starts(const uint32_t* __restrict__ flag, const uint64_t* __restrict__ run_idx,
                             uint64_t m, uint64_t* __restrict__ run_start) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  if (flag[i]) run_start[run_idx[i]] = i;
  if (i == 0) run_start[run_idx[m]] = m;  // sentinel: run_idx[m] == number of runs
}

__global__ void k_run_keep(const uint64_t* __restrict__ run_start, uint64_t runs,
                           uint32_t* __restrict__ keep) {
  uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (r >= runs) return;
  keep[r] = run_start[r + 1] - run_start[r] >= 2 ? 1u : 0u;
}

__global__ void k_cells_compact(const uint64_t* __restrict__ run_start, const uint32_t* __restrict__ keep,
                                const uint64_t* __restrict__ keep_idx, uint64_t runs,
                                const uint32_t* __restrict__ sorted_keys, uint32_t tile_rows,
                                uint64_t* __restrict__ cell_start, uint32_t* __restrict__ cell_len,
                                uint32_t* __restrict__ cell_key, uint64_t* __restrict__ cell_pairs,
                                uint32_t* __restrict__ cell_tiles, uint32_t join_max,
                                unsigned long long* __restrict__ max_len) {
  // max_len[0]: largest cell; max_len[1]: sum of n over the kept cells
  uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (r >= runs || !keep[r]) return;
  uint64_t c = keep_idx[r];
  uint64_t s = run_start[r];
  uint64_t len = run_start[r + 1] - s;
  cell_start[c] = s;
  cell_len[c] = static_cast<uint32_t>(len);
  cell_key[c] = sorted_keys[s];
  cell_pairs[c] = len * (len - 1) / 2;
  // cells the hash join takes (k_join) need no all-pairs tiles
  cell_tiles[c] = len > join_max ? static_cast<uint32_t>((len + tile_rows - 1) / tile_rows) : 0u;
  atomicMax(max_len, static_cast<unsigned long long>(len));
  atomicAdd(max_len + 1, static_cast<unsigned long long>(len));
}

__global__ void k_all_pairs_tiles(const uint32_t* __restrict__ cell_len, uint64_t cells,
                                  uint32_t tile_rows, uint32_t* __restrict__ cell_tiles) {
  uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (c >= cells) return;
  cell_tiles[c] = (cell_len[c] + tile_rows - 1) / tile_rows;
}

__global__ void k_item_cells(const uint64_t* __restrict__ item_off, uint64_t cells,
                             uint32_t* __restrict__ item_cell) {
  uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (c >= cells) return;
  for (uint64_t i = item_off[c]; i < item_off[c + 1]; ++i) item_cell[i] = static_cast<uint32_t>(c);
}

inline unsigned blocks_for(uint64_t n, unsigned tb) { return static_cast<unsigned>((n + tb - 1) / tb); }

}  // namespace

int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

void build_cells_from_records(CellSet& cs, uint32_t* keys, uint32_t* vals, uint64_t m,
                              uint64_t key_limit, uint32_t tile_rows, cudaStream_t s) {
  const unsigned tb = 256;
  {  // ND_JOIN=0 routes every cell through the all-pairs kernel (A/B tests)
    const char* j = getenv("ND_JOIN");
    cs.join_enabled = !(j && j[0] == '0');
  }
  cs.records = m;
  cs.tile_rows = tile_rows;
  cs.ncells = 0;
  cs.cell_records = 0;
  cs.items = 0;
  cs.candidate_pairs = 0;
  if (m == 0) return;
  radix_sort_u32(keys, vals, m, bits_for(key_limit ? key_limit - 1 : 0xFFFFFFFFu), cs.sort, s);
  cs.sorted_rows = vals;
  uint32_t* flag = cs.flag.as<uint32_t>(m);
  uint64_t* run_idx = cs.run_idx.as<uint64_t>(m + 1);
  k_heads<<<blocks_for(m, tb), tb, 0, s>>>(keys, m, flag);
  ND_CHECK_LAUNCH();
  scan_u32_to_u64(flag, run_idx, m, cs.scan, s);
  uint64_t runs = 0;
  ND_CUDA(cudaMemcpyAsync(&runs, run_idx + m, sizeof runs, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  uint64_t* run_start = cs.run_start.as<uint64_t>(runs + 1);
  k_run_starts<<<blocks_for(m, tb), tb, 0, s>>>(flag, run_idx, m, run_start);
  ND_CHECK_LAUNCH();
  uint32_t* keep = cs.flag.as<uint32_t>(m);  // reuse (runs <= m)
  k_run_keep<<<blocks_for(runs, tb), tb, 0, s>>>(run_start, runs, keep);
  ND_CHECK_LAUNCH();
  uint64_t* keep_idx = cs.run_idx.as<uint64_t>(m + 1);  // reuse
  scan_u32_to_u64(keep, keep_idx, runs, cs.scan, s);
  uint64_t cells = 0;
  ND_CUDA(cudaMemcpyAsync(&cells, keep_idx + runs, sizeof cells, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  cs.ncells = cells;
  if (cells == 0) return;
  cs.cell_start = cs.cstart.as<uint64_t>(cells);
  cs.cell_len = cs.clen.as<uint32_t>(cells);
  cs.cell_key = cs.ckey.as<uint32_t>(cells);
  uint64_t* cpairs = cs.cpairs.as<uint64_t>(cells + 1);
  uint32_t* ctiles = cs.ctiles.as<uint32_t>(cells);
  unsigned long long* dmax = reinterpret_cast<unsigned long long*>(cs.maxbuf.as<uint64_t>(2));
  ND_CUDA(cudaMemsetAsync(dmax, 0, 2 * sizeof(uint64_t), s));
  k_cells_compact<<<blocks_for(runs, tb), tb, 0, s>>>(run_start, keep, keep_idx, runs, keys,
                                                      tile_rows, cs.cell_start, cs.cell_len,
                                                      cs.cell_key, cpairs, ctiles,
                                                      cs.join_enabled ? kJoinMax : 0u, dmax);
  ND_CHECK_LAUNCH();
  uint64_t* pair_off = cs.pair_off.as<uint64_t>(cells + 1);
  scan_u64(cpairs, pair_off, cells, cs.scan, s);
  cs.item_off = cs.ioff.as<uint64_t>(cells + 1);
  scan_u32_to_u64(ctiles, cs.item_off, cells, cs.scan, s);
  uint64_t tail[4];
  ND_CUDA(cudaMemcpyAsync(&tail[0], pair_off + cells, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaMemcpyAsync(&tail[1], cs.item_off + cells, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaMemcpyAsync(&tail[2], dmax, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  cs.candidate_pairs = tail[0];
  cs.items = tail[1];
  cs.max_len = cs.join_enabled ? tail[2] : 0;
  cs.cell_records = tail[3];
  cs.item_cell = cs.icell.as<uint32_t>(cs.items + 1);
  if (cs.items)
    k_item_cells<<<blocks_for(cells, tb), tb, 0, s>>>(cs.item_off, cells, cs.item_cell);
  ND_CHECK_LAUNCH();
}

// The hash joins cannot take this compare (launch_compare: P > kJoinMaxP):
// give every cell all-pairs tiles, so that no cell of <= kJoinMax documents
// is left without a kernel (every cell is compared, compare.cpp:24-67).
void cells_all_pairs_tiles(CellSet& cs, cudaStream_t s) {
  if (!cs.join_enabled || cs.ncells == 0) {
    cs.join_enabled = false;
    return;
  }
  const unsigned tb = 256;
  const uint64_t cells = cs.ncells;
  uint32_t* ctiles = cs.ctiles.as<uint32_t>(cells);
  k_all_pairs_tiles<<<blocks_for(cells, tb), tb, 0, s>>>(cs.cell_len, cells, cs.tile_rows, ctiles);
  ND_CHECK_LAUNCH();
  cs.item_off = cs.ioff.as<uint64_t>(cells + 1);
  scan_u32_to_u64(ctiles, cs.item_off, cells, cs.scan, s);
  uint64_t items = 0;
  ND_CUDA(cudaMemcpyAsync(&items, cs.item_off + cells, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  cs.items = items;
  cs.join_enabled = false;
  cs.max_len = 0;
  cs.item_cell = cs.icell.as<uint32_t>(cs.items + 1);
  if (cs.items) {
    k_item_cells<<<blocks_for(cells, tb), tb, 0, s>>>(cs.item_off, cells, cs.item_cell);
    ND_CHECK_LAUNCH();
  }
}

void make_records(const uint32_t* band, uint64_t n, uint32_t bands, uint32_t K, uint32_t doc_base,
                  uint32_t* keys, uint32_t* vals, cudaStream_t s) {
  const uint64_t m = n * bands;
  if (static_cast<uint64_t>(bands) * K > 0xFFFFFFFFull)
    fail(ND_ERR_CONFIG, "bands * bucket_count exceeds 2^32 cells");
  if (m) {
    k_records<<<blocks_for(m, 256), 256, 0, s>>>(band, n, bands, K, doc_base, keys, vals);
    ND_CHECK_LAUNCH();
  }
}

void build_cells_from_bands(CellSet& cs, const uint32_t* band, uint64_t n, uint32_t bands,
                            uint32_t K, uint32_t tile_rows, cudaStream_t s) {
  const uint64_t m = n * bands;
  uint32_t* keys = cs.rec_keys.as<uint32_t>(m);
  uint32_t* vals = cs.rec_vals.as<uint32_t>(m);
  make_records(band, n, bands, K, 0, keys, vals, s);
  build_cells_from_records(cs, keys, vals, m, static_cast<uint64_t>(bands) * K, tile_rows, s);
}

}  // namespace ndb
