// Internal declarations shared by the neardup_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_internal.hpp"
#include "neardup_b200.h"

namespace ndb {

#define ND_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::ndb::fail(ND_ERR_DEVICE, std::string(#call) + ": " + cudaGetErrorString(e_) +   \
                                     " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// every kernel launch site ends with ND_CHECK_LAUNCH(); it also counts launches
// (nd_launch_count) so benchmarks can report how many of our kernels ran.
extern std::atomic<uint64_t> g_launches;
#define ND_CHECK_LAUNCH()                                   \
  do {                                                      \
    ::ndb::g_launches.fetch_add(1, std::memory_order_relaxed); \
    ND_CUDA(cudaGetLastError());                            \
  } while (0)

// ---------------------------------------------------------------------------
// Device-side per-function constants for the rolling hash (see k_signature.cu).
// Struct-of-arrays, padded to Hp (a power of two >= 8) functions.
struct DevFamily {
  uint32_t* q = nullptr;     // base
  uint32_t* qln = nullptr;   // (p - q^L mod p) mod p
  uint32_t* m = nullptr;     // floor(2^40 / p)
  uint32_t* negp = nullptr;  // (uint32_t)(-p)
  uint32_t* c3 = nullptr;    // 0x4B000000 * p mod 2^32  (fq variant)
  float* qp = nullptr;       // fl(q / p)
  float* qlnp = nullptr;     // fl(QLn / p)
  float* c1e = nullptr;      // -2^23 * qp + 2^-5
  uint32_t H = 0;            // real hash count
  uint32_t Hp = 0;           // padded hash count
  uint32_t L = 0;
};

// Simple growable device scratch buffer.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* get(size_t want) {
    if (want > bytes) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      bytes = 0;
      size_t cap = want < 4096 ? 4096 : want + want / 8;
      ND_CUDA(cudaMalloc(&ptr, cap));
      bytes = cap;
    }
    return ptr;
  }
  template <class T>
  T* as(size_t count) {
    return static_cast<T*>(get(count * sizeof(T)));
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

struct PinnedBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* get(size_t want) {
    if (want > bytes) {
      if (ptr) cudaFreeHost(ptr);
      ptr = nullptr;
      bytes = 0;
      ND_CUDA(cudaMallocHost(&ptr, want));
      bytes = want;
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

// ---- kernels / launchers (k_*.cu) -----------------------------------------
// K1: signatures + band keys over device-resident packed text.
// Returns ND_ERR_SHORT through the flag buffer when a document has no window.
struct SigScratch {
  DevBuf seg_count, item_off, item_doc, flags, multi_docs, scan_tmp;
  void release() {
    for (DevBuf* b : {&seg_count, &item_off, &item_doc, &flags, &multi_docs, &scan_tmp}) b->release();
  }
};
// h_offsets: optional host copy of d_offsets; when given, planning happens on
// the host and the launch is fully asynchronous for single-item documents.
void launch_signatures(const DevFamily& fam, const uint8_t* d_bytes, const uint64_t* d_offsets,
                       uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                       uint32_t* d_band, SigScratch& scratch, cudaStream_t stream,
                       bool check_short, const uint64_t* h_offsets);

// State of the last dedup run held by a context (results stay on device
// until fetched).
struct DedupState {
  DevBuf sig, band, cell_count, cell_off, cell_docs, cand, pairs, pairs_tmp, labels, tmp, tmp2,
      sort_tmp, stats;
  std::vector<uint64_t> doc_ids;        // row -> doc id
  std::vector<uint64_t> pair_lo, pair_hi;
  std::vector<uint32_t> pair_m;
  std::vector<uint64_t> members, group_start;
  uint64_t documents = 0, distinct_pairs = 0;
  bool valid = false;
  void release() {
    for (DevBuf* b : {&sig, &band, &cell_count, &cell_off, &cell_docs, &cand, &pairs, &pairs_tmp,
                      &labels, &tmp, &tmp2, &sort_tmp, &stats})
      b->release();
  }
};

// exclusive scan of u64 counts (n entries) into out (n+1 entries, out[n] = total)
void scan_u64(const uint64_t* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp, cudaStream_t s);
void scan_u32_to_u64(const uint32_t* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp,
                     cudaStream_t s);

int sm_count();

}  // namespace ndb
