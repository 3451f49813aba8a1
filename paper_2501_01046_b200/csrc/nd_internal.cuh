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
  uint32_t* m45 = nullptr;   // floor(2^45 / p)  (codepoint units, "wide" variant)
  uint32_t* p = nullptr;     // modulus           ("exact" variant)
  unsigned long long* rf = nullptr;  // floor(2^64 / p) = reduce_factor (minhash.hpp:24)
  uint32_t H = 0;            // real hash count
  uint32_t Hp = 0;           // padded hash count
  uint32_t L = 0;
  uint32_t unit = 0;         // 0 = byte, 1 = codepoint (ShingleUnit, text.hpp:23-26);
                             // 2 = internal view of code points < 2^16 as u16 units
  void* jit = nullptr;        // K1j kernel specialised for this family (k1_jit.cpp), or null
  // codepoint family: K1j over 16-bit units (documents whose code points are
  // all < 2^16 and some >= 256), or null
  void* jit16 = nullptr;
  // codepoint family whose functions all lie in the byte fq domain: documents
  // whose code points are all < 256 run the byte kernels over narrowed units
  bool narrow_ok = false;
  // true when some function lies outside the domain the fast arithmetics are
  // proven for (byte fq: 2^21 <= p < 2^23, q < 2^16; codepoint wide:
  // 0x10FFFF < p < 2^23, q < 2^16): K1 then runs the 64-bit Barrett
  // reduction of the reference itself (minhash.cpp:61-67), exact for p < 2^31
  bool exact = false;
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
// Scratch for radix_sort_* (k_sort.cu).
struct SortScratch {
  DevBuf keys_alt, vals_alt, hist, offs, scan;
  void release() {
    for (DevBuf* b : {&keys_alt, &vals_alt, &hist, &offs, &scan}) b->release();
  }
};
struct SigScratch {
  DevBuf seg_count, item_off, item_doc, flags, multi_docs, scan_tmp, units, unit_off, unit_cnt,
      item_counter, order_keys, order_vals, units8, units16, wide, cls_cnt;
  SortScratch sort;  // K1j: items ordered by length
  void release() {
    for (DevBuf* b : {&seg_count, &item_off, &item_doc, &flags, &multi_docs, &scan_tmp, &units,
                      &unit_off, &unit_cnt, &item_counter, &order_keys, &order_vals, &units8,
                      &units16, &wide, &cls_cnt})
      b->release();
    sort.release();
  }
};
// K1j: family-specialised signature kernel (k1_jit.cpp)
bool k1_jit_eligible(const DevFamily& fam);
// uw: bytes per text unit (1, or 2 for code points < 2^16)
void* k1_jit_prepare(const nd_hash_fn* fns, uint32_t H, uint32_t L, int uw = 1);
double k1_jit_compile_seconds(const void* handle);
uint32_t k1_jit_passes(const void* handle);
std::string k1_jit_source(const nd_hash_fn* fns, uint32_t H, uint32_t L, int uw = 1);
uint64_t k1_jit_resident_warps(const void* handle);
// Chunk gate: a K1j launch raises *flag to its epoch when its first warp
// enters the last pass; k1_gate_wait holds a stream until then, so the next
// chunk's launch fills the SMs the last pass frees instead of interleaving
// its passes with the running launch's (k_signature.cu)
struct K1Gate {
  unsigned int* flag = nullptr;
  unsigned int epoch = 0;
};
void k1_gate_wait(const unsigned int* flag, unsigned int epoch, cudaStream_t s);
void k1_jit_launch(const void* handle, const uint8_t* d_text, const uint64_t* d_offsets,
                   const uint32_t* order, const uint32_t* item_doc, const uint64_t* item_off,
                   uint32_t n_items, uint32_t seg_len, uint32_t* d_sig,
                   unsigned long long* counter, cudaStream_t s, const K1Gate* gate = nullptr);
// UTF-8 -> codepoint units (k_utf8.cu): units_out[unit_off_out[d] ..
// unit_off_out[d+1]) are document d's units (decode_codepoints, text.cpp:101-113).
// Codepoint classes of a decoded batch (k_utf8.cu): per document 0 (all
// code points < 256), 1 (< 2^16) or 2; the documents of class < wide_from
// get 16-bit units in u16 (at the same unit offsets), the others u32 units.
struct CodepointClasses {
  DevBuf* cls_buf = nullptr;
  DevBuf* cnt_buf = nullptr;
  DevBuf* u16_buf = nullptr;
  uint32_t wide_from = 1;
  // outputs
  const uint32_t* cls = nullptr;
  const uint16_t* u16 = nullptr;
  uint64_t total = 0;
  uint32_t n_wide = 0, n_astral = 0;  // documents of class >= 1 / class 2
};
void decode_codepoints_device(const uint8_t* d_text, const uint64_t* d_offsets, uint64_t n,
                              DevBuf& units_buf, DevBuf& unit_off_buf, DevBuf& count_buf,
                              DevBuf& scan_tmp, cudaStream_t s, const uint32_t** units_out,
                              const uint64_t** unit_off_out, CodepointClasses* classes = nullptr);
// h_offsets: optional host copy of d_offsets; when given, planning happens on
// the host and the launch is fully asynchronous for single-item documents.
void launch_signatures(const DevFamily& fam, const uint8_t* d_bytes, const uint64_t* d_offsets,
                       uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                       uint32_t* d_band, SigScratch& scratch, cudaStream_t stream,
                       bool check_short, const uint64_t* h_offsets,
                       const K1Gate* gate = nullptr, const uint32_t* doc_class = nullptr,
                       uint32_t class_lo = 0, uint32_t class_hi = 0);

// Stable LSD radix sort of (key, value) pairs by the low key_bits bits.
void radix_sort_u32(uint32_t* keys, uint32_t* vals, uint64_t n, int key_bits, SortScratch& sc,
                    cudaStream_t s);
void radix_sort_u64(uint64_t* keys, uint32_t* vals, uint64_t n, int key_bits, SortScratch& sc,
                    cudaStream_t s);

int bits_for(uint64_t maxval);  // number of bits needed to hold maxval

// K2 output: non-singleton LSH cells as CSR over sorted rows (k_cells.cu).
constexpr uint32_t kCmpRows = 128;  // rows per compare work item (128 threads x kR)
constexpr uint32_t kJoinMax = 4096;  // largest cell the hash join (k_join) takes
constexpr uint32_t kJoinMaxP = 510;  // largest H - min_matches + 1 the joins' 9-bit tags take
struct CellSet {
  DevBuf rec_keys, rec_vals, flag, run_idx, run_start, cstart, clen, ckey, cpairs, ctiles, pair_off,
      ioff, icell, scan, maxbuf, fps;
  bool join_enabled = true;     // cells <= kJoinMax use the hash join
  uint64_t max_len = 0;         // largest non-singleton cell
  SortScratch sort;
  uint64_t records = 0, ncells = 0, items = 0, candidate_pairs = 0;
  uint64_t cell_records = 0;    // sum of n over non-singleton cells
  uint32_t tile_rows = kCmpRows;
  const uint32_t* sorted_rows = nullptr;  // rows of all records, grouped by cell
  uint64_t* cell_start = nullptr;         // per non-singleton cell
  uint32_t* cell_len = nullptr;
  uint32_t* cell_key = nullptr;           // band*K + bucket
  uint64_t* item_off = nullptr;           // per cell: first compare item
  uint32_t* item_cell = nullptr;          // per item: its cell
  void release() {
    for (DevBuf* b : {&rec_keys, &rec_vals, &flag, &run_idx, &run_start, &cstart, &clen, &ckey,
                      &cpairs, &ctiles, &pair_off, &ioff, &icell, &scan, &maxbuf, &fps})
      b->release();
    sort.release();
  }
};
// records: keys = cell ids (< key_limit), vals = rows; both are permuted.
void build_cells_from_records(CellSet& cs, uint32_t* keys, uint32_t* vals, uint64_t m,
                              uint64_t key_limit, uint32_t tile_rows, cudaStream_t s);
// re-tiles every cell for the all-pairs kernel (joins not applicable)
void cells_all_pairs_tiles(CellSet& cs, cudaStream_t s);
void make_records(const uint32_t* band, uint64_t n, uint32_t bands, uint32_t K, uint32_t doc_base,
                  uint32_t* keys, uint32_t* vals, cudaStream_t s);
void build_cells_from_bands(CellSet& cs, const uint32_t* band, uint64_t n, uint32_t bands,
                            uint32_t K, uint32_t tile_rows, cudaStream_t s);

// K3 output: accepted pairs, packed keys lo << nb | hi with match counts.
struct PairSet {
  DevBuf dkeys, dvals, dcount, flag, idx, scan, dlo, dhi, dmc;
  SortScratch sort;
  uint64_t* keys = nullptr;
  uint32_t* vals = nullptr;
  unsigned long long* counter = nullptr;
  uint64_t cap = 0, count = 0, distinct = 0;
  int nb = 1;
  uint32_t *lo = nullptr, *hi = nullptr, *mc = nullptr;  // distinct, sorted by (lo, hi)
  void release() {
    for (DevBuf* b : {&dkeys, &dvals, &dcount, &flag, &idx, &scan, &dlo, &dhi, &dmc}) b->release();
    sort.release();
  }
};
int compare_prefilter_width(uint32_t H, uint32_t min_match);
// Signature rows as K3 reads them: one table (world == 1), or the rows of
// `world` ranks in peer memory (global row g lives on the rank r with
// row_base[r] <= g < row_base[r+1]; bases[] are IPC-mapped peer pointers).
struct SigView {
  const uint32_t* base0 = nullptr;
  const uint32_t* const* bases = nullptr;  // device array [world]
  const uint64_t* row_base = nullptr;      // device array [world + 1]
  uint32_t world = 1;
  uint32_t H = 0;
  // K3's block fingerprints of the same rows (k_block_fps), fpNB per row:
  // one table (fp0) or one per rank (fp_bases, peer memory); fpNB = 0: none
  const uint32_t* fp0 = nullptr;
  const uint32_t* const* fp_bases = nullptr;
  uint32_t fpNB = 0;
  __host__ __device__ SigView() {}
  __host__ __device__ SigView(const uint32_t* b, uint32_t h) : base0(b), H(h) {}
  // the rank r with row_base[r] <= g < row_base[r + 1]: binary search over
  // the world + 1 bases (3 probes for 8 ranks, world <= 64)
  __device__ __forceinline__ uint32_t rank_of(uint32_t g) const {
    uint32_t r = 0;
#pragma unroll
    for (uint32_t step = 32; step > 0; step >>= 1)
      if (r + step < world && g >= row_base[r + step]) r += step;
    return r;
  }
  __device__ __forceinline__ const uint32_t* row(uint32_t g) const {
    if (world <= 1) return base0 + static_cast<uint64_t>(g) * H;
    const uint32_t r = rank_of(g);
    return bases[r] + (static_cast<uint64_t>(g) - row_base[r]) * H;
  }
  __device__ __forceinline__ const uint32_t* fp(uint32_t g) const {
    if (world <= 1) return fp0 + static_cast<uint64_t>(g) * fpNB;
    const uint32_t r = rank_of(g);
    return fp_bases[r] + (static_cast<uint64_t>(g) - row_base[r]) * fpNB;
  }
};
// K3's block shape for (H, min_matches): NB = H - min_matches + 1 blocks of
// BW positions (1 = the per-position join); k_block_fps of n rows into fps
void join_block_shape(uint32_t H, uint32_t min_match, uint32_t* NB, int* BW);
void block_fingerprints(const uint32_t* sig, uint64_t nrows, uint32_t H, uint32_t NB, int BW,
                        uint32_t* fps, cudaStream_t s);
// nrows: rows of d_sig (block fingerprints are precomputed for a one-table view)
void launch_compare(CellSet& cs, const SigView& d_sig, uint32_t H, uint32_t min_match,
                    int nb, uint64_t* out_key, uint32_t* out_m, unsigned long long* count,
                    uint64_t cap, cudaStream_t s, uint64_t nrows = 0);
uint64_t unique_pairs(PairSet& ps, cudaStream_t s);
// packs (lo, hi, m) triples (lo < hi not required) into ps.keys/ps.vals
void pack_pairs(PairSet& ps, const uint32_t* lo, const uint32_t* hi, const uint32_t* m,
                uint64_t count, cudaStream_t s);

// K4 output: components as groups of rows (k_union.cu).
struct GroupSet {
  DevBuf parent, flagbuf, in_edge, idx, keys, vals, rflag, dnear, ridx, gflag, gidx, gstart, drem,
      scan;
  SortScratch sort;
  uint64_t members = 0, groups = 0, removals = 0;
  uint32_t* member_rows = nullptr;  // groups by representative, members ascending
  uint64_t* group_start = nullptr;  // groups + 1
  uint32_t* near = nullptr;         // all members, ascending
  uint32_t* removal = nullptr;      // members that are not representatives, ascending
  void release() {
    for (DevBuf* b : {&parent, &flagbuf, &in_edge, &idx, &keys, &vals, &rflag, &dnear, &ridx,
                      &gflag, &gidx, &gstart, &drem, &scan})
      b->release();
    sort.release();
  }
};
void components(GroupSet& gs, const uint32_t* lo, const uint32_t* hi, uint64_t e, uint64_t n,
                cudaStream_t s);

// State of the last dedup run held by a context (results stay on device
// until fetched).
// K3g, the global block join of the in-memory dedup (k_gjoin.cu)
constexpr uint32_t kGJoinMaxBlocks = 64;
// block-major fingerprints of a batch's rows, fps[k * m + i] for the m rows
// of one table, or one such table per shard of a device group (peer memory;
// shard r holds rows row_base[r] .. row_base[r+1])
struct FpCols {
  const uint32_t* base0 = nullptr;
  const uint32_t* const* bases = nullptr;
  const uint64_t* row_base = nullptr;
  uint32_t world = 1;
};
// block k's column of FpCols: fingerprint of global row g
struct FpCol {
  const uint32_t* base = nullptr;  // world == 1: fps + k * n
  const uint32_t* const* bases = nullptr;
  const uint64_t* row_base = nullptr;
  uint32_t world = 1;
  uint32_t k = 0;
  __device__ __forceinline__ uint32_t get(uint64_t g) const {
    if (world <= 1) return base[g];
    uint32_t r = 0;
#pragma unroll
    for (uint32_t step = 32; step > 0; step >>= 1)
      if (r + step < world && g >= row_base[r + step]) r += step;
    const uint64_t m = row_base[r + 1] - row_base[r];
    return bases[r][static_cast<uint64_t>(k) * m + (g - row_base[r])];
  }
};
struct GJoin {
  DevBuf fps_buf, table_buf, link_buf, cnt, acc;
  uint32_t* fps = nullptr;                  // [NB][n] block fingerprints
  unsigned long long* table = nullptr;      // 2^tbits chain heads
  unsigned long long* link = nullptr;       // [n] (fingerprint << 32 | row) chained before
  unsigned long long* acc_d = nullptr;      // candidate pairs, cells, records, emitted
  int tbits = 10;
  void release() {
    for (DevBuf* b : {&fps_buf, &table_buf, &link_buf, &cnt, &acc}) b->release();
  }
};
struct GJoinCounts {
  uint64_t candidate_pairs, ncells, cell_records, emitted;
};
bool global_join_eligible(uint64_t n, uint32_t H, uint32_t B, uint32_t K, uint32_t mm);
// free device memory (cudaMemGetInfo), cached per device; re-queried when
// `need` is at least half of free * num / den (k_gjoin.cu)
uint64_t device_free_bytes(uint64_t need, uint64_t num, uint64_t den);
// reference counters from a histogram of the cells (async, into g.acc_d)
void gj_cell_counts(GJoin& g, const uint32_t* band, uint64_t n, uint32_t B, uint32_t K,
                    cudaStream_t s);
// the pieces, for device groups (nd_multi.cu): reset the counters, one
// shard's cell histogram, the counters from `parts` histograms (device array
// of pointers), block-major fingerprints of m rows, and the join of the given
// blocks over fingerprint columns / rows / band ids that may live on peers
void gj_reset(GJoin& g, cudaStream_t s);
void gj_cell_hist(GJoin& g, const uint32_t* band, uint64_t n, uint32_t B, uint32_t K,
                  cudaStream_t s, unsigned int* bad = nullptr);
void gj_cell_stats(GJoin& g, const uint32_t* const* d_cnts, uint32_t parts, uint64_t cells,
                   cudaStream_t s);
void gj_fps(const uint32_t* sig, uint64_t n, uint32_t H, uint32_t mm, uint32_t* fps,
            cudaStream_t s);
void gj_join(GJoin& g, const FpCols& fc, const SigView& sv, const SigView& bv, uint64_t n,
             uint32_t mm, const std::vector<uint32_t>& blocks, int nb, uint64_t* out_key,
             uint32_t* out_m, unsigned long long* count, uint64_t cap, cudaStream_t s);
// accepted pairs, each once, and the emitted-pairs counter (async)
void gj_pairs(GJoin& g, const uint32_t* sig, const uint32_t* band, uint64_t n, uint32_t H,
              uint32_t B, uint32_t mm, int nb, uint64_t* out_key, uint32_t* out_m,
              unsigned long long* count, uint64_t cap, cudaStream_t s);
GJoinCounts gj_read(GJoin& g, cudaStream_t s);

struct DedupState {
  DevBuf sig, band, text, offs;
  CellSet cells;
  GJoin gj;
  PairSet pairs;
  GroupSet groups;
  SigScratch sig_scratch;
  std::vector<uint64_t> doc_ids;  // row -> doc id (empty = identity)
  // out-of-core dedup: signature rows + band ids stay in host memory
  std::vector<uint32_t> host_sig, host_band;
  bool sig_on_host = false;
  uint32_t intervals = 1;         // bucket intervals of the last dedup
  const char* compare_kind = "";  // K3 of the last dedup: "global" (K3g) or "cells"
  uint64_t documents = 0;
  uint32_t K = 0;
  uint32_t bands = 0;             // band keys per row in band
  uint32_t H = 0;                 // hashes per row in sig
  bool valid = false;
  void release() {
    for (DevBuf* b : {&sig, &band, &text, &offs}) b->release();
    cells.release();
    gj.release();
    pairs.release();
    groups.release();
    sig_scratch.release();
  }
};

// band keys for n signature rows already on the device (d_docs: n scratch words)
void launch_band_keys(const uint32_t* d_sig, uint64_t n, uint32_t H, uint32_t bands, uint32_t rows,
                      uint32_t K, uint32_t* d_band, uint32_t* d_docs, cudaStream_t s);

// exclusive scan of counts (n entries) into out (n+1 entries, out[n] = total)
void scan_u64(const uint64_t* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp, cudaStream_t s);
void scan_u32_to_u64(const uint32_t* d_in, uint64_t* d_out, uint64_t n, DevBuf& tmp,
                     cudaStream_t s);

// mode-1 synthetic text into device memory (synth.cu)
void synth_text_device(const nd_synth_spec& s, const uint64_t* d_offsets, uint8_t* d_bytes,
                       DevBuf& scratch, cudaStream_t stream);

int sm_count();

}  // namespace ndb
