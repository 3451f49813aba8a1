// Definition of the opaque nd_ctx and shared C-ABI plumbing.
#pragma once

#include <functional>
#include <string>
#include <vector>

#include "nd_internal.cuh"

// One context per device: streams, uploaded family, scratch, last dedup.
struct nd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // ordering stream for all device work
  bool own_stream = false;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy engines for host entry points
  static constexpr int kSlots = 3;
  struct Slot {  // triple-buffered chunk of the host pipeline (nd_signatures)
    ndb::DevBuf text, off, sig, band;
    ndb::SigScratch scratch;
    cudaStream_t comp = nullptr;
    cudaEvent_t h2d_done = nullptr, comp_done = nullptr, d2h_done = nullptr;
  } slot[kSlots];
  ndb::PinnedBuf pinned_off;
  ndb::DevBuf gate_flag;        // K1Gate flag of this context's chunked K1j launches
  unsigned int gate_epoch = 0;
  // a gate for the next chunked K1j launch (null flag: gating off,
  // ND_K1J_GATE=0, or not a K1j family)
  ndb::K1Gate* next_gate(ndb::K1Gate& g);
  bool gate_on() const;
  ndb::DevBuf ring[3];          // text chunks streaming through h2d_signatures
  cudaStream_t ring_stream[3] = {nullptr, nullptr, nullptr};
  ndb::SigScratch ring_scratch[3];
  ndb::DevBuf synth_buf;
  ndb::DevBuf fam_buf, sig_in_text, sig_in_off;
  ndb::DevFamily fam;
  std::vector<nd_hash_fn> family_host;
  ndb::SigScratch sig_scratch;
  ndb::DedupState dedup;        // last nd_dedup / nd_dedup_device
  ndb::DedupState api, api2;    // last nd_compare_cells / nd_union
  ndb::DedupState h2d_state;    // text staging of nd_signatures_h2d
  ndb::SortScratch stage_sort;  // nd_stage_cell_records
  struct Peer {                 // signature rows of every rank in peer memory (nd_peer.cu)
    ndb::DevBuf own, bases, row_base, band_bases, fp_bases;
    std::vector<void*> opened;  // IPC mappings of the other ranks' rows
    ndb::SigView view;
    // nd_peer_export_gjoin: each rank's allocation also holds its band ids
    // and block fingerprints (K3g over peer memory)
    ndb::SigView band_view;
    ndb::FpCols fps;
    uint32_t world = 0, H = 0, B = 0, mm = 0, NB = 0;
    uint64_t rows = 0;
  } peer;
  // multi-device group (nd_ctx_create_multi): one sub-context per shard;
  // the group's own fields serve single-device calls on its first device
  std::vector<nd_ctx*> shards;
  struct Multi {                // per-shard exchange buffers (nd_multi.cu)
    ndb::DevBuf send_keys, send_vals, first_cell, split, bases, row_bases, row_base, pair_lo,
        pair_hi, pair_m, fps, fp_bases;
    ndb::SortScratch sort;
    ndb::PairSet final_pairs;
    std::vector<uint64_t> ranges;  // group: document range of each shard, last dedup
    bool last_valid = false;
    void release() {
      for (auto* b : {&send_keys, &send_vals, &first_cell, &split, &bases, &row_bases, &row_base,
                      &pair_lo, &pair_hi, &pair_m, &fps, &fp_bases})
        b->release();
      sort.release();
      final_pairs.release();
    }
  } multi;
  uint64_t hbm_budget = 0;      // compare-stage HBM budget (0 = 70 % of free memory)
  uint64_t family_seed = 0;
  bool family_derived = false;  // family came from derive_family(family_seed, ...)
  std::string err;
  std::string k1_note;          // why K1j is not used for the uploaded family (if it is not)

  ~nd_ctx();
  void ensure_streams();
  void ensure_ring_streams();
  void require_family() const;
};

namespace ndb {
int guarded_impl(nd_ctx* ctx, const std::function<void()>& fn);
// multi-device group contexts (nd_multi.cu)
bool is_group(const nd_ctx* ctx);
void family_upload_one(nd_ctx* ctx, const nd_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit);
void multi_family_upload(nd_ctx* g, const nd_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit);
void multi_signatures(nd_ctx* g, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                      uint32_t bands, uint32_t rows, uint32_t K, uint32_t* sig_out,
                      uint32_t* band_out);
void multi_dedup(nd_ctx* g, const uint8_t* bytes, const uint64_t* offsets,
                 const uint64_t* doc_ids, uint64_t n, const nd_params& p, nd_dedup_stats* stats);
void multi_fetch_signatures(nd_ctx* g, uint32_t* sig, uint32_t* band);
uint64_t h2d_chunk_bytes(const DevFamily& fam, size_t chunk_index);
// nd_signatures' host pipeline (chunks in, signature rows + band ids out)
void signatures_host(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                     uint32_t bands, uint32_t rows, uint32_t K, uint32_t* sig_out,
                     uint32_t* band_out);
// shared by nd_dedup.cu and nd_stages.cu
void validate(const nd_params& p);                 // RunConfig::validate, artifact fields
void ensure_family(nd_ctx* ctx, const nd_params& p);  // derive + upload when it changed
// K3 + distinct pairs over st.cells (grows the pair buffer on overflow)
void compare_and_unique(DedupState& st, const uint32_t* d_sig, uint32_t H, uint32_t mm,
                        uint64_t nrows, cudaStream_t s);
void compare_pairs(DedupState& st, const SigView& d_sig, uint32_t H, uint32_t mm, uint64_t nrows,
                   cudaStream_t s);
void compare_and_unique(DedupState& st, const SigView& d_sig, uint32_t H, uint32_t mm,
                        uint64_t nrows, cudaStream_t s);
// signatures of a host batch into device buffers (pipelined H2D, text kept in st.text)
void h2d_signatures(nd_ctx* ctx, DedupState& st, const uint8_t* bytes, const uint64_t* offsets,
                    uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                    uint32_t* d_band);
}
