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
  struct Slot {  // double-buffered chunk of the host pipeline
    ndb::DevBuf text, off, sig, band;
    ndb::SigScratch scratch;
    cudaStream_t comp = nullptr;
    cudaEvent_t h2d_done = nullptr, comp_done = nullptr, d2h_done = nullptr;
  } slot[2];
  ndb::PinnedBuf pinned_off;
  ndb::DevBuf synth_buf;
  ndb::DevBuf fam_buf, sig_in_text, sig_in_off;
  ndb::DevFamily fam;
  std::vector<nd_hash_fn> family_host;
  ndb::SigScratch sig_scratch;
  ndb::DedupState dedup;        // last nd_dedup / nd_dedup_device
  ndb::DedupState api, api2;    // last nd_compare_cells / nd_union
  ndb::DedupState h2d_state;    // text staging of nd_signatures_h2d
  ndb::SortScratch stage_sort;  // nd_stage_cell_records
  uint64_t family_seed = 0;
  bool family_derived = false;  // family came from derive_family(family_seed, ...)
  std::string err;

  ~nd_ctx();
  void ensure_streams();
  void require_family() const;
};

namespace ndb {
int guarded_impl(nd_ctx* ctx, const std::function<void()>& fn);
}
