// neardup_b200.hpp -- drop-in C++ facade over the C-ABI (neardup_b200.h) in the
// reference's own types (include/neardup/*.hpp of the neardup library).
//
// Include it inside the reference tree (it includes the reference's headers)
// and call neardup::b200::X where pipeline.cpp calls neardup::X:
//   signature_batch / signature_of_document   minhash.hpp:71-78
//   band_bucket_ids                           lsh.hpp:38-40
//   compare_pass                              compare.hpp:49-52
//   union_components (union_pairs + components) dedup_graph.hpp:34-43
//   dedup_in_memory (run_dedup's three stages, in HBM)  pipeline.hpp:100
// Status codes are rethrown as the reference's exception types, so the CLI's
// exit codes (tools/main.cpp:18-21) are unchanged; device failures become
// std::runtime_error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "neardup/compare.hpp"
#include "neardup/dedup_graph.hpp"
#include "neardup/lsh.hpp"
#include "neardup/minhash.hpp"
#include "neardup/pipeline.hpp"
#include "neardup/util.hpp"
#include "neardup_b200.h"

namespace neardup::b200 {

[[noreturn]] inline void rethrow(int rc, const char* msg) {
  std::string m = msg ? msg : "";
  switch (rc) {
    case ND_ERR_CONFIG: throw ConfigError(m);
    case ND_ERR_IO: throw IoError(m);
    case ND_ERR_PREREQ: throw PrerequisiteError(m);
    case ND_ERR_SHORT: throw ShortDocumentError(m);
    default: throw std::runtime_error("neardup_b200: " + m);
  }
}

// One device context (streams, uploaded family, scratch).  Not reentrant.
class Device {
 public:
  explicit Device(int device = 0) {
    if (int rc = nd_ctx_create(device, &ctx_); rc != ND_OK) rethrow(rc, nd_last_error_global());
  }
  ~Device() { nd_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  nd_ctx* get() const { return ctx_; }
  void check(int rc) const {
    if (rc != ND_OK) rethrow(rc, nd_last_error(ctx_));
  }
  void upload(const HashFamily& f) {
    static_assert(sizeof(HashFunctionParams) == sizeof(nd_hash_fn), "layout mirrors nd_hash_fn");
    check(nd_family_upload(ctx_, reinterpret_cast<const nd_hash_fn*>(f.functions.data()),
                           f.hash_count, f.shingle_len, static_cast<uint32_t>(f.unit)));
  }

 private:
  nd_ctx* ctx_ = nullptr;
};

// signature_batch (minhash.cpp:164-177): order preserved, short docs reported
// through on_short and skipped.
inline std::vector<Signature> signature_batch(Device& dev, std::span<const CleanDocument> docs,
                                              const HashFamily& family,
                                              const std::function<void(uint64_t)>& on_short = {}) {
  std::string bytes;
  std::vector<uint64_t> offsets{0};
  std::vector<uint64_t> ids;
  for (const CleanDocument& d : docs) {
    // units: bytes, or code points (nd_codepoint_count == text.cpp:88-99)
    const uint64_t units = family.unit == ShingleUnit::kByte
                               ? d.text.size()
                               : nd_codepoint_count(reinterpret_cast<const uint8_t*>(d.text.data()),
                                                    d.text.size());
    if (units < family.shingle_len) {
      if (on_short) on_short(d.doc_id);
      continue;
    }
    bytes += d.text;
    offsets.push_back(bytes.size());
    ids.push_back(d.doc_id);
  }
  std::vector<Signature> out(ids.size());
  if (ids.empty()) return out;
  dev.upload(family);
  std::vector<uint32_t> sig(ids.size() * family.hash_count);
  dev.check(nd_signatures(dev.get(), reinterpret_cast<const uint8_t*>(bytes.data()), offsets.data(),
                          ids.size(), 0, 0, 0, sig.data(), nullptr));
  for (size_t i = 0; i < ids.size(); ++i) {
    out[i].doc_id = ids[i];
    out[i].values.assign(sig.begin() + i * family.hash_count,
                         sig.begin() + (i + 1) * family.hash_count);
  }
  return out;
}

inline std::vector<uint32_t> band_bucket_ids(Device& dev, std::span<const uint32_t> signature,
                                             uint32_t bands, uint32_t rows, uint32_t bucket_count) {
  if (bucket_count == 0) throw ConfigError("bucket count must be positive");
  std::vector<uint32_t> ids(bands);
  dev.check(nd_band_keys(dev.get(), signature.data(), 1, static_cast<uint32_t>(signature.size()),
                         bands, rows, bucket_count, ids.data()));
  return ids;
}

// compare_pass (compare.cpp:69-86) over a GatherResult.
inline std::vector<DuplicatePair> compare_pass(Device& dev, const GatherResult& gathered,
                                               uint32_t hash_count,
                                               const SimilarityThreshold& threshold) {
  // one row per distinct doc id (ascending), cells as CSR row lists
  std::vector<uint64_t> ids;
  for (const auto& b : gathered.buckets) ids.insert(ids.end(), b.doc_ids.begin(), b.doc_ids.end());
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  std::vector<uint32_t> sigs(ids.size() * hash_count);
  std::vector<uint64_t> offs{0};
  std::vector<uint32_t> rows;
  for (const auto& b : gathered.buckets) {
    for (size_t k = 0; k < b.doc_ids.size(); ++k) {
      uint32_t r = static_cast<uint32_t>(std::lower_bound(ids.begin(), ids.end(), b.doc_ids[k]) - ids.begin());
      std::copy_n(b.signatures.begin() + k * hash_count, hash_count, sigs.begin() + size_t(r) * hash_count);
      rows.push_back(r);
    }
    offs.push_back(rows.size());
  }
  uint64_t n = 0;
  dev.check(nd_compare_cells(dev.get(), sigs.data(), ids.size(), hash_count, offs.data(), rows.data(),
                             offs.size() - 1, threshold.value.num, threshold.value.den, &n));
  std::vector<uint32_t> lo(n), hi(n), m(n);
  dev.check(nd_pairs_fetch(dev.get(), lo.data(), hi.data(), m.data()));
  std::vector<DuplicatePair> out(n);
  for (uint64_t i = 0; i < n; ++i) out[i] = {ids[lo[i]], ids[hi[i]], m[i]};
  return out;
}

// union_pairs + components (dedup_graph.cpp:48-81).
inline std::vector<DuplicateGroup> union_components(Device& dev, std::span<const DuplicatePair> pairs) {
  std::vector<uint64_t> ids;
  for (const auto& p : pairs) {
    ids.push_back(p.lo);
    ids.push_back(p.hi);
  }
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  auto rank = [&](uint64_t d) {
    return static_cast<uint32_t>(std::lower_bound(ids.begin(), ids.end(), d) - ids.begin());
  };
  std::vector<uint32_t> lo, hi;
  for (const auto& p : pairs) {
    lo.push_back(rank(p.lo));
    hi.push_back(rank(p.hi));
  }
  uint64_t nm = 0, ng = 0;
  dev.check(nd_union(dev.get(), lo.data(), hi.data(), lo.size(), static_cast<uint32_t>(ids.size()), &nm, &ng));
  std::vector<uint32_t> members(nm);
  std::vector<uint64_t> start(ng + 1);
  dev.check(nd_groups_fetch(dev.get(), members.data(), start.data()));
  std::vector<DuplicateGroup> groups(ng);
  for (uint64_t g = 0; g < ng; ++g) {
    for (uint64_t k = start[g]; k < start[g + 1]; ++k) groups[g].members.push_back(ids[members[k]]);
    groups[g].representative = groups[g].members.front();
  }
  return groups;
}

// run_dedup's hash -> gather-compare -> union stages (pipeline.cpp:510-532)
// over in-memory surviving documents (ascending doc_ids), all in HBM; returns
// the same DedupReport emit_report builds (dedup_graph.cpp:83-102).
inline DedupReport dedup_in_memory(Device& dev, std::span<const CleanDocument> docs,
                                   const RunConfig& c, uint64_t* candidate_pairs = nullptr) {
  std::string bytes;
  std::vector<uint64_t> offsets{0}, ids;
  for (const CleanDocument& d : docs) {
    bytes += d.text;
    offsets.push_back(bytes.size());
    ids.push_back(d.doc_id);
  }
  nd_params p{};
  p.hash_count = c.hash_count;
  p.bands = c.bands;
  p.rows = c.rows;
  p.shingle_len = c.shingle_len;
  p.unit = static_cast<uint32_t>(c.unit);
  p.threshold_num = c.threshold.num;
  p.threshold_den = c.threshold.den;
  p.scale_num = c.bucket_scale.num;
  p.scale_den = c.bucket_scale.den;
  p.seed = c.seed;
  nd_dedup_stats st{};
  dev.check(nd_dedup(dev.get(), reinterpret_cast<const uint8_t*>(bytes.data()), offsets.data(),
                     ids.data(), ids.size(), &p, &st));
  std::vector<uint64_t> members(st.near_duplicates), start(st.duplicate_groups + 1);
  dev.check(nd_dedup_fetch_groups(dev.get(), members.data(), start.data()));
  std::vector<DuplicateGroup> groups(st.duplicate_groups);
  for (uint64_t g = 0; g < st.duplicate_groups; ++g) {
    groups[g].members.assign(members.begin() + start[g], members.begin() + start[g + 1]);
    groups[g].representative = groups[g].members.front();
  }
  if (candidate_pairs) *candidate_pairs = st.candidate_pairs;
  return emit_report(std::move(groups), st.documents, st.distinct_pairs);
}

}  // namespace neardup::b200
