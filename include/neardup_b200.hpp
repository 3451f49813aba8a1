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
//   run_hash_stage / run_compare_stage / run_union_stage / run_dedup
//     (pipeline.hpp:69-100, the staged on-disk workflow: the same workspace
//     bytes as the reference, with the JSON side files written through the
//     reference's own nlohmann::ordered_json)
// Status codes are rethrown as the reference's exception types, so the CLI's
// exit codes (tools/main.cpp:18-21) are unchanged; device failures become
// std::runtime_error.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
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
#include <unistd.h>

#include <nlohmann/json.hpp>

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

// One device context (streams, uploaded family, scratch), or one context over
// a list of devices (nd_ctx_create_multi: signature_batch and run_dedup shard
// their batches over the GPUs, one host thread per device).  Not reentrant.
class Device {
 public:
  explicit Device(int device = 0) {
    if (int rc = nd_ctx_create(device, &ctx_); rc != ND_OK) rethrow(rc, nd_last_error_global());
  }
  explicit Device(std::span<const int> devices) {
    if (int rc = nd_ctx_create_multi(devices.data(), static_cast<int>(devices.size()), &ctx_);
        rc != ND_OK)
      rethrow(rc, nd_last_error_global());
  }
  int shards() const { return nd_ctx_shard_count(ctx_); }
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


// ---- the staged, file-backed workflow (pipeline.hpp:62-100) -----------------
namespace detail {
namespace fs = std::filesystem;
using ojson = nlohmann::ordered_json;

// write_file_bytes (util.cpp:132-140): write, flush, optional fsync, close
inline void write_text(const std::string& path, const std::string& bytes, bool fsync_file = false) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw IoError("cannot create '" + path + "'");
  bool ok = bytes.empty() || std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size();
  if (ok && std::fflush(f) != 0) ok = false;
  if (ok && fsync_file && ::fsync(fileno(f)) != 0) ok = false;
  if (std::fclose(f) != 0) ok = false;
  if (!ok) throw IoError("write failed for '" + path + "'");
}
inline std::string read_text(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open '" + path + "'");
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
// pipeline.cpp:79-99
inline std::vector<std::string> expand_inputs(const std::vector<std::string>& inputs) {
  std::vector<std::string> paths;
  for (const std::string& e : inputs) {
    std::error_code ec;
    if (fs::is_directory(e, ec)) {
      std::vector<std::string> found;
      for (const auto& it : fs::directory_iterator(e, ec))
        if (it.is_regular_file() && it.path().extension() == ".jsonl") found.push_back(it.path().string());
      std::sort(found.begin(), found.end());
      paths.insert(paths.end(), found.begin(), found.end());
    } else if (fs::is_regular_file(e, ec)) {
      paths.push_back(e);
    } else {
      throw IoError("input '" + e + "' does not exist");
    }
  }
  return paths;
}
inline std::string signatures_dir(const RunConfig& c) { return c.workspace + "/signatures"; }
inline std::string pairs_dir(const RunConfig& c) { return c.workspace + "/pairs"; }
// pipeline.cpp:101-105
inline std::string signature_file_name(uint64_t ordinal, const std::string& source) {
  char prefix[16];
  std::snprintf(prefix, sizeof prefix, "%05llu", static_cast<unsigned long long>(ordinal));
  return std::string(prefix) + "_" + fs::path(source).stem().string() + ".feds";
}
// pipeline.cpp:107-118
inline nd_feds_header header_template(const RunConfig& c, uint32_t K) {
  nd_feds_header h{};
  h.hash_count = c.hash_count;
  h.bands = c.bands;
  h.rows = c.rows;
  h.bucket_count = K;
  h.shingle_len = c.shingle_len;
  h.unit = static_cast<uint32_t>(c.unit);
  h.family_seed = c.seed;
  h.scale_num = c.bucket_scale.num;
  h.scale_den = c.bucket_scale.den;
  return h;
}
// pipeline.cpp:252-265
inline ojson parameters(const RunConfig& c) {
  ojson p;
  p["text_field"] = c.text_field;
  p["hash_count"] = c.hash_count;
  p["bands"] = c.bands;
  p["rows"] = c.rows;
  p["shingle_len"] = c.shingle_len;
  p["unit"] = std::string(shingle_unit_name(c.unit));
  p["threshold"] = c.threshold.str();
  p["bucket_scale"] = c.bucket_scale.str();
  p["min_chars"] = c.min_chars;
  p["seed"] = c.seed;
  return p;
}
inline void ingest_check(int rc) {
  if (rc != ND_OK) rethrow(rc, nd_ingest_last_error());
}
inline const char* reason_name(uint32_t r) {
  static const char* names[] = {"", "invalid_json", "not_an_object", "missing_text_field",
                                "text_field_not_string", "below_min_chars",
                                "too_short_to_shingle"};
  return r < 7 ? names[r] : "unknown";
}
// pipeline.cpp:267-286 + load_run_manifest (:356-378)
inline ojson load_json(const std::string& path, const std::string& stage) {
  if (!fs::exists(path))
    throw PrerequisiteError("'" + path + "' is missing; run the " + stage + " stage first");
  ojson j = ojson::parse(read_text(path), nullptr, false);
  if (j.is_discarded() || !j.is_object()) throw IoError("'" + path + "' is not valid JSON");
  return j;
}
inline void check_hash(const ojson& j, const RunConfig& c, const std::string& path) {
  if (j.value("config_hash", static_cast<uint64_t>(0)) != c.config_hash())
    throw ConfigError("configuration changed since '" + path + "' was written; rerun the earlier stages");
}
}  // namespace detail

// run_hash_stage (pipeline.cpp:288-339): the multi-threaded loader
// (nd_jsonl_*), K1 per input file straight into its .feds file (nd_hash_file)
inline HashStageOutput run_hash_stage(Device& dev, const RunConfig& config) {
  namespace fs = std::filesystem;
  config.validate();
  fs::create_directories(detail::signatures_dir(config));
  fs::create_directories(detail::pairs_dir(config));
  std::vector<std::string> paths = detail::expand_inputs(config.inputs);
  if (paths.empty()) throw ConfigError("no input files given");
  std::sort(paths.begin(), paths.end());
  for (size_t i = 1; i < paths.size(); ++i)
    if (paths[i] == paths[i - 1]) throw ConfigError("duplicate input file '" + paths[i] + "'");
  HashStageOutput out;
  RejectLog rejects;
  uint64_t offset = 0;
  for (const std::string& p : paths) {  // build_manifest (corpus.cpp:109-141)
    nd_jsonl* f = nullptr;
    detail::ingest_check(nd_jsonl_load(p.c_str(), config.text_field.c_str(), config.min_chars,
                                       config.shingle_len, static_cast<uint32_t>(config.unit), 0,
                                       0, &f));
    uint64_t rec = 0, surv = 0, nb = 0, nrej = 0;
    nd_jsonl_counts(f, &rec, &surv, &nb, &nrej);
    std::vector<uint64_t> lines(nrej);
    std::vector<uint32_t> why(nrej);
    detail::ingest_check(nd_jsonl_rejects(f, lines.data(), why.data()));
    nd_jsonl_free(f);
    for (uint64_t r = 0; r < nrej; ++r) rejects.add(p, lines[r], detail::reason_name(why[r]));
    FileStats st;
    st.path = p;
    st.records = rec;
    st.surviving = surv;
    st.record_offset = offset;
    offset += rec;
    out.manifest.total_records += rec;
    out.manifest.total_surviving += surv;
    out.manifest.files.push_back(st);
  }
  if (out.manifest.total_surviving == 0)
    throw ConfigError("no documents survive preprocessing; nothing to deduplicate");
  out.bucket_count = choose_bucket_count(out.manifest.total_surviving, config.bucket_scale);
  const nd_feds_header base = detail::header_template(config, out.bucket_count);
  for (size_t i = 0; i < out.manifest.files.size(); ++i) {
    const FileStats& st = out.manifest.files[i];
    const std::string sig_path =
        detail::signatures_dir(config) + "/" + detail::signature_file_name(i, st.path);
    nd_jsonl* f = nullptr;
    detail::ingest_check(nd_jsonl_load(st.path.c_str(), config.text_field.c_str(),
                                       config.min_chars, config.shingle_len,
                                       static_cast<uint32_t>(config.unit), 0, 1, &f));
    uint64_t rec = 0, surv = 0, nb = 0, nrej = 0;
    nd_jsonl_counts(f, &rec, &surv, &nb, &nrej);
    if (rec != st.records) {
      nd_jsonl_free(f);
      throw PrerequisiteError("'" + st.path + "' changed since the manifest was built");
    }
    std::vector<uint8_t> bytes(nb + 1);
    std::vector<uint64_t> offs(surv + 1), ids(surv);
    detail::ingest_check(nd_jsonl_documents(f, st.record_offset, bytes.data(), offs.data(),
                                            ids.data(), nullptr));
    nd_jsonl_free(f);
    nd_feds_header h = base;
    h.source_ordinal = i;
    dev.check(nd_hash_file(dev.get(), bytes.data(), offs.data(), ids.data(), surv, &h,
                           sig_path.c_str(), config.fsync_files));
    out.signature_files.push_back(sig_path);
    out.total_signature_bytes += fs::file_size(sig_path);
  }
  rejects.write_jsonl(config.workspace + "/rejects.jsonl");
  detail::ojson doc;
  doc["format_version"] = 1;
  doc["config_hash"] = config.config_hash();
  doc["parameters"] = detail::parameters(config);
  doc["bucket_count"] = out.bucket_count;
  doc["totals"] = {{"records", out.manifest.total_records},
                   {"surviving", out.manifest.total_surviving},
                   {"signature_bytes", out.total_signature_bytes}};
  detail::ojson files = detail::ojson::array();
  for (size_t i = 0; i < out.manifest.files.size(); ++i) {
    const FileStats& f = out.manifest.files[i];
    detail::ojson e;
    e["path"] = f.path;
    e["records"] = f.records;
    e["surviving"] = f.surviving;
    e["record_offset"] = f.record_offset;
    e["signature_file"] = fs::path(out.signature_files[i]).filename().string();
    files.push_back(e);
  }
  doc["files"] = files;
  detail::write_text(config.workspace + "/run_manifest.json", doc.dump(2) + "\n",
                     config.fsync_files);  // pipeline.cpp:335
  return out;
}

// run_compare_stage (pipeline.cpp:382-432) on the GPU (nd_compare_stage)
inline CompareStageOutput run_compare_stage(Device& dev, const RunConfig& config) {
  namespace fs = std::filesystem;
  config.validate();
  const std::string mpath = config.workspace + "/run_manifest.json";
  detail::ojson m = detail::load_json(mpath, "hash");
  detail::check_hash(m, config, mpath);
  std::vector<std::string> feds, sources;
  uint32_t K = 0;
  uint64_t total_bytes = 0;
  try {
    K = m.at("bucket_count").get<uint32_t>();
    total_bytes = m.at("totals").at("signature_bytes").get<uint64_t>();
    for (const auto& e : m.at("files")) {
      sources.push_back(e.at("path").get<std::string>());
      feds.push_back(detail::signatures_dir(config) + "/" + e.at("signature_file").get<std::string>());
    }
  } catch (const detail::ojson::exception&) {
    throw IoError("'" + mpath + "' is missing required fields");
  }
  if (!config.inputs.empty()) {
    std::vector<std::string> cur = detail::expand_inputs(config.inputs);
    std::sort(cur.begin(), cur.end());
    if (cur != sources)
      throw PrerequisiteError("input files differ from the hashed manifest; rerun the hash stage");
  }
  if (config.buckets_per_pass && *config.buckets_per_pass < 1)
    throw ConfigError("buckets-per-pass override must be at least 1");
  std::vector<const char*> fp;
  for (const auto& f : feds) fp.push_back(f.c_str());
  const nd_feds_header ex = detail::header_template(config, K);
  nd_compare_stage_stats st{};
  fs::create_directories(detail::pairs_dir(config));
  dev.check(nd_compare_stage(dev.get(), fp.data(), static_cast<uint32_t>(fp.size()), &ex,
                             total_bytes, config.workers, config.memory_budget,
                             config.buckets_per_pass.value_or(0), config.threshold.num,
                             config.threshold.den, detail::pairs_dir(config).c_str(),
                             config.fsync_files, &st));
  std::vector<uint32_t> passes(config.workers);
  uint32_t C = 0;
  dev.check(nd_plan_gather(total_bytes, K, config.bands, config.workers, config.memory_budget,
                           config.buckets_per_pass.value_or(0), &C, passes.data()));
  CompareStageOutput out;
  out.buckets_per_pass = st.buckets_per_pass;
  out.pass_count = st.pass_count;
  out.candidate_pairs = st.candidate_pairs;
  out.emitted_pairs = st.emitted_pairs;
  out.gather_peak_bytes = st.gather_peak_bytes;
  for (uint32_t w = 0; w < config.workers; ++w)
    for (uint32_t p = 0; p < passes[w]; ++p)
      out.pair_files.push_back(detail::pairs_dir(config) + "/w" + std::to_string(w) + "_p" +
                               std::to_string(p) + ".pairs");
  std::sort(out.pair_files.begin(), out.pair_files.end());
  detail::ojson doc;
  doc["config_hash"] = config.config_hash();
  doc["bucket_count"] = K;
  doc["buckets_per_pass"] = out.buckets_per_pass;
  doc["pass_count"] = out.pass_count;
  doc["workers"] = config.workers;
  doc["memory_budget"] = config.memory_budget;
  doc["candidate_pairs"] = out.candidate_pairs;
  doc["emitted_pairs"] = out.emitted_pairs;
  doc["gather_peak_bytes"] = out.gather_peak_bytes;
  detail::ojson files = detail::ojson::array();
  for (const auto& f : out.pair_files) files.push_back(fs::path(f).filename().string());
  doc["pair_files"] = files;
  detail::write_text(config.workspace + "/compare_stage.json", doc.dump(2) + "\n",
                     config.fsync_files);  // pipeline.cpp:444
  return out;
}

// run_union_stage (pipeline.cpp:434-508) on the GPU (nd_union_stage)
inline DedupReport run_union_stage(Device& dev, const RunConfig& config) {
  config.validate();
  const std::string mpath = config.workspace + "/run_manifest.json";
  detail::ojson m = detail::load_json(mpath, "hash");
  detail::check_hash(m, config, mpath);
  const std::string spath = config.workspace + "/compare_stage.json";
  detail::ojson stage = detail::load_json(spath, "gather-compare");
  detail::check_hash(stage, config, spath);
  std::vector<std::string> files;
  uint64_t surviving = 0, records = 0;
  try {
    surviving = m.at("totals").at("surviving").get<uint64_t>();
    records = m.at("totals").at("records").get<uint64_t>();
    for (const auto& n : stage.at("pair_files"))
      files.push_back(detail::pairs_dir(config) + "/" + n.get<std::string>());
  } catch (const detail::ojson::exception&) {
    throw IoError("'" + spath + "' is missing required fields");
  }
  std::vector<const char*> fp;
  for (const auto& f : files) fp.push_back(f.c_str());
  nd_dedup_stats st{};
  dev.check(nd_union_stage(dev.get(), fp.data(), static_cast<uint32_t>(fp.size()), surviving,
                           records, config.workspace.c_str(), config.fsync_files, &st));
  std::vector<uint64_t> members(st.near_duplicates), start(st.duplicate_groups + 1);
  dev.check(nd_dedup_fetch_groups(dev.get(), members.data(), start.data()));
  std::vector<DuplicateGroup> groups(st.duplicate_groups);
  for (uint64_t g = 0; g < st.duplicate_groups; ++g) {
    groups[g].members.assign(members.begin() + start[g], members.begin() + start[g + 1]);
    groups[g].representative = groups[g].members.front();
  }
  return emit_report(std::move(groups), surviving, st.distinct_pairs);
}

// run_dedup (pipeline.cpp:510-532): the three stages + timings.json
inline DedupReport run_dedup(Device& dev, const RunConfig& config, StageTimings* timings = nullptr) {
  using clock = std::chrono::steady_clock;
  StageTimings t;
  auto t0 = clock::now();
  run_hash_stage(dev, config);
  auto t1 = clock::now();
  run_compare_stage(dev, config);
  auto t2 = clock::now();
  DedupReport rep = run_union_stage(dev, config);
  auto t3 = clock::now();
  t.hash_seconds = std::chrono::duration<double>(t1 - t0).count();
  t.compare_seconds = std::chrono::duration<double>(t2 - t1).count();
  t.union_seconds = std::chrono::duration<double>(t3 - t2).count();
  detail::ojson j;
  j["workers"] = config.workers;
  j["hash_seconds"] = t.hash_seconds;
  j["compare_seconds"] = t.compare_seconds;
  j["union_seconds"] = t.union_seconds;
  j["total_seconds"] = t.total();
  detail::write_text(config.workspace + "/timings.json", j.dump(2) + "\n");
  if (timings) *timings = t;
  return rep;
}

}  // namespace neardup::b200
