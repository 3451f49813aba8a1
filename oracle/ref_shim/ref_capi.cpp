// extern "C" bridge onto the UNMODIFIED reference library (TEST INFRASTRUCTURE ONLY).
//
// Compiled together with /root/reference/proj/src/*.cpp (in place, never
// copied) by oracle/Makefile into oracle/_ref/libneardup_ref.so.  Only
// tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
// load it, as the checker or as the timed CPU baseline -- never as product.
//
// Every function wraps the reference's own public API:
//   derive_family            minhash.hpp:42   (minhash.cpp:71-105)
//   signature_of_document    minhash.hpp:71   (minhash.cpp:133-162)
//   band_bucket_ids          lsh.hpp:38       (lsh.cpp:42-60)
//   choose_bucket_count      lsh.hpp:33       (lsh.cpp:26-40)
//   compare_pass             compare.hpp:52   (compare.cpp:69-86)
//   union_pairs/components/emit_report  dedup_graph.hpp:34-55
//   generate_synthetic/write_synthetic  synthetic.hpp:57-63
//   run_dedup                pipeline.hpp:100 (pipeline.cpp:510-532)
//   run_eval_accuracy        pipeline.hpp:114 (pipeline.cpp:534-585)
#include <algorithm>
#include <chrono>
#include <filesystem>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "neardup/compare.hpp"
#include "neardup/corpus.hpp"
#include "neardup/dedup_graph.hpp"
#include "neardup/lsh.hpp"
#include "neardup/minhash.hpp"
#include "neardup/oracle.hpp"
#include "neardup/pipeline.hpp"
#include "neardup/sigstore.hpp"
#include "neardup/synthetic.hpp"
#include "neardup/util.hpp"

using namespace neardup;

namespace {
thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_error = e.what();
    return 2;
  } catch (const IoError& e) {
    g_error = e.what();
    return 3;
  } catch (const PrerequisiteError& e) {
    g_error = e.what();
    return 4;
  } catch (const ShortDocumentError& e) {
    g_error = e.what();
    return 6;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

// layout shared with include/neardup_b200.h's nd_hash_fn (24 bytes)
struct FnOut {
  uint32_t modulus, base, base_inverse, base_power;
  uint64_t reduce_factor;
};
static_assert(sizeof(FnOut) == 24);
}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_derive_family(uint64_t seed, uint32_t H, uint32_t L, uint32_t unit, FnOut* out) {
  return guarded([&] {
    HashFamily fam = derive_family(seed, H, L, static_cast<ShingleUnit>(unit));
    for (uint32_t i = 0; i < H; ++i) {
      const auto& f = fam.functions[i];
      out[i] = {f.modulus, f.base, f.base_inverse, f.base_power, f.reduce_factor};
    }
  });
}

uint32_t ref_choose_bucket_count(uint64_t n, uint64_t num, uint64_t den) {
  uint32_t k = 0;
  if (guarded([&] { k = choose_bucket_count(n, Ratio(num, den)); }) != 0) return 0;
  return k;
}

uint32_t ref_min_matches(uint32_t H, uint64_t num, uint64_t den) {
  return SimilarityThreshold{Ratio(num, den)}.min_matches(H);
}

// Signature + band ids for a packed batch, through the reference's own
// per-document functions, parallelised the way the hash stage does it
// (parallel_for_index, pipeline.cpp:214-218).  K == 0 skips banding.
int ref_signatures(const uint8_t* bytes, const uint64_t* offsets, const uint64_t* doc_ids,
                   uint64_t n, uint64_t seed, uint32_t H, uint32_t L, uint32_t unit,
                   uint32_t bands, uint32_t rows, uint32_t K, unsigned workers,
                   uint32_t* sig_out, uint32_t* band_out) {
  return guarded([&] {
    HashFamily fam = derive_family(seed, H, L, static_cast<ShingleUnit>(unit));
    parallel_for_index(n, workers, [&](uint64_t i) {
      CleanDocument doc;
      doc.doc_id = doc_ids ? doc_ids[i] : i;
      doc.text.assign(reinterpret_cast<const char*>(bytes + offsets[i]), offsets[i + 1] - offsets[i]);
      doc.char_count = doc.text.size();
      Signature sig = signature_of_document(doc, fam);
      std::memcpy(sig_out + i * H, sig.values.data(), H * sizeof(uint32_t));
      if (K != 0 && band_out) {
        std::vector<uint32_t> ids = band_bucket_ids(sig.values, bands, rows, K);
        std::memcpy(band_out + i * bands, ids.data(), bands * sizeof(uint32_t));
      }
    });
  });
}

// compare_pass over in-memory cells given as CSR lists of row indices into a
// signature matrix (rows ascending inside each cell, as scan_gather leaves
// them).  Output: sorted distinct (lo, hi, match) triples as malloc'd arrays.
int ref_compare_cells(const uint32_t* sigs, const uint64_t* doc_ids, uint32_t H,
                      const uint64_t* cell_offsets, const uint32_t* cell_rows, uint64_t ncells,
                      uint64_t thr_num, uint64_t thr_den, uint32_t tile,
                      uint64_t** lo_out, uint64_t** hi_out, uint32_t** m_out, uint64_t* npairs) {
  return guarded([&] {
    GatherResult gathered;
    for (uint64_t c = 0; c < ncells; ++c) {
      GatheredBucket b;
      b.key = {0, static_cast<uint32_t>(c)};
      for (uint64_t k = cell_offsets[c]; k < cell_offsets[c + 1]; ++k) {
        uint32_t r = cell_rows[k];
        b.doc_ids.push_back(doc_ids ? doc_ids[r] : r);
        b.signatures.insert(b.signatures.end(), sigs + static_cast<uint64_t>(r) * H,
                            sigs + static_cast<uint64_t>(r + 1) * H);
      }
      gathered.buckets.push_back(std::move(b));
    }
    std::vector<DuplicatePair> pairs =
        compare_pass(gathered, H, SimilarityThreshold{Ratio(thr_num, thr_den)}, tile);
    *npairs = pairs.size();
    *lo_out = static_cast<uint64_t*>(std::malloc(8 * (pairs.size() + 1)));
    *hi_out = static_cast<uint64_t*>(std::malloc(8 * (pairs.size() + 1)));
    *m_out = static_cast<uint32_t*>(std::malloc(4 * (pairs.size() + 1)));
    for (size_t i = 0; i < pairs.size(); ++i) {
      (*lo_out)[i] = pairs[i].lo;
      (*hi_out)[i] = pairs[i].hi;
      (*m_out)[i] = pairs[i].match_count;
    }
  });
}

// Kernel-only CPU baseline of the compare step: cells are
// gathered into GatheredBuckets (scan_gather's copies, timed apart), then
// compare_bucket (compare.cpp:24-67) runs over every cell with the
// reference's own parallel_for_index (util.cpp:81-122) -- parallel over cells,
// not capped at one worker per band like run_compare_stage
// (pipeline.cpp:387-420) -- and the accepted pairs are sorted + uniqued
// (compare_pass, compare.cpp:77-84).  Times in seconds; counts out.
int ref_compare_cells_timed(const uint32_t* sigs, uint32_t H, const uint64_t* cell_offsets,
                            const uint32_t* cell_rows, uint64_t ncells, uint64_t thr_num,
                            uint64_t thr_den, unsigned workers, double* gather_s,
                            double* compare_s, double* unique_s, uint64_t* emitted,
                            uint64_t* distinct, uint64_t** lo_out, uint64_t** hi_out) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    std::vector<GatheredBucket> cells(ncells);
    parallel_for_index(ncells, workers, [&](uint64_t c) {
      GatheredBucket& b = cells[c];
      b.key = {0, static_cast<uint32_t>(c)};
      for (uint64_t k = cell_offsets[c]; k < cell_offsets[c + 1]; ++k) {
        const uint32_t r = cell_rows[k];
        b.doc_ids.push_back(r);
        b.signatures.insert(b.signatures.end(), sigs + static_cast<uint64_t>(r) * H,
                            sigs + static_cast<uint64_t>(r + 1) * H);
      }
    });
    auto t1 = clk::now();
    const SimilarityThreshold thr{Ratio(thr_num, thr_den)};
    std::vector<std::vector<DuplicatePair>> out(ncells);
    parallel_for_index(ncells, workers,
                       [&](uint64_t c) { out[c] = compare_bucket(cells[c], H, thr); });
    auto t2 = clk::now();
    std::vector<DuplicatePair> all;
    for (auto& v : out) all.insert(all.end(), v.begin(), v.end());
    *emitted = all.size();
    std::sort(all.begin(), all.end(), [](const DuplicatePair& a, const DuplicatePair& b) {
      return a.lo != b.lo ? a.lo < b.lo : a.hi < b.hi;
    });
    all.erase(std::unique(all.begin(), all.end(),
                          [](const DuplicatePair& a, const DuplicatePair& b) {
                            return a.lo == b.lo && a.hi == b.hi;
                          }),
              all.end());
    auto t3 = clk::now();
    *distinct = all.size();
    *gather_s = std::chrono::duration<double>(t1 - t0).count();
    *compare_s = std::chrono::duration<double>(t2 - t1).count();
    *unique_s = std::chrono::duration<double>(t3 - t2).count();
    *lo_out = static_cast<uint64_t*>(std::malloc(8 * (all.size() + 1)));
    *hi_out = static_cast<uint64_t*>(std::malloc(8 * (all.size() + 1)));
    for (size_t i = 0; i < all.size(); ++i) {
      (*lo_out)[i] = all[i].lo;
      (*hi_out)[i] = all[i].hi;
    }
  });
}

// union_pairs + components (dedup_graph.cpp:48-81) timed inside the library
int ref_union_timed(const uint64_t* lo, const uint64_t* hi, uint64_t npairs, double* seconds,
                    uint64_t* ngroups, uint64_t* nmembers) {
  return guarded([&] {
    std::vector<DuplicatePair> pairs(npairs);
    for (uint64_t i = 0; i < npairs; ++i) pairs[i] = {lo[i], hi[i], 0};
    auto t0 = std::chrono::steady_clock::now();
    UnionFind uf = union_pairs(pairs);
    std::vector<DuplicateGroup> groups = components(uf);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint64_t m = 0;
    for (const auto& g : groups) m += g.members.size();
    *ngroups = groups.size();
    *nmembers = m;
  });
}

// all_pairs_dupset (oracle.cpp:53-108): docs with any partner above the
// threshold; out receives the sorted doc ids, *nout their count.
int ref_all_pairs_dupset(const uint32_t* sigs, const uint64_t* doc_ids, uint64_t n, uint32_t H,
                         uint64_t thr_num, uint64_t thr_den, unsigned workers, uint64_t* out,
                         uint64_t* nout) {
  return guarded([&] {
    std::vector<Signature> s(n);
    for (uint64_t i = 0; i < n; ++i) {
      s[i].doc_id = doc_ids ? doc_ids[i] : i;
      s[i].values.assign(sigs + i * H, sigs + (i + 1) * H);
    }
    OracleGuard g;
    g.override_refusal = true;
    g.warn_above = ~0ull;
    NearDuplicateSet set = all_pairs_dupset(s, H, SimilarityThreshold{Ratio(thr_num, thr_den)}, g, workers);
    for (size_t i = 0; i < set.doc_ids.size(); ++i) out[i] = set.doc_ids[i];
    *nout = set.doc_ids.size();
  });
}

// union_pairs + components: groups flattened as (rep, member) rows in output
// order (groups sorted by rep, members ascending).
int ref_union(const uint64_t* lo, const uint64_t* hi, uint64_t npairs, uint64_t** rep_out,
              uint64_t** member_out, uint64_t* nrows, uint64_t* ngroups) {
  return guarded([&] {
    std::vector<DuplicatePair> pairs(npairs);
    for (uint64_t i = 0; i < npairs; ++i) pairs[i] = {lo[i], hi[i], 0};
    UnionFind uf = union_pairs(pairs);
    std::vector<DuplicateGroup> groups = components(uf);
    uint64_t rows = 0;
    for (const auto& g : groups) rows += g.members.size();
    *rep_out = static_cast<uint64_t*>(std::malloc(8 * (rows + 1)));
    *member_out = static_cast<uint64_t*>(std::malloc(8 * (rows + 1)));
    uint64_t k = 0;
    for (const auto& g : groups) {
      for (uint64_t m : g.members) {
        (*rep_out)[k] = g.representative;
        (*member_out)[k] = m;
        ++k;
      }
    }
    *nrows = rows;
    *ngroups = groups.size();
  });
}

// generate_synthetic -> packed bytes + offsets (malloc'd) and optionally the
// reference's own JSONL writer (corpus_path non-null).
int ref_generate_synthetic(uint64_t doc_count, uint64_t group_count, uint32_t gmin, uint32_t gmax,
                           uint64_t edit_num, uint64_t edit_den, uint32_t len_min,
                           uint32_t len_max, uint64_t seed, uint32_t L, const char* corpus_path,
                           const char* truth_path, uint8_t** bytes_out, uint64_t** offsets_out,
                           uint64_t* nbytes) {
  return guarded([&] {
    SyntheticSpec spec;
    spec.doc_count = doc_count;
    spec.group_count = group_count;
    spec.group_size_min = gmin;
    spec.group_size_max = gmax;
    spec.edit_rate = Ratio(edit_num, edit_den);
    spec.base_len_min = len_min;
    spec.base_len_max = len_max;
    spec.seed = seed;
    SyntheticCorpus corpus = generate_synthetic(spec, L, ShingleUnit::kByte);
    if (corpus_path && truth_path) write_synthetic(corpus, corpus_path, truth_path);
    uint64_t total = 0;
    for (const auto& t : corpus.texts) total += t.size();
    *bytes_out = static_cast<uint8_t*>(std::malloc(total + 1));
    *offsets_out = static_cast<uint64_t*>(std::malloc(8 * (corpus.texts.size() + 1)));
    uint64_t off = 0;
    for (size_t i = 0; i < corpus.texts.size(); ++i) {
      (*offsets_out)[i] = off;
      std::memcpy(*bytes_out + off, corpus.texts[i].data(), corpus.texts[i].size());
      off += corpus.texts[i].size();
    }
    (*offsets_out)[corpus.texts.size()] = off;
    *nbytes = off;
  });
}

// The reference pipeline as shipped: hash -> gather-compare -> union on a
// JSONL corpus, artifacts in `workspace`.  timings[3] = hash/compare/union s.
int ref_run_dedup(const char* input, const char* workspace, uint32_t H, uint32_t bands,
                  uint32_t rows, uint32_t L, uint64_t thr_num, uint64_t thr_den,
                  uint64_t scale_num, uint64_t scale_den, uint64_t min_chars, uint64_t seed,
                  unsigned workers, uint64_t memory_budget, double* timings,
                  uint64_t* candidate_pairs, uint32_t unit) {
  return guarded([&] {
    RunConfig c;
    c.unit = static_cast<ShingleUnit>(unit);
    c.inputs = {input};
    c.workspace = workspace;
    c.hash_count = H;
    c.bands = bands;
    c.rows = rows;
    c.shingle_len = L;
    c.threshold = Ratio(thr_num, thr_den);
    c.bucket_scale = Ratio(scale_num, scale_den);
    c.min_chars = min_chars;
    c.seed = seed;
    c.workers = workers;
    if (memory_budget) c.memory_budget = memory_budget;
    StageTimings t;
    using clock = std::chrono::steady_clock;
    auto t0 = clock::now();
    run_hash_stage(c);
    auto t1 = clock::now();
    CompareStageOutput cmp = run_compare_stage(c);
    auto t2 = clock::now();
    run_union_stage(c);
    auto t3 = clock::now();
    if (timings) {
      timings[0] = std::chrono::duration<double>(t1 - t0).count();
      timings[1] = std::chrono::duration<double>(t2 - t1).count();
      timings[2] = std::chrono::duration<double>(t3 - t2).count();
    }
    if (candidate_pairs) *candidate_pairs = cmp.candidate_pairs;
  });
}

// run_eval_accuracy over one input (file or directory) with the default
// artifact-shaping parameters except workers / oracle override.
int ref_eval_accuracy(const char* input, const char* workspace, unsigned workers,
                      int oracle_override) {
  return guarded([&] {
    RunConfig c;
    c.inputs = {input};
    c.workspace = workspace;
    c.workers = workers;
    c.oracle_override = oracle_override != 0;
    run_eval_accuracy(c);
  });
}

// build_manifest + surviving_documents (corpus.cpp:109-163) over one input
// (file or directory, expanded like the pipeline); rejects written with
// RejectLog::write_jsonl; survivors returned packed (malloc'd).
int ref_load_corpus(const char* input, const char* text_field, uint64_t min_chars, uint32_t L,
                    uint32_t unit, const char* rejects_path, uint64_t* records,
                    uint64_t* surviving, uint8_t** bytes, uint64_t** offsets, uint64_t** ids,
                    uint64_t** chars) {
  return guarded([&] {
    std::vector<std::string> paths;
    namespace fs = std::filesystem;
    if (fs::is_directory(input)) {
      for (const auto& e : fs::directory_iterator(input))
        if (e.is_regular_file() && e.path().extension() == ".jsonl") paths.push_back(e.path().string());
      std::sort(paths.begin(), paths.end());
    } else {
      paths.push_back(input);
    }
    IngestOptions o;
    o.text_field = text_field;
    o.min_chars = min_chars;
    o.shingle_len = L;
    o.unit = static_cast<ShingleUnit>(unit);
    RejectLog rej;
    CorpusManifest m = build_manifest(paths, o, &rej);
    rej.write_jsonl(rejects_path);
    std::string all;
    std::vector<uint64_t> off{0}, id, ch;
    for (size_t i = 0; i < m.files.size(); ++i)
      for (const CleanDocument& d : surviving_documents(m, i, o)) {
        all += d.text;
        off.push_back(all.size());
        id.push_back(d.doc_id);
        ch.push_back(d.char_count);
      }
    *records = m.total_records;
    *surviving = m.total_surviving;
    *bytes = static_cast<uint8_t*>(std::malloc(all.size() + 1));
    std::memcpy(*bytes, all.data(), all.size());
    auto dup = [](const std::vector<uint64_t>& v) {
      auto* p = static_cast<uint64_t*>(std::malloc(8 * (v.size() + 1)));
      std::memcpy(p, v.data(), 8 * v.size());
      return p;
    };
    *offsets = dup(off);
    *ids = dup(id);
    *chars = dup(ch);
  });
}

}  // extern "C"
