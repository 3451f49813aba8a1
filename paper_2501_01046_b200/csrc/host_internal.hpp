// Host-only internals (compiled by g++/nvcc host pass; no CUDA types).
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "neardup_b200.h"

namespace ndb {

// Exceptions mapped to ND_ERR_* at the C-ABI boundary (nd_capi.cu).
struct NdError : std::runtime_error {
  int code;
  NdError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw NdError(code, msg); }

uint64_t bounded_random(std::mt19937_64& rng, uint64_t bound);
std::vector<nd_hash_fn> derive_family(uint64_t seed, uint32_t H, uint32_t L, uint32_t unit);
uint32_t choose_bucket_count(uint64_t n, uint64_t num, uint64_t den);
uint32_t min_matches(uint32_t H, uint64_t num, uint64_t den);
uint64_t mod_pow_checked(uint64_t base, uint64_t exp, uint64_t mod);
bool is_prime(uint32_t n);
uint32_t hash_window_direct(const uint32_t* w, uint32_t len, const nd_hash_fn& f);
uint32_t roll_next(uint32_t state, uint32_t outgoing, uint32_t incoming, const nd_hash_fn& f);

// synthetic corpus (synth.cu)
void synth_generate(const nd_synth_spec& spec, uint8_t* bytes, uint64_t* offsets,
                    uint64_t* nbytes_out);

// report writers (host_report.cpp): groups as doc ids in output order
void write_report(const std::string& dir, const std::vector<uint64_t>& members,
                  const std::vector<uint64_t>& group_start, const std::vector<uint64_t>& near,
                  const std::vector<uint64_t>& removals, uint64_t total_documents,
                  uint64_t total_records, uint64_t distinct_pairs, bool fsync_files = false);

// staged-workflow artifacts (host_feds.cpp)
constexpr uint64_t kFedsHeaderBytes = 72;
uint64_t feds_record_bytes(const nd_feds_header& h);
std::string feds_serialize(const nd_feds_header& h);
nd_feds_header feds_read_header(const std::string& path, uint64_t* file_size);
bool feds_run_compatible(const nd_feds_header& a, const nd_feds_header& b);
void feds_write(const std::string& path, nd_feds_header h, const uint64_t* doc_ids,
                const uint32_t* sig, const uint32_t* band, uint64_t n, bool fsync_file);
void feds_read_records(const std::string& path, const nd_feds_header& h, uint64_t* doc_ids,
                       uint32_t* sig, uint32_t* band);
void pairs_write(const std::string& path, const uint64_t* lo, const uint64_t* hi,
                 const uint32_t* m, uint64_t n, bool fsync_file);
void pairs_read(const std::string& path, std::vector<uint64_t>& lo, std::vector<uint64_t>& hi,
                std::vector<uint32_t>& m);
uint32_t plan_gather(uint64_t total_bytes, uint32_t K, const std::vector<uint32_t>& worker_bands,
                     uint64_t budget, uint32_t override_c, std::vector<uint32_t>& passes);

// document loader (host_ingest.cpp)
struct JsonlFile {
  struct Block {                                      // one thread's contiguous lines
    uint64_t lines = 0, records = 0;                  // local counts
    uint64_t line_base = 0, record_base = 0, doc_base = 0, byte_base = 0;
    std::vector<std::pair<uint64_t, uint8_t>> rejects;  // (1-based global line, reason)
    std::vector<uint64_t> ordinal, chars, lens;       // per survivor (ordinal: local)
    std::string bytes;                                // survivors' NFC text (keep_text)
  };
  std::vector<Block> blocks;
  uint64_t records = 0, surviving = 0, text_bytes = 0, nrejects = 0;
};
void load_jsonl(const std::string& path, const std::string& field, uint64_t min_chars,
                uint32_t shingle_len, uint32_t unit, unsigned threads, bool keep_text,
                JsonlFile& out);
void jsonl_documents(const JsonlFile& f, uint64_t record_offset, uint8_t* bytes,
                     uint64_t* offsets, uint64_t* doc_ids, uint64_t* char_counts);
bool nfc_normalize_into(std::string_view in, std::string& out);
std::string nfc_normalize(std::string_view in);
uint64_t codepoint_count(std::string_view t);
int parse_jsonl_line(std::string_view line, const std::string& field, std::string& text);
int parse_jsonl_line_nlohmann(std::string_view line, const std::string& field, std::string& text);
// strict-subset fast path; -1 = undecided (use parse_jsonl_line)
int parse_jsonl_line_fast(std::string_view line, const std::string& field, std::string& text,
                          bool* ascii);

}  // namespace ndb
