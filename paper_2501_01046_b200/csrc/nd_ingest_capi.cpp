// C-ABI of the host document loader (host_ingest.cpp); see include/neardup_b200.h.
#include <cstring>
#include <string>

#include "host_internal.hpp"

struct nd_jsonl {
  ndb::JsonlFile f;
  bool keep_text = false;
};

namespace {
thread_local std::string g_ingest_error;

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return ND_OK;
  } catch (const ndb::NdError& e) {
    g_ingest_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_ingest_error = e.what();
    return ND_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* nd_ingest_last_error(void) { return g_ingest_error.c_str(); }

int nd_jsonl_load(const char* path, const char* text_field, uint64_t min_chars,
                  uint32_t shingle_len, uint32_t unit, uint32_t threads, int keep_text,
                  nd_jsonl** out) {
  return guarded([&] {
    if (!path || !text_field || !out) ndb::fail(ND_ERR_CONFIG, "null argument");
    if (unit > 1) ndb::fail(ND_ERR_CONFIG, "unknown shingle unit");
    auto* h = new nd_jsonl();
    try {
      ndb::load_jsonl(path, text_field, min_chars, shingle_len, unit, threads, keep_text != 0, h->f);
    } catch (...) {
      delete h;
      throw;
    }
    h->keep_text = keep_text != 0;
    *out = h;
  });
}

void nd_jsonl_counts(const nd_jsonl* h, uint64_t* records, uint64_t* surviving,
                     uint64_t* text_bytes, uint64_t* rejects) {
  if (records) *records = h->f.records;
  if (surviving) *surviving = h->f.surviving;
  if (text_bytes) *text_bytes = h->f.text_bytes;
  if (rejects) *rejects = h->f.nrejects;
}

int nd_jsonl_rejects(const nd_jsonl* h, uint64_t* lines, uint32_t* reasons) {
  return guarded([&] {
    size_t i = 0;
    for (const auto& b : h->f.blocks)
      for (const auto& r : b.rejects) {
        if (lines) lines[i] = r.first;
        if (reasons) reasons[i] = r.second;
        ++i;
      }
  });
}

int nd_jsonl_documents(const nd_jsonl* h, uint64_t record_offset, uint8_t* bytes,
                       uint64_t* offsets, uint64_t* doc_ids, uint64_t* char_counts) {
  return guarded([&] {
    if ((bytes || offsets) && !h->keep_text)
      ndb::fail(ND_ERR_CONFIG, "loaded without keep_text; no document text kept");
    ndb::jsonl_documents(h->f, record_offset, bytes, offsets, doc_ids, char_counts);
  });
}

void nd_jsonl_free(nd_jsonl* h) { delete h; }

int nd_nfc_normalize(const uint8_t* in, uint64_t len, uint8_t* out, uint64_t cap,
                     uint64_t* out_len) {
  return guarded([&] {
    std::string r = ndb::nfc_normalize(std::string_view(reinterpret_cast<const char*>(in), len));
    *out_len = r.size();
    if (out && cap >= r.size() && !r.empty()) std::memcpy(out, r.data(), r.size());
  });
}

uint64_t nd_codepoint_count(const uint8_t* s, uint64_t len) {
  return ndb::codepoint_count(std::string_view(reinterpret_cast<const char*>(s), len));
}

int nd_parse_jsonl_line(const char* line, uint64_t len, const char* field, uint32_t* reason,
                        uint8_t* text_out, uint64_t cap, uint64_t* text_len) {
  return nd_parse_jsonl_line_mode(line, len, field, 0, reason, text_out, cap, text_len);
}

int nd_parse_jsonl_line_mode(const char* line, uint64_t len, const char* field, int mode,
                             uint32_t* reason, uint8_t* text_out, uint64_t cap,
                             uint64_t* text_len) {
  return guarded([&] {
    std::string t;
    const std::string f(field);
    const std::string_view v(line, len);
    int r;
    if (mode == 2) {
      r = ndb::parse_jsonl_line_fast(v, f, t, nullptr);
      if (r < 0) r = 255;
    } else if (mode == 1) {
      r = ndb::parse_jsonl_line_nlohmann(v, f, t);
    } else {
      r = ndb::parse_jsonl_line(v, f, t);
    }
    *reason = static_cast<uint32_t>(r);
    *text_len = t.size();
    if (text_out && cap >= t.size() && !t.empty()) std::memcpy(text_out, t.data(), t.size());
  });
}

}  // extern "C"
