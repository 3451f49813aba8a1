// Host document loader: the reference's corpus.cpp / text.cpp path as a
// multi-threaded C++ pass over each JSONL file.
//
//   line split        for_each_raw_document (corpus.cpp:56-82): '\n' lines, one
//                     trailing '\r' dropped, blank lines are neither records nor
//                     rejects, record ordinals count valid records
//   parse_jsonl_line  corpus.cpp:31-54 with the same parser (nlohmann::json, so
//                     acceptance -- including its UTF-8 and surrogate checks --
//                     and the decoded text are the reference's)
//   nfc_normalize     text.cpp:70-86: ill-formed UTF-8 -> U+FFFD per maximal
//                     subpart, then Unicode NFC (UAX #15) from the tables in
//                     unicode_tables.inc (ICU in the reference); a quick check
//                     (ASCII, or NFC_QC=Yes with ordered combining classes)
//                     returns most texts untouched
//   codepoint_count   text.cpp:88-99
//   preprocess / can_shingle / build_manifest filters (corpus.cpp:93-141):
//                     "below_min_chars", "too_short_to_shingle"
// Lines are split into contiguous blocks, one per thread; ordinals and the
// reject log are stitched back in line order, so the result is independent
// of the thread count.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include <nlohmann/json.hpp>

#include "host_internal.hpp"

namespace ndb {
namespace {

#include "unicode_tables.inc"

constexpr uint16_t kQcNo = 1u << 8, kQcMaybe = 1u << 9;
constexpr uint32_t SBase = 0xAC00, LBase = 0x1100, VBase = 0x1161, TBase = 0x11A7;
constexpr uint32_t LCount = 19, VCount = 21, TCount = 28, NCount = VCount * TCount,
                   SCount = LCount * NCount;

inline uint16_t ucd(uint32_t cp) { return cp < 0x110000 ? kUcdBlocks[kUcdIndex[cp >> 8]][cp & 255] : 0; }
inline uint32_t ccc(uint32_t cp) { return ucd(cp) & 0xFF; }

// U8_NEXT-equivalent decode step (Unicode Table 3-7); -1 = ill-formed
// maximal subpart, i advanced past it
int32_t next_cp(const uint8_t* s, size_t& i, size_t len) {
  const uint32_t b0 = s[i++];
  if (b0 < 0x80) return static_cast<int32_t>(b0);
  int need;
  uint32_t c, lo = 0x80, hi = 0xBF;
  if (b0 >= 0xC2 && b0 <= 0xDF) {
    need = 1;
    c = b0 & 0x1F;
  } else if (b0 >= 0xE0 && b0 <= 0xEF) {
    need = 2;
    c = b0 & 0x0F;
    if (b0 == 0xE0) lo = 0xA0;
    if (b0 == 0xED) hi = 0x9F;
  } else if (b0 >= 0xF0 && b0 <= 0xF4) {
    need = 3;
    c = b0 & 0x07;
    if (b0 == 0xF0) lo = 0x90;
    if (b0 == 0xF4) hi = 0x8F;
  } else {
    return -1;
  }
  for (int k = 0; k < need; ++k) {
    if (i >= len) return -1;
    const uint32_t b = s[i];
    if (b < lo || b > hi) return -1;
    lo = 0x80;
    hi = 0xBF;
    c = (c << 6) | (b & 0x3F);
    ++i;
  }
  return static_cast<int32_t>(c);
}

void put_utf8(std::string& out, uint32_t c) {
  if (c < 0x80) {
    out += static_cast<char>(c);
  } else if (c < 0x800) {
    out += static_cast<char>(0xC0 | (c >> 6));
    out += static_cast<char>(0x80 | (c & 0x3F));
  } else if (c < 0x10000) {
    out += static_cast<char>(0xE0 | (c >> 12));
    out += static_cast<char>(0x80 | ((c >> 6) & 0x3F));
    out += static_cast<char>(0x80 | (c & 0x3F));
  } else {
    out += static_cast<char>(0xF0 | (c >> 18));
    out += static_cast<char>(0x80 | ((c >> 12) & 0x3F));
    out += static_cast<char>(0x80 | ((c >> 6) & 0x3F));
    out += static_cast<char>(0x80 | (c & 0x3F));
  }
}

void decompose(uint32_t c, std::vector<uint32_t>& out) {
  if (c >= SBase && c < SBase + SCount) {  // Hangul (UAX #15 / ch. 3.12)
    const uint32_t s = c - SBase;
    out.push_back(LBase + s / NCount);
    out.push_back(VBase + (s % NCount) / TCount);
    if (s % TCount) out.push_back(TBase + s % TCount);
    return;
  }
  const uint32_t* k = std::lower_bound(std::begin(kDecompKeys), std::end(kDecompKeys), c);
  if (k != std::end(kDecompKeys) && *k == c) {
    const size_t i = static_cast<size_t>(k - kDecompKeys);
    out.insert(out.end(), kDecompPool + kDecompOff[i], kDecompPool + kDecompOff[i + 1]);
  } else {
    out.push_back(c);
  }
}

// primary composite of (a, b) or 0
uint32_t compose_pair(uint32_t a, uint32_t b) {
  if (a >= LBase && a < LBase + LCount && b >= VBase && b < VBase + VCount)
    return SBase + ((a - LBase) * VCount + (b - VBase)) * TCount;
  if (a >= SBase && a < SBase + SCount && (a - SBase) % TCount == 0 && b > TBase &&
      b < TBase + TCount)
    return a + (b - TBase);
  const uint64_t key = (static_cast<uint64_t>(a) << 21) | b;
  const uint64_t* k = std::lower_bound(std::begin(kCompKeys), std::end(kCompKeys), key);
  if (k != std::end(kCompKeys) && *k == key) return kCompVals[k - kCompKeys];
  return 0;
}

}  // namespace

// text.cpp:70-86.  Returns true and leaves `out` untouched when `in` is
// already well-formed NFC (the common case); otherwise writes the result.
bool nfc_normalize_into(std::string_view in, std::string& out) {
  const auto* s = reinterpret_cast<const uint8_t*>(in.data());
  const size_t len = in.size();
  size_t i = 0;
  while (i < len && s[i] < 0x80) ++i;
  if (i == len) return true;  // ASCII
  // quick check over the rest: well-formed, NFC_QC=Yes, combining classes in order
  bool quick = true;
  uint32_t last = 0;
  for (size_t j = i; j < len;) {
    if (s[j] < 0x80) {
      ++j;
      last = 0;
      continue;
    }
    const int32_t c = next_cp(s, j, len);
    if (c < 0) {
      quick = false;
      break;
    }
    const uint16_t f = ucd(static_cast<uint32_t>(c));
    const uint32_t cc = f & 0xFF;
    if ((f & (kQcNo | kQcMaybe)) || (cc && last > cc)) {
      quick = false;
      break;
    }
    last = cc;
  }
  if (quick) return true;
  // decode (ill-formed -> U+FFFD) + full canonical decomposition
  std::vector<uint32_t> d;
  d.reserve(len);
  for (size_t j = 0; j < len;) {
    const int32_t c = next_cp(s, j, len);
    decompose(c < 0 ? 0xFFFDu : static_cast<uint32_t>(c), d);
  }
  // canonical ordering: stable sort of each run of non-starters by class
  for (size_t a = 0; a < d.size();) {
    if (ccc(d[a]) == 0) {
      ++a;
      continue;
    }
    size_t b = a;
    while (b < d.size() && ccc(d[b]) != 0) ++b;
    std::stable_sort(d.begin() + a, d.begin() + b,
                     [](uint32_t x, uint32_t y) { return ccc(x) < ccc(y); });
    a = b;
  }
  // canonical composition (UAX #15 sample algorithm)
  if (!d.empty()) {
    size_t starter = 0, w = 1;
    uint32_t last_cc = ccc(d[0]);
    if (last_cc != 0) last_cc = 256;  // text starting with a non-starter
    for (size_t r = 1; r < d.size(); ++r) {
      const uint32_t c = d[r], cc = ccc(c);
      const uint32_t comp = compose_pair(d[starter], c);
      if (comp && (last_cc < cc || last_cc == 0)) {
        d[starter] = comp;
        continue;
      }
      if (cc == 0) starter = w;
      last_cc = cc;
      d[w++] = c;
    }
    d.resize(w);
  }
  out.clear();
  out.reserve(len);
  for (uint32_t c : d) put_utf8(out, c);
  return false;
}

std::string nfc_normalize(std::string_view in) {
  std::string out;
  if (nfc_normalize_into(in, out)) return std::string(in);
  return out;
}

// text.cpp:88-99 (ill-formed bytes count one per maximal subpart)
uint64_t codepoint_count(std::string_view t) {
  const auto* s = reinterpret_cast<const uint8_t*>(t.data());
  uint64_t n = 0;
  for (size_t i = 0; i < t.size();) {
    if (s[i] < 0x80) {
      ++i;
    } else {
      next_cp(s, i, t.size());
    }
    ++n;
  }
  return n;
}

// parse_jsonl_line (corpus.cpp:31-54); reason codes: 0 ok, 1 invalid_json,
// 2 not_an_object, 3 missing_text_field, 4 text_field_not_string.
// nlohmann's SAX interface drives the same lexer and parser as the DOM parse
// the reference does (so acceptance is identical) without building the DOM;
// the DOM's object insertion keeps the LAST value of a repeated key, and so
// does this handler.
namespace {
struct FieldSax {
  const std::string* field;
  std::string* text;
  int depth = 0;
  bool top_object = false, first = true, pending = false, found = false, is_string = false;
  void value_event(bool str) {
    if (first) {
      first = false;
      top_object = false;
    }
    if (depth == 1 && pending) {
      found = true;
      is_string = str;
      pending = false;
    }
  }
  bool null() { value_event(false); return true; }
  bool boolean(bool) { value_event(false); return true; }
  bool number_integer(nlohmann::json::number_integer_t) { value_event(false); return true; }
  bool number_unsigned(nlohmann::json::number_unsigned_t) { value_event(false); return true; }
  bool number_float(nlohmann::json::number_float_t, const std::string&) {
    value_event(false);
    return true;
  }
  bool string(std::string& v) {
    const bool take = depth == 1 && pending;
    value_event(true);
    if (take) text->swap(v);
    return true;
  }
  bool binary(nlohmann::json::binary_t&) { value_event(false); return true; }
  bool start_object(std::size_t) {
    if (first) {
      first = false;
      top_object = true;
    } else {
      value_event(false);
    }
    ++depth;
    return true;
  }
  bool key(std::string& k) {
    if (depth == 1) pending = k == *field;
    return true;
  }
  bool end_object() { --depth; return true; }
  bool start_array(std::size_t) {
    if (first) {
      first = false;
      top_object = false;
    } else {
      value_event(false);
    }
    ++depth;
    return true;
  }
  bool end_array() { --depth; return true; }
  bool parse_error(std::size_t, const std::string&, const nlohmann::detail::exception&) {
    return false;
  }
};
}  // namespace

int parse_jsonl_line(std::string_view line, const std::string& field, std::string& text) {
  FieldSax h;
  h.field = &field;
  h.text = &text;
  if (!nlohmann::json::sax_parse(line, &h, nlohmann::json::input_format_t::json, true)) return 1;
  if (!h.top_object) return 2;
  if (!h.found) return 3;
  if (!h.is_string) return 4;
  return 0;
}

// One file: records, surviving documents (packed), rejects in line order.
void load_jsonl(const std::string& path, const std::string& field, uint64_t min_chars,
                uint32_t shingle_len, uint32_t unit, unsigned threads, bool keep_text,
                JsonlFile& out) {
  if (shingle_len == 0) fail(ND_ERR_CONFIG, "shingle length must be positive");
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) fail(ND_ERR_IO, "cannot open '" + path + "': " + std::strerror(errno));
  std::string buf;
  {
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
    const bool ok = buf.empty() || std::fread(buf.data(), 1, buf.size(), f) == buf.size();
    std::fclose(f);
    if (!ok) fail(ND_ERR_IO, "read failed for '" + path + "'");
  }
  // line starts (std::getline semantics: a final line without '\n' counts)
  std::vector<size_t> starts;
  starts.push_back(0);
  for (const char* p = buf.data(); (p = static_cast<const char*>(std::memchr(p, '\n', buf.data() + buf.size() - p)));) {
    ++p;
    starts.push_back(static_cast<size_t>(p - buf.data()));
  }
  if (starts.back() == buf.size()) starts.pop_back();  // no line after the final '\n'
  const size_t nlines = starts.size();
  starts.push_back(buf.size() + 1);  // sentinel: end of the last line (+1 for its '\n')

  struct Block {
    uint64_t records = 0;
    std::vector<std::pair<uint64_t, uint8_t>> rejects;  // (line, reason)
    std::string bytes;
    std::vector<uint64_t> lens, ordinal, chars;         // ordinal: within the block
  };
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = static_cast<unsigned>(std::min<size_t>(threads, std::max<size_t>(1, nlines / 256)));
  std::vector<Block> blocks(threads);
  auto work = [&](unsigned t) {
    Block& b = blocks[t];
    const size_t l0 = nlines * t / threads, l1 = nlines * (t + 1) / threads;
    std::string text, norm;
    for (size_t l = l0; l < l1; ++l) {
      size_t a = starts[l], e = starts[l + 1] - 1;  // [a, e) without '\n'
      if (e > a && buf[e - 1] == '\r') --e;
      if (e == a) continue;
      const int why = parse_jsonl_line(std::string_view(buf.data() + a, e - a), field, text);
      if (why) {
        b.rejects.push_back({l + 1, static_cast<uint8_t>(why)});
        continue;
      }
      const uint64_t ord = b.records++;
      const std::string& clean = nfc_normalize_into(text, norm) ? text : norm;
      const uint64_t chars = codepoint_count(clean);
      if (chars < min_chars) {
        b.rejects.push_back({l + 1, 5});
        continue;
      }
      const uint64_t units = unit == 0 ? clean.size() : chars;
      if (units < shingle_len) {
        b.rejects.push_back({l + 1, 6});
        continue;
      }
      b.ordinal.push_back(ord);
      b.chars.push_back(chars);
      if (keep_text) {
        b.bytes += clean;
        b.lens.push_back(clean.size());
      }
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < threads; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();

  out = JsonlFile{};
  uint64_t base = 0, nbytes = 0, ndocs = 0;
  for (auto& b : blocks) {
    ndocs += b.ordinal.size();
    nbytes += b.bytes.size();
  }
  out.ordinal.reserve(ndocs);
  out.chars.reserve(ndocs);
  if (keep_text) {
    out.bytes.reserve(nbytes);
    out.offsets.reserve(ndocs + 1);
    out.offsets.push_back(0);
  }
  for (auto& b : blocks) {
    for (auto& r : b.rejects) out.rejects.push_back(r);
    for (size_t k = 0; k < b.ordinal.size(); ++k) {
      out.ordinal.push_back(base + b.ordinal[k]);
      out.chars.push_back(b.chars[k]);
      if (keep_text) out.offsets.push_back(out.offsets.back() + b.lens[k]);
    }
    if (keep_text) out.bytes += b.bytes;
    base += b.records;
    std::string().swap(b.bytes);
  }
  out.records = base;
}

}  // namespace ndb
