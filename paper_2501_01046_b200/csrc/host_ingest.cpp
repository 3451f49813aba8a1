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
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

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

// Fast path for parse_jsonl_line: a recursive-descent scanner for a strict
// SUBSET of the JSON nlohmann accepts -- objects, arrays, strings whose
// escapes are the single-character ones, well-formed UTF-8 (Unicode Table
// 3-7, the ranges nlohmann's lexer checks), integers of at most 18 digits,
// true/false/null, whitespace ' ' '\t' '\n' '\r'.  Inside that subset
// nlohmann accepts exactly the same lines and decodes the same text; anything
// else (\u escapes, fractions/exponents, long numbers, a BOM, deep nesting,
// every error) returns -1 and the line goes to nlohmann, whose verdict is
// then final.  *ascii: the captured text is pure ASCII.
namespace {
struct Fast {
  const unsigned char* p;
  const unsigned char* e;
  const std::string* field;
  std::string* text;
  bool top_object = false, found = false, is_string = false, ascii = true;
  static bool ws(unsigned c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
  void skip() {
    while (p < e && ws(*p)) ++p;
  }
  // string body after the opening quote; out may be null (validate only)
  bool str(std::string* out, bool* asc) {
    const unsigned char* run = p;
    for (;;) {
      while (p < e && *p >= 0x20 && *p < 0x80 && *p != '"' && *p != '\\') ++p;
      if (p >= e) return false;
      const unsigned c = *p;
      if (c == '"') {
        if (out) out->append(reinterpret_cast<const char*>(run), p - run);
        ++p;
        return true;
      }
      if (c < 0x20) return false;
      if (c == '\\') {
        if (out) out->append(reinterpret_cast<const char*>(run), p - run);
        if (p + 1 >= e) return false;
        char d;
        switch (p[1]) {
          case '"': d = '"'; break;
          case '\\': d = '\\'; break;
          case '/': d = '/'; break;
          case 'b': d = '\b'; break;
          case 'f': d = '\f'; break;
          case 'n': d = '\n'; break;
          case 'r': d = '\r'; break;
          case 't': d = '\t'; break;
          default: return false;  // \u.. and invalid escapes: nlohmann decides
        }
        if (out) out->push_back(d);
        p += 2;
        run = p;
        continue;
      }
      // c >= 0x80: one well-formed UTF-8 sequence
      size_t i = static_cast<size_t>(p - run), len = static_cast<size_t>(e - run);
      if (next_cp(run, i, len) < 0) return false;
      if (asc) *asc = false;
      p = run + i;
    }
  }
  bool number() {
    if (p < e && *p == '-') ++p;
    if (p >= e || *p < '0' || *p > '9') return false;
    const unsigned char* d0 = p;
    if (*p == '0') {
      ++p;
    } else {
      while (p < e && *p >= '0' && *p <= '9') ++p;
    }
    if (p - d0 > 18) return false;
    if (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E')) return false;
    return true;
  }
  bool lit(const char* w, size_t n) {
    if (static_cast<size_t>(e - p) < n || std::memcmp(p, w, n) != 0) return false;
    p += n;
    return true;
  }
  // capture: this value is the field's value at depth 1
  bool value(int depth, bool capture) {
    if (p >= e || depth > 64) return false;
    const unsigned c = *p;
    if (capture) {
      found = true;
      is_string = c == '"';
    }
    switch (c) {
      case '"': {
        ++p;
        if (capture) {
          text->clear();
          ascii = true;
          return str(text, &ascii);
        }
        return str(nullptr, nullptr);
      }
      case '{': {
        ++p;
        skip();
        if (p < e && *p == '}') {
          ++p;
          return true;
        }
        for (;;) {
          if (p >= e || *p != '"') return false;
          ++p;
          bool match = false;
          if (depth == 0) {
            key.clear();
            if (!str(&key, nullptr)) return false;
            match = key == *field;
          } else if (!str(nullptr, nullptr)) {
            return false;
          }
          skip();
          if (p >= e || *p != ':') return false;
          ++p;
          skip();
          if (!value(depth + 1, match)) return false;
          skip();
          if (p < e && *p == ',') {
            ++p;
            skip();
            continue;
          }
          if (p < e && *p == '}') {
            ++p;
            return true;
          }
          return false;
        }
      }
      case '[': {
        ++p;
        skip();
        if (p < e && *p == ']') {
          ++p;
          return true;
        }
        for (;;) {
          if (!value(depth + 1, false)) return false;
          skip();
          if (p < e && *p == ',') {
            ++p;
            skip();
            continue;
          }
          if (p < e && *p == ']') {
            ++p;
            return true;
          }
          return false;
        }
      }
      case 't': return lit("true", 4);
      case 'f': return lit("false", 5);
      case 'n': return lit("null", 4);
      default: return number();
    }
  }
  std::string key;
};
}  // namespace

int parse_jsonl_line_fast(std::string_view line, const std::string& field, std::string& text,
                          bool* ascii) {
  Fast f;
  f.p = reinterpret_cast<const unsigned char*>(line.data());
  f.e = f.p + line.size();
  f.field = &field;
  f.text = &text;
  if (line.size() >= 3 && f.p[0] == 0xEF && f.p[1] == 0xBB && f.p[2] == 0xBF) return -1;  // BOM
  f.skip();
  f.top_object = f.p < f.e && *f.p == '{';
  if (!f.value(0, false)) return -1;
  f.skip();
  if (f.p != f.e) return -1;
  if (!f.top_object) return 2;
  if (!f.found) return 3;
  if (!f.is_string) return 4;
  if (ascii) *ascii = f.ascii;
  return 0;
}

int parse_jsonl_line(std::string_view line, const std::string& field, std::string& text) {
  const int r = parse_jsonl_line_fast(line, field, text, nullptr);
  if (r >= 0) return r;
  return parse_jsonl_line_nlohmann(line, field, text);
}

int parse_jsonl_line_nlohmann(std::string_view line, const std::string& field, std::string& text) {
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
  const int fd = open(path.c_str(), O_RDONLY);
  if (fd < 0) fail(ND_ERR_IO, "cannot open '" + path + "': " + std::strerror(errno));
  struct stat sb;
  if (fstat(fd, &sb) != 0) {
    close(fd);
    fail(ND_ERR_IO, "read failed for '" + path + "'");
  }
  const size_t size = static_cast<size_t>(sb.st_size);
  const char* buf = nullptr;
  void* map = MAP_FAILED;
  if (size) {
    map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (map == MAP_FAILED) {
      close(fd);
      fail(ND_ERR_IO, "read failed for '" + path + "'");
    }
    madvise(map, size, MADV_SEQUENTIAL);
    buf = static_cast<const char*>(map);
  }
  close(fd);
  struct Unmap {
    void* m;
    size_t n;
    ~Unmap() {
      if (m != MAP_FAILED) munmap(m, n);
    }
  } unmap{map, size};

  // T byte ranges, each starting at a line start (getline semantics: lines end
  // at '\n'; a final line without '\n' counts, nothing after a final '\n')
  if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
  threads = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(threads, size / (1 << 16))));
  std::vector<size_t> cut(threads + 1, size);
  cut[0] = 0;
  for (unsigned t = 1; t < threads; ++t) {
    size_t c = std::max(cut[t - 1], size * t / threads);
    const void* nl = c < size ? std::memchr(buf + c, '\n', size - c) : nullptr;
    cut[t] = nl ? static_cast<size_t>(static_cast<const char*>(nl) - buf) + 1 : size;
  }
  out = JsonlFile{};
  out.blocks.resize(threads);
  auto work = [&](unsigned t) {
    JsonlFile::Block& b = out.blocks[t];
    std::string text, norm;
    size_t a = cut[t];
    const size_t end = cut[t + 1];
    if (keep_text) b.bytes.reserve(end - a);  // decoded text is at most the line bytes, bar NFC growth
    while (a < end) {
      const void* nl = std::memchr(buf + a, '\n', end - a);
      const size_t stop = nl ? static_cast<size_t>(static_cast<const char*>(nl) - buf) : end;
      const uint64_t line_no = ++b.lines;  // local; made global after the join
      size_t e = stop;
      const size_t next = nl ? stop + 1 : end;
      if (e > a && buf[e - 1] == '\r') --e;
      if (e == a) {
        a = next;
        continue;
      }
      const std::string_view line(buf + a, e - a);
      a = next;
      bool ascii = false;
      int why = parse_jsonl_line_fast(line, field, text, &ascii);
      if (why < 0) {
        ascii = false;
        why = parse_jsonl_line(line, field, text);
      }
      if (why) {
        b.rejects.push_back({line_no, static_cast<uint8_t>(why)});
        continue;
      }
      const uint64_t ord = b.records++;
      // ASCII text is NFC and has one code point per byte
      const std::string& clean = ascii || nfc_normalize_into(text, norm) ? text : norm;
      const uint64_t chars = ascii ? clean.size() : codepoint_count(clean);
      if (chars < min_chars) {
        b.rejects.push_back({line_no, 5});
        continue;
      }
      const uint64_t units = unit == 0 ? clean.size() : chars;
      if (units < shingle_len) {
        b.rejects.push_back({line_no, 6});
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
  // local line numbers and ordinals -> global
  uint64_t lines = 0, records = 0;
  for (auto& b : out.blocks) {
    b.line_base = lines;
    b.record_base = records;
    b.doc_base = out.surviving;
    b.byte_base = out.text_bytes;
    for (auto& r : b.rejects) r.first += lines;
    lines += b.lines;
    records += b.records;
    out.surviving += b.ordinal.size();
    out.text_bytes += b.bytes.size();
  }
  out.records = records;
  out.nrejects = 0;
  for (auto& b : out.blocks) out.nrejects += b.rejects.size();
}

// survivors into caller buffers, one thread per block
void jsonl_documents(const JsonlFile& f, uint64_t record_offset, uint8_t* bytes,
                     uint64_t* offsets, uint64_t* doc_ids, uint64_t* char_counts) {
  auto copy = [&](size_t t) {
    const JsonlFile::Block& b = f.blocks[t];
    uint64_t o = b.byte_base;
    if (bytes && !b.bytes.empty()) std::memcpy(bytes + b.byte_base, b.bytes.data(), b.bytes.size());
    for (size_t k = 0; k < b.ordinal.size(); ++k) {
      const uint64_t i = b.doc_base + k;
      if (doc_ids) doc_ids[i] = record_offset + b.record_base + b.ordinal[k];
      if (char_counts) char_counts[i] = b.chars[k];
      if (offsets) {
        offsets[i] = o;
        o += b.lens[k];
      }
    }
  };
  std::vector<std::thread> th;
  for (size_t t = 1; t < f.blocks.size(); ++t) th.emplace_back(copy, t);
  if (!f.blocks.empty()) copy(0);
  for (auto& x : th) x.join();
  if (offsets) offsets[f.surviving] = f.text_bytes;
}

}  // namespace ndb
