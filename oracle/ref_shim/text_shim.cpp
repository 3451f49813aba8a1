// ICU-free implementation of the reference's text.hpp (TEST INFRASTRUCTURE ONLY).
//
// The reference's src/text.cpp needs ICU headers (text.cpp:3-6) that this image
// does not ship.  This shim provides the same six functions so that the
// reference's own sources can be compiled into oracle/_ref/ as the parity
// checker.  It is exact for input that is already NFC (every synthetic corpus
// here is ASCII, synthetic.cpp:15), which the harness asserts:
//   * text_units (byte)         == text.cpp:115-122 (raw bytes, widened)
//   * decode_codepoints         == U8_NEXT decoding with U+FFFD for ill-formed
//                                  maximal subparts (text.cpp:101-113)
//   * nfc_normalize             == identity on well-formed UTF-8, ill-formed
//                                  subparts rewritten to U+FFFD (text.cpp:70-86)
// This file is never linked into the product library.
#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "neardup/text.hpp"
#include "neardup/util.hpp"

namespace neardup {

std::string_view shingle_unit_name(ShingleUnit unit) {
  return unit == ShingleUnit::kByte ? "byte" : "codepoint";
}

ShingleUnit parse_shingle_unit(std::string_view name) {
  if (name == "byte") return ShingleUnit::kByte;
  if (name == "codepoint") return ShingleUnit::kCodepoint;
  throw ConfigError("unknown shingle unit '" + std::string(name) + "' (expected byte or codepoint)");
}

namespace {

// Decodes one scalar starting at s[i]; advances i past the well-formed
// sequence or past the maximal ill-formed subpart.  Returns -1 when ill-formed.
int32_t next_scalar(const uint8_t* s, size_t& i, size_t len) {
  uint8_t b0 = s[i++];
  if (b0 < 0x80) return b0;
  int need;
  uint32_t cp;
  uint8_t lo = 0x80, hi = 0xBF;
  if (b0 >= 0xC2 && b0 <= 0xDF) {
    need = 1;
    cp = b0 & 0x1F;
  } else if (b0 >= 0xE0 && b0 <= 0xEF) {
    need = 2;
    cp = b0 & 0x0F;
    if (b0 == 0xE0) lo = 0xA0;
    if (b0 == 0xED) hi = 0x9F;
  } else if (b0 >= 0xF0 && b0 <= 0xF4) {
    need = 3;
    cp = b0 & 0x07;
    if (b0 == 0xF0) lo = 0x90;
    if (b0 == 0xF4) hi = 0x8F;
  } else {
    return -1;
  }
  for (int k = 0; k < need; ++k) {
    if (i >= len) return -1;
    uint8_t b = s[i];
    if (b < lo || b > hi) return -1;
    lo = 0x80;
    hi = 0xBF;
    cp = (cp << 6) | (b & 0x3F);
    ++i;
  }
  return static_cast<int32_t>(cp);
}

}  // namespace

std::string nfc_normalize(std::string_view utf8) {
  std::string out;
  out.reserve(utf8.size());
  const auto* s = reinterpret_cast<const uint8_t*>(utf8.data());
  size_t i = 0;
  while (i < utf8.size()) {
    size_t start = i;
    int32_t c = next_scalar(s, i, utf8.size());
    if (c < 0) {
      out.append("\xef\xbf\xbd");
    } else {
      out.append(utf8.substr(start, i - start));
    }
  }
  return out;
}

uint64_t codepoint_count(std::string_view utf8) {
  const auto* s = reinterpret_cast<const uint8_t*>(utf8.data());
  uint64_t count = 0;
  size_t i = 0;
  while (i < utf8.size()) {
    next_scalar(s, i, utf8.size());
    ++count;
  }
  return count;
}

std::vector<uint32_t> decode_codepoints(std::string_view utf8) {
  const auto* s = reinterpret_cast<const uint8_t*>(utf8.data());
  std::vector<uint32_t> out;
  out.reserve(utf8.size());
  size_t i = 0;
  while (i < utf8.size()) {
    int32_t c = next_scalar(s, i, utf8.size());
    out.push_back(c < 0 ? 0xFFFDu : static_cast<uint32_t>(c));
  }
  return out;
}

std::vector<uint32_t> text_units(std::string_view utf8, ShingleUnit unit) {
  if (unit == ShingleUnit::kCodepoint) return decode_codepoints(utf8);
  std::vector<uint32_t> out(utf8.size());
  for (size_t i = 0; i < utf8.size(); ++i) out[i] = static_cast<unsigned char>(utf8[i]);
  return out;
}

}  // namespace neardup
