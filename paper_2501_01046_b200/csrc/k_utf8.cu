// Codepoint shingle units on the GPU: UTF-8 -> Unicode scalar values.
//
// Replaces text_units(.., kCodepoint) = decode_codepoints (text.cpp:101-113):
// ICU's U8_NEXT walk, one unit per well-formed sequence and one U+FFFD per
// maximal ill-formed subpart (a lead byte followed by the longest valid prefix
// of its trail bytes; a stray trail byte or an invalid lead is a subpart of
// one byte).
//
// The decoder's unit boundaries are LOCAL: a byte that is not a trail byte
// (10xxxxxx) always starts a unit (no sequence ever consumes it), and a trail
// byte at i belongs to the unit started by the nearest non-trail byte j in
// [i-3, i-1] iff that unit's length exceeds i-j; otherwise it is a one-byte
// ill-formed unit of its own.  So every byte position decides "starts a
// unit?" and "which value?" from at most 3 bytes behind and 3 ahead, and one
// warp walks a document 32 bytes per step: ballot + popc rank the unit
// starts, the first pass counts units per document, the second writes them.
#include "nd_internal.cuh"

namespace ndb {
namespace {

__device__ __forceinline__ bool is_trail(uint32_t b) { return (b & 0xC0u) == 0x80u; }

// The unit starting at s[j] (j < len): its length in bytes and its value
// (the scalar, or 0xFFFD when ill-formed).  Same acceptance ranges as U8_NEXT
// (Unicode Table 3-7: E0 A0..BF, ED 80..9F, F0 90..BF, F4 80..8F).
__device__ __forceinline__ int unit_at(const uint8_t* __restrict__ s, uint64_t len, uint64_t j,
                                       uint32_t& cp) {
  const uint32_t b0 = s[j];
  if (b0 < 0x80u) {
    cp = b0;
    return 1;
  }
  int need;
  uint32_t c, lo = 0x80u, hi = 0xBFu;
  if (b0 >= 0xC2u && b0 <= 0xDFu) {
    need = 1;
    c = b0 & 0x1Fu;
  } else if (b0 >= 0xE0u && b0 <= 0xEFu) {
    need = 2;
    c = b0 & 0x0Fu;
    if (b0 == 0xE0u) lo = 0xA0u;
    if (b0 == 0xEDu) hi = 0x9Fu;
  } else if (b0 >= 0xF0u && b0 <= 0xF4u) {
    need = 3;
    c = b0 & 0x07u;
    if (b0 == 0xF0u) lo = 0x90u;
    if (b0 == 0xF4u) hi = 0x8Fu;
  } else {
    cp = 0xFFFDu;  // stray trail byte or invalid lead (C0, C1, F5..FF)
    return 1;
  }
  int k = 0;
  for (; k < need; ++k) {
    if (j + 1 + k >= len) break;
    const uint32_t b = s[j + 1 + k];
    if (b < lo || b > hi) break;
    lo = 0x80u;
    hi = 0xBFu;
    c = (c << 6) | (b & 0x3Fu);
  }
  cp = k == need ? c : 0xFFFDu;
  return 1 + k;
}

__device__ __forceinline__ bool starts_unit(const uint8_t* __restrict__ s, uint64_t len,
                                            uint64_t i) {
  if (!is_trail(s[i])) return true;
  for (uint64_t d = 1; d <= 3 && d <= i; ++d) {
    const uint64_t j = i - d;
    if (!is_trail(s[j])) {
      uint32_t cp;
      return static_cast<uint64_t>(unit_at(s, len, j, cp)) <= d;
    }
  }
  return true;
}

constexpr int kWarps = 8;

// pass 1: units per document (one warp per document)
__global__ void __launch_bounds__(kWarps * 32)
    k_utf8_count(const uint8_t* __restrict__ text, const uint64_t* __restrict__ offsets,
                 uint64_t n, uint32_t* __restrict__ units) {
  const uint64_t d = static_cast<uint64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (d >= n) return;
  const uint8_t* s = text + offsets[d];
  const uint64_t len = offsets[d + 1] - offsets[d];
  uint32_t count = 0;
  for (uint64_t i = lane; i < len; i += 32) count += starts_unit(s, len, i);
#pragma unroll
  for (int o = 16; o; o >>= 1) count += __shfl_xor_sync(0xFFFFFFFFu, count, o);
  if (lane == 0) units[d] = count;
}

// pass 2: the units themselves, at unit_off[d] (exclusive scan of pass 1)
__global__ void __launch_bounds__(kWarps * 32)
    k_utf8_decode(const uint8_t* __restrict__ text, const uint64_t* __restrict__ offsets,
                  uint64_t n, const uint64_t* __restrict__ unit_off, uint32_t* __restrict__ out) {
  const uint64_t d = static_cast<uint64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (d >= n) return;
  const uint8_t* s = text + offsets[d];
  const uint64_t len = offsets[d + 1] - offsets[d];
  uint32_t* o = out + unit_off[d];
  const unsigned below = (1u << lane) - 1u;
  uint64_t written = 0;
  for (uint64_t b = 0; b < len; b += 32) {
    const uint64_t i = b + lane;
    bool st = false;
    uint32_t cp = 0;
    if (i < len) {
      st = starts_unit(s, len, i);
      if (st) unit_at(s, len, i, cp);
    }
    const unsigned m = __ballot_sync(0xFFFFFFFFu, st);
    if (st) o[written + __popc(m & below)] = cp;
    written += __popc(m);
  }
}

}  // namespace

void decode_codepoints_device(const uint8_t* d_text, const uint64_t* d_offsets, uint64_t n,
                              DevBuf& units_buf, DevBuf& unit_off_buf, DevBuf& count_buf,
                              DevBuf& scan_tmp, cudaStream_t s, const uint32_t** units_out,
                              const uint64_t** unit_off_out) {
  uint32_t* cnt = count_buf.as<uint32_t>(n);
  uint64_t* uoff = unit_off_buf.as<uint64_t>(n + 1);
  const unsigned blocks = static_cast<unsigned>((n + kWarps - 1) / kWarps);
  k_utf8_count<<<blocks, kWarps * 32, 0, s>>>(d_text, d_offsets, n, cnt);
  ND_CHECK_LAUNCH();
  scan_u32_to_u64(cnt, uoff, n, scan_tmp, s);
  uint64_t total = 0;
  ND_CUDA(cudaMemcpyAsync(&total, uoff + n, sizeof total, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  uint32_t* units = units_buf.as<uint32_t>(total + 1);
  k_utf8_decode<<<blocks, kWarps * 32, 0, s>>>(d_text, d_offsets, n, uoff, units);
  ND_CHECK_LAUNCH();
  *units_out = units;
  *unit_off_out = uoff;
}

}  // namespace ndb
