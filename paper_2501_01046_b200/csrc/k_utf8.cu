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

// Word-parallel walk (round 2): a warp reads its document as aligned 4-byte
// words, 128 bytes per step (one LDG.32 per lane); every byte decides
// "starts a unit?" and its value from the 3 bytes on either side, which come
// from the neighbouring lanes' words (shuffles; lane 31 also reads the word
// after the step, lane 0 gets the previous step's last word).  Bytes outside
// the document read as 0 -- a non-trail byte, which ends a sequence exactly
// where unit_at's length checks would (and no position outside is decoded).
struct Ctx12 {
  uint32_t prev, cur, next;  // bytes at offsets -4..-1, 0..3, 4..7 of the lane's word
  __device__ __forceinline__ uint32_t at(int o) const {  // o in [-4, 7], unrolled
    return o < 0 ? (prev >> (8 * (o + 4))) & 0xFFu
         : o < 4 ? (cur >> (8 * o)) & 0xFFu
                 : (next >> (8 * (o - 4))) & 0xFFu;
  }
};

// byte K of the word as a lead: unit length (unit_at's; 0 for a trail byte)
// and value (the scalar, or U+FFFD when ill-formed)
template <int K>
__device__ __forceinline__ uint32_t lead_at(const Ctx12& c, uint32_t& cp) {
  const uint32_t b0 = c.at(K);
  cp = b0;
  if (b0 < 0x80u) return 1;
  if (is_trail(b0)) {
    cp = 0xFFFDu;  // only decoded when no lead covers it: a unit of its own
    return 0;
  }
  int need;
  uint32_t v, lo = 0x80u, hi = 0xBFu;
  if (b0 >= 0xC2u && b0 <= 0xDFu) {
    need = 1;
    v = b0 & 0x1Fu;
  } else if (b0 >= 0xE0u && b0 <= 0xEFu) {
    need = 2;
    v = b0 & 0x0Fu;
    if (b0 == 0xE0u) lo = 0xA0u;
    if (b0 == 0xEDu) hi = 0x9Fu;
  } else if (b0 >= 0xF0u && b0 <= 0xF4u) {
    need = 3;
    v = b0 & 0x07u;
    if (b0 == 0xF0u) lo = 0x90u;
    if (b0 == 0xF4u) hi = 0x8Fu;
  } else {
    cp = 0xFFFDu;  // invalid lead (C0, C1, F5..FF)
    return 1;
  }
  int k = 0;
  const uint32_t b1 = c.at(K + 1);
  if (b1 >= lo && b1 <= hi) {
    v = (v << 6) | (b1 & 0x3Fu);
    k = 1;
    if (need >= 2) {
      const uint32_t b2 = c.at(K + 2);
      if (is_trail(b2)) {
        v = (v << 6) | (b2 & 0x3Fu);
        k = 2;
        if (need == 3) {
          const uint32_t b3 = c.at(K + 3);
          if (is_trail(b3)) {
            v = (v << 6) | (b3 & 0x3Fu);
            k = 3;
          }
        }
      }
    }
  }
  cp = k == need ? v : 0xFFFDu;
  return 1 + k;
}

// the lane's word: bytes at document positions pos .. pos+3, 0 outside [0, len)
__device__ __forceinline__ uint32_t masked_word(const uint32_t* w, int64_t pos, int64_t len) {
  if (pos + 3 < 0 || pos >= len) return 0u;
  uint32_t v = __ldg(w);
  if (pos < 0) v &= 0xFFFFFFFFu << (8 * static_cast<int>(-pos));
  if (pos + 4 > len) v &= 0xFFFFFFFFu >> (8 * static_cast<int>(pos + 4 - len));
  return v;
}

// one step of the walk: the 4 bytes of this lane -> start mask + values.
// A byte starts a unit unless it is a trail byte covered by the nearest
// non-trail byte j within 3 before it (len(j) > distance): non-trail bytes
// end every sequence, so no other lead can cover it.  Unit lengths of the 3
// bytes before the word come from the lane below (lane 0: the previous step).
__device__ __forceinline__ uint32_t step_units(const uint32_t* aw, int64_t pos0, int64_t len,
                                               int lane, uint32_t& carry, uint32_t& lcarry,
                                               uint32_t (&cp)[4]) {
  const int64_t pos = pos0 + 4 * lane;
  const uint32_t w = masked_word(aw + lane, pos, len);
  Ctx12 c;
  c.cur = w;
  c.prev = __shfl_up_sync(0xFFFFFFFFu, w, 1);
  if (lane == 0) c.prev = carry;
  c.next = __shfl_down_sync(0xFFFFFFFFu, w, 1);
  if (lane == 31) c.next = masked_word(aw + 32, pos + 4, len);
  carry = __shfl_sync(0xFFFFFFFFu, w, 31);
  uint32_t valid = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) valid |= (pos + k >= 0 && pos + k < len) ? (1u << k) : 0u;
  uint32_t l4;  // unit lengths of the 4 bytes, 3 bits each
  if (((c.prev | c.cur | c.next) & 0x80808080u) == 0u) {  // ASCII context
#pragma unroll
    for (int k = 0; k < 4; ++k) cp[k] = (w >> (8 * k)) & 0xFFu;
    l4 = 01111u;
  } else {
    const uint32_t n0 = lead_at<0>(c, cp[0]), n1 = lead_at<1>(c, cp[1]);
    const uint32_t n2 = lead_at<2>(c, cp[2]), n3 = lead_at<3>(c, cp[3]);
    l4 = n0 | (n1 << 3) | (n2 << 6) | (n3 << 9);
  }
  uint32_t lp = __shfl_up_sync(0xFFFFFFFFu, l4, 1);
  if (lane == 0) lp = lcarry;
  lcarry = __shfl_sync(0xFFFFFFFFu, l4, 31);
  if (l4 == 01111u) return valid;  // every byte leads a unit
  // lens of positions -4..3 (a trail byte has length 0)
  const uint32_t l8 = lp | (l4 << 12);
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t lk = (l8 >> (3 * (k + 4))) & 7u;
    bool st = lk != 0;
    if (!st) {
      st = true;  // three trail bytes before it (or the document start): its own unit
#pragma unroll
      for (int d = 3; d >= 1; --d) {  // the nearest non-trail byte wins
        const uint32_t lj = (l8 >> (3 * (k + 4 - d))) & 7u;
        if (lj != 0) st = lj <= static_cast<uint32_t>(d);
      }
    }
    m |= st ? (1u << k) : 0u;
  }
  return m & valid;
}

// pass 1: units per document (one warp per document); CLS: also the
// document's class by its largest code point (0: < 256, 1: < 2^16, 2: above),
// cls_cnt[0] counting classes >= 1 and cls_cnt[1] class 2
template <bool CLS>
__global__ void __launch_bounds__(kWarps * 32)
    k_utf8_count(const uint8_t* __restrict__ text, const uint64_t* __restrict__ offsets,
                 uint64_t n, uint32_t* __restrict__ units, uint32_t* __restrict__ cls,
                 uint32_t* __restrict__ cls_cnt) {
  const uint64_t d = static_cast<uint64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (d >= n) return;
  const uint8_t* s = text + offsets[d];
  const int64_t len = static_cast<int64_t>(offsets[d + 1] - offsets[d]);
  const uint32_t* aw = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(s) & ~uintptr_t{3});
  int64_t pos0 = -static_cast<int64_t>(reinterpret_cast<uintptr_t>(s) & 3);
  uint32_t count = 0, carry = 0, lcarry = 01111u, mx = 0;
  uint32_t cp[4];
  for (; pos0 < len; pos0 += 128, aw += 32) {
    const uint32_t m = step_units(aw, pos0, len, lane, carry, lcarry, cp);
    count += __popc(m);
    if (CLS) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (m & (1u << k)) mx = max(mx, cp[k]);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) count += __shfl_xor_sync(0xFFFFFFFFu, count, o);
  if (CLS) mx = __reduce_max_sync(0xFFFFFFFFu, mx);
  if (lane == 0) {
    units[d] = count;
    if (CLS) {
      const uint32_t c = mx >= 0x10000u ? 2u : mx >= 256u ? 1u : 0u;
      cls[d] = c;
      if (c) atomicAdd(cls_cnt, 1u);
      if (c == 2) atomicAdd(cls_cnt + 1, 1u);
    }
  }
}

// pass 2: the units themselves, at unit_off[d] (exclusive scan of pass 1):
// as u32, or -- cls given -- as u16 (out16) for the documents of class
// < wide_from and u32 for the others
__global__ void __launch_bounds__(kWarps * 32)
    k_utf8_decode(const uint8_t* __restrict__ text, const uint64_t* __restrict__ offsets,
                  uint64_t n, const uint64_t* __restrict__ unit_off, uint32_t* __restrict__ out,
                  const uint32_t* __restrict__ cls, uint32_t wide_from,
                  uint16_t* __restrict__ out16) {
  const uint64_t d = static_cast<uint64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (d >= n) return;
  const uint8_t* s = text + offsets[d];
  const int64_t len = static_cast<int64_t>(offsets[d + 1] - offsets[d]);
  const uint32_t* aw = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(s) & ~uintptr_t{3});
  int64_t pos0 = -static_cast<int64_t>(reinterpret_cast<uintptr_t>(s) & 3);
  uint32_t* o = out + unit_off[d];
  uint16_t* o16 = out16 ? out16 + unit_off[d] : nullptr;
  const bool narrow = cls && cls[d] < wide_from;
  const unsigned below = (1u << lane) - 1u;
  uint64_t written = 0;
  uint32_t carry = 0, lcarry = 01111u;
  for (; pos0 < len; pos0 += 128, aw += 32) {
    uint32_t cp[4];
    const uint32_t m = step_units(aw, pos0, len, lane, carry, lcarry, cp);
    const uint32_t cnt = __popc(m);  // 0..4: the lane's rank from three bit ballots
    const unsigned b0 = __ballot_sync(0xFFFFFFFFu, cnt & 1u);
    const unsigned b1 = __ballot_sync(0xFFFFFFFFu, cnt & 2u);
    const unsigned b2 = __ballot_sync(0xFFFFFFFFu, cnt & 4u);
    uint32_t at = __popc(b0 & below) + 2 * __popc(b1 & below) + 4 * __popc(b2 & below);
    if (narrow) {
      uint16_t* dst = o16 + written;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (m & (1u << k)) dst[at++] = static_cast<uint16_t>(cp[k]);
    } else {
      uint32_t* dst = o + written;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (m & (1u << k)) dst[at++] = cp[k];
    }
    written += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
  }
}

}  // namespace

void decode_codepoints_device(const uint8_t* d_text, const uint64_t* d_offsets, uint64_t n,
                              DevBuf& units_buf, DevBuf& unit_off_buf, DevBuf& count_buf,
                              DevBuf& scan_tmp, cudaStream_t s, const uint32_t** units_out,
                              const uint64_t** unit_off_out, CodepointClasses* classes) {
  uint32_t* cnt = count_buf.as<uint32_t>(n);
  uint64_t* uoff = unit_off_buf.as<uint64_t>(n + 1);
  const unsigned blocks = static_cast<unsigned>((n + kWarps - 1) / kWarps);
  uint32_t* cls = nullptr;
  uint32_t* cls_cnt = nullptr;
  if (classes) {
    cls = classes->cls_buf->as<uint32_t>(n);
    cls_cnt = classes->cnt_buf->as<uint32_t>(4);
    ND_CUDA(cudaMemsetAsync(cls_cnt, 0, 4 * sizeof(uint32_t), s));
    k_utf8_count<true><<<blocks, kWarps * 32, 0, s>>>(d_text, d_offsets, n, cnt, cls, cls_cnt);
  } else {
    k_utf8_count<false><<<blocks, kWarps * 32, 0, s>>>(d_text, d_offsets, n, cnt, nullptr, nullptr);
  }
  ND_CHECK_LAUNCH();
  scan_u32_to_u64(cnt, uoff, n, scan_tmp, s);
  uint64_t h[2] = {0, 0};
  uint32_t hc[2] = {0, 0};
  ND_CUDA(cudaMemcpyAsync(&h[0], uoff + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  if (classes) ND_CUDA(cudaMemcpyAsync(hc, cls_cnt, sizeof hc, cudaMemcpyDeviceToHost, s));
  ND_CUDA(cudaStreamSynchronize(s));
  const uint64_t total = h[0];
  uint32_t* units = units_buf.as<uint32_t>(total + 1);
  uint16_t* u16 = nullptr;
  if (classes) {
    classes->total = total;
    classes->n_wide = hc[0];
    classes->n_astral = hc[1];
    classes->cls = cls;
    u16 = classes->u16_buf->as<uint16_t>(total + 16);
    classes->u16 = u16;
  }
  k_utf8_decode<<<blocks, kWarps * 32, 0, s>>>(d_text, d_offsets, n, uoff, units, cls,
                                                classes ? classes->wide_from : 0u, u16);
  ND_CHECK_LAUNCH();
  *units_out = units;
  *unit_off_out = uoff;
}

}  // namespace ndb
