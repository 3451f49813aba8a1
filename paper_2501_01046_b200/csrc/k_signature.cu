// K1: MinHash signatures + LSH band keys, one warp per work item.
//
// Replaces signature_of_document (minhash.cpp:133-162) and band_bucket_ids
// (lsh.cpp:42-60) as called by the hash stage (pipeline.cpp:214-218).
//
// Arithmetic.  For hash function (p, q) the window value is
//   h_w = sum_{i<L} c_{w+i} q^i mod p          (hash_window_direct, minhash.cpp:111-119)
// Any exact evaluation gives the same bits and the signature is the min over
// windows, so each work item is walked BACKWARD with the Horner-shift
// recurrence (instead of the reference's forward Eq.5 update, minhash.cpp:121-131)
//   u   = q*c_{w+1} + c_out*QLn + c_in,   QLn = (p - q^L mod p) mod p
//   c_w = u mod p                          (u < 2^39 + 2^31)
// The window state starts at 0 one position past the item's last character
// and is warmed up over L-1 partial windows (c_out = 0 beyond the item), so no
// separate direct evaluation of the first window is needed.
//
// Reduction, "fq" variant (default).  ncu on the all-integer variant showed the
// FMA-heavy pipe (the only one that executes IMAD / IMAD.WIDE / IMAD.HI) at 90%
// while ALU sat at 42% and FMA-lite idle.  The quotient k = floor(u/p) is
// therefore ESTIMATED in FP32 on the FMA-lite pipe and only three plain 32-bit
// IMADs remain on FMA-heavy (10 instructions per hash-window, 3/3/4 over
// heavy/lite/alu):
//   SB = c | 0x4B000000                 LOP3        float(SB) = 2^23 + c exactly
//   t1 = fma(c_out, QLn/p, -2^23 q/p + 2^-5)   FFMA
//   R  = fma(float(SB), q/p, t1)        FFMA        R in [u/p + 0.015, u/p + 0.048]
//   Kb = bits(R + (2^23 - 0.5), round-down)   FADD.RM   Kb = 0x4B000000 + floor(R - 1/2)
//   r  = q*c + (c_out*QLn + c_in) - Kb*p + 0x4B000000*p  (3 IMAD + IADD, mod 2^32)
//   c' = min(r, r - p) (unsigned)       VIADDMNMX   r in [0, 2p) -> canonical
//   sig = min(sig, c')                  VIMNMX
// floor(R - 1/2) is Q or Q-1 (Q = floor(u/p)) because the FP32 error of R is
// < 0.017 (derivation in DESIGN.md), so r = u - k*p lies in [0, 2p).
// The "int" variant (ND_K1_KERNEL=int) keeps the all-integer Barrett
// reduction (IMAD.WIDE + SHF + IMAD.HI) for comparison.
//
// Codepoint units ("wide" variant).  Scalar values reach 0x10FFFF, so
// c_out*QLn needs 44 bits and the FP32 quotient estimate is no longer exact
// enough; the units (decoded by k_utf8.cu) are u32 and each step is
//   u = q*c + c_out*QLn + c_in          (2 IMAD.WIDE, u < p*(q + 2^21) < 2^44)
//   k = umulhi(u >> 13, floor(2^45/p))  (k in {Q-1, Q}: the error is below
//                                        u/2^45 + 2^13/p < 0.55)
//   c' = min(r, r - p), r = u - k*p     (r in [0, 2p))
//
// Layout.  A warp owns one work item.  Its 32 lanes form Z groups of 32/Z
// lanes; lane l of a group owns functions [l*F, l*F+F) of the padded family
// (Hp = 32*F/Z; pad functions are copies of function 0 and never stored), and
// group z walks the z-th of Z equal slices of the item's windows (the min
// over a partition of windows is the min of the partial minima, so the
// slices meet through a warp shuffle).  Characters are staged per group in
// shared memory as (byte, float) pairs and read back as broadcast LDS.
// Documents longer than kSeg windows are split into several work items that
// meet through atomicMin; their band keys come from a follow-up pass.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "nd_internal.cuh"

namespace ndb {
namespace {

#ifndef ND_K1_WARPS
#define ND_K1_WARPS 4
#endif
#ifndef ND_K1_MINBLOCKS
#define ND_K1_MINBLOCKS 0  // 0: no min-blocks hint (ptxas chose 96 registers)
#endif
// resident blocks per SM the register allocation must allow: the fq kernel
// with 8 functions per lane fits 96 registers (5 blocks of 4 warps); the
// persistent item loop would otherwise let ptxas take 128 (4 blocks)
#if ND_K1_MINBLOCKS > 0
#define ND_K1_BOUNDS __launch_bounds__(ND_K1_WARPS * 32, ND_K1_MINBLOCKS)
#else
#define ND_K1_BOUNDS __launch_bounds__(ND_K1_WARPS * 32, k1_min_blocks(A, F, SL))
#endif
#ifndef ND_K1_UNROLL4
#define ND_K1_UNROLL4 1
#endif
#ifndef ND_K1_ASM_ORDER
#define ND_K1_ASM_ORDER 0
#endif
#ifndef ND_K1_I2F
#define ND_K1_I2F 1  // float operand = I2FP(256c) instead of the 2^23-biased word
#endif
constexpr int kWarps = ND_K1_WARPS;  // warps per block
constexpr int kLMax = 64;           // max shingle length
// positions staged per chunk and group: (char, float) pairs, 8 B each
__host__ __device__ constexpr int chunk_for(int Z) { return Z >= 4 ? 128 : 256; }
constexpr uint32_t kSeg = 8192;     // max windows per work item
constexpr uint32_t kMagicBits = 0x4B000000u;  // bits of 2^23f

struct FamPtrs {
  const uint32_t* q;
  const uint32_t* qln;
  const uint32_t* m;
  const uint32_t* negp;
  const uint32_t* c3;     // 0x4B000000 * p mod 2^32
  const float* qp;        // fl(q / p)
  const float* qlnp;      // fl(QLn / p)
  const float* c1e;       // -2^23 * qp + 2^-5 (exact)
  const uint32_t* m45;    // floor(2^45 / p)
  const uint32_t* p;      // modulus (exact variant)
  const unsigned long long* rf;  // floor(2^64 / p) (exact variant)
};

// ---------------------------------------------------------------------------
// planning: per-document segment counts, short-document detection
__global__ void k_plan(const uint64_t* __restrict__ offsets, uint64_t n, uint32_t L,
                       uint32_t* __restrict__ seg_count, uint32_t* __restrict__ flags,
                       uint32_t seg_len) {
  uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (d >= n) return;
  uint64_t len = offsets[d + 1] - offsets[d];
  uint32_t nseg = 1;
  if (len < L) {
    atomicOr(&flags[0], 1u);  // ShortDocumentError
  } else {
    uint64_t nwin = len - L + 1;
    uint64_t s = (nwin + seg_len - 1) / seg_len;
    nseg = static_cast<uint32_t>(s);
    if (s > 1) atomicAdd(&flags[1], 1u);  // multi-item document count
  }
  seg_count[d] = nseg;
}

__global__ void k_item_scatter(const uint64_t* __restrict__ item_off, uint64_t n,
                               uint32_t* __restrict__ item_doc, uint32_t* __restrict__ multi_docs,
                               uint32_t* __restrict__ nmulti) {
  uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (d >= n) return;
  uint64_t b = item_off[d], e = item_off[d + 1];
  for (uint64_t i = b; i < e; ++i) item_doc[i] = static_cast<uint32_t>(d);
  if (e - b > 1) multi_docs[atomicAdd(nmulti, 1u)] = static_cast<uint32_t>(d);
}

__global__ void k_fill_multi(const uint32_t* __restrict__ multi_docs, uint32_t nmulti, uint32_t H,
                             uint32_t* __restrict__ sig) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       i < static_cast<uint64_t>(nmulti) * H; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t d = multi_docs[i / H];
    sig[d * H + i % H] = 0xFFFFFFFFu;
  }
}

// any byte >= 0x80 in text[lo, hi)?  (a codepoint batch of pure ASCII has
// units == bytes: it runs the byte path on the text as it is)
__global__ void k_any_high(const uint8_t* __restrict__ text, uint64_t lo, uint64_t hi,
                           unsigned int* __restrict__ flag) {
  const uint64_t a = (lo + 15) & ~uint64_t{15}, b = hi & ~uint64_t{15};
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  if (a < b) {
    const uint4* v = reinterpret_cast<const uint4*>(text + a);
    for (uint64_t i = tid; i < (b - a) / 16; i += stride) {
      const uint4 w = __ldg(v + i);
      acc |= w.x | w.y | w.z | w.w;
    }
    for (uint64_t i = lo + tid; i < a; i += stride) acc |= text[i];
    for (uint64_t i = b + tid; i < hi; i += stride) acc |= text[i];
  } else {
    for (uint64_t i = lo + tid; i < hi; i += stride) acc |= text[i];
  }
  if (__any_sync(0xFFFFFFFFu, (acc & 0x80808080u) != 0) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// class-0 codepoint documents (all units < 256) run the byte kernels over
// their units narrowed to bytes
__global__ void k_u16_to_u8(const uint16_t* __restrict__ units, uint64_t m,
                            uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint8_t>(units[i]);
}

// seg_count of the documents outside [lo, hi] of their class -> 0 (no items)
__global__ void k_keep_class(const uint32_t* __restrict__ cls, uint64_t n, uint32_t lo,
                             uint32_t hi, uint32_t* __restrict__ seg_count) {
  const uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (d < n && (cls[d] < lo || cls[d] > hi)) seg_count[d] = 0;
}

// K1j work order: items by descending window count (stable), so the 32
// items a warp takes have nearly equal lengths
__global__ void k_item_len_keys(const uint64_t* __restrict__ offsets,
                                const uint32_t* __restrict__ item_doc,
                                const uint64_t* __restrict__ item_off, uint64_t n_items, uint32_t L,
                                uint32_t seg_len, uint32_t* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n_items) return;
  uint64_t doc = i, ws = 0;
  if (item_doc) {
    doc = item_doc[i];
    ws = (i - item_off[doc]) * seg_len;
  }
  const uint64_t nwin = offsets[doc + 1] - offsets[doc] - L + 1;
  const uint64_t w = min(nwin - ws, static_cast<uint64_t>(seg_len));
  keys[i] = 16383u - static_cast<uint32_t>(w);  // kSeg < 2^14
  vals[i] = static_cast<uint32_t>(i);
}

// one thread holds its stream until *flag >= epoch (bounded: after ~4 s it
// gives up, and the next launch simply runs alongside)
__global__ void k_gate_wait(const unsigned int* __restrict__ flag, unsigned int epoch) {
  const long long t0 = clock64();
  while (*reinterpret_cast<const volatile unsigned int*>(flag) < epoch) {
    if (clock64() - t0 > 8000000000ll) break;
    __nanosleep(1000);
  }
}

__global__ void k_iota_docs(uint32_t* __restrict__ v, uint64_t n) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = static_cast<uint32_t>(i);
}

// band keys from finished signature rows (multi-item documents)
__global__ void k_bands_from_rows(const uint32_t* __restrict__ docs, uint32_t ndocs,
                                  const uint32_t* __restrict__ sig, uint32_t H, uint32_t bands,
                                  uint32_t rows, uint32_t K, uint32_t* __restrict__ band) {
  uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<uint64_t>(ndocs) * bands) return;
  uint64_t d = docs[i / bands];
  uint32_t j = static_cast<uint32_t>(i % bands);
  const uint32_t* row = sig + d * H + static_cast<uint64_t>(j) * rows;
  uint64_t sum = 0;  // rows * 2^23 never wraps 64 bits (lsh.cpp:54)
  for (uint32_t r = 0; r < rows; ++r) sum += row[r];
  band[d * bands + j] = K ? static_cast<uint32_t>(sum % K) : static_cast<uint32_t>(sum);
}

// ---------------------------------------------------------------------------
enum class Arith { kInt, kFq, kWide, kExact };
// register caps (blocks of 4 warps per SM) that reproduce the allocation of
// the one-item-per-warp kernel: fq F=4/8/16 -> 80/96/168 registers, int and
// wide F<=4/8/16 -> 64/80/128
__host__ __device__ constexpr int k1_min_blocks(Arith a, int f, int sl = 1) {
  return sl == 2 ? (f <= 4 ? 6 : 4)
                 : a == Arith::kFq ? (f <= 4 ? 6 : f <= 8 ? 5 : 3) : (f <= 4 ? 8 : f <= 8 ? 6 : 4);
}

template <Arith A, int F>
struct Consts;

template <int F>
struct Consts<Arith::kInt, F> {
  uint32_t q[F], qln[F], m[F], negp[F];
  __device__ void load(const FamPtrs& fp, int base) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      q[f] = fp.q[base + f];
      qln[f] = fp.qln[base + f];
      m[f] = fp.m[base + f];
      negp[f] = fp.negp[base + f];
    }
  }
  // one rolling step for all F functions: all-integer Barrett reduction
  template <bool kMin>
  __device__ __forceinline__ void step(uint32_t cin, uint32_t cout, float /*cout_f*/,
                                       uint32_t (&s)[F], uint32_t (&mn)[F]) const {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      uint32_t a = cout * qln[f] + cin;
      uint64_t u = static_cast<uint64_t>(q[f]) * s[f] + a;
      uint32_t lo = static_cast<uint32_t>(u);
      uint32_t t = __funnelshift_r(lo, static_cast<uint32_t>(u >> 32), 8);
      uint32_t k = __umulhi(t, m[f]);  // M = floor(2^40 / p): k in {Q-1, Q}
      uint32_t r = lo + k * negp[f];
      uint32_t c = min(r, r + negp[f]);
      s[f] = c;
      if (kMin) mn[f] = min(mn[f], c);
    }
  }
};

template <int F>
struct Consts<Arith::kWide, F> {
  uint32_t q[F], qln[F], m[F], negp[F];
  __device__ void load(const FamPtrs& fp, int base) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      q[f] = fp.q[base + f];
      qln[f] = fp.qln[base + f];
      m[f] = fp.m45[base + f];
      negp[f] = fp.negp[base + f];
    }
  }
  // one rolling step for all F functions with units up to 0x10FFFF
  template <bool kMin>
  __device__ __forceinline__ void step(uint32_t cin, uint32_t cout, float /*cout_f*/,
                                       uint32_t (&s)[F], uint32_t (&mn)[F]) const {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      uint64_t u = static_cast<uint64_t>(cout) * qln[f] + cin;
      u += static_cast<uint64_t>(q[f]) * s[f];
      const uint32_t lo = static_cast<uint32_t>(u);
      const uint32_t t = __funnelshift_r(lo, static_cast<uint32_t>(u >> 32), 13);
      const uint32_t k = __umulhi(t, m[f]);
      const uint32_t r = lo + k * negp[f];
      const uint32_t c = min(r, r + negp[f]);
      s[f] = c;
      if (kMin) mn[f] = min(mn[f], c);
    }
  }
};

// Families outside the fast arithmetics' proven domain (hand-built
// HashFunctionParams, see nd_family_upload): the reference's own Barrett
// reduction with reduce_factor = floor(2^64/p) (minhash.cpp:61-67) over a
// 64-bit u = q*c + c_out*QLn + c_in < 2^63 (p < 2^31).  k = umulhi64(u, rf)
// is Q or Q-1 (u/2^64 < 1), so r = u - k*p lies in [0, 2p) < 2^32 and one
// unsigned min canonicalises it.  Not a throughput path.
template <int F>
struct Consts<Arith::kExact, F> {
  uint32_t q[F], qln[F], p[F];
  unsigned long long rf[F];
  __device__ void load(const FamPtrs& fp, int base) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      q[f] = fp.q[base + f];
      qln[f] = fp.qln[base + f];
      p[f] = fp.p[base + f];
      rf[f] = fp.rf[base + f];
    }
  }
  template <bool kMin>
  __device__ __forceinline__ void step(uint32_t cin, uint32_t cout, float /*cout_f*/,
                                       uint32_t (&s)[F], uint32_t (&mn)[F]) const {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const unsigned long long u = static_cast<unsigned long long>(cout) * qln[f] + cin +
                                   static_cast<unsigned long long>(q[f]) * s[f];
      const unsigned long long k = __umul64hi(u, rf[f]);
      const uint32_t r = static_cast<uint32_t>(u) - static_cast<uint32_t>(k) * p[f];
      const uint32_t c = min(r, r - p[f]);
      s[f] = c;
      if (kMin) mn[f] = min(mn[f], c);
    }
  }
};

#if ND_K1_I2F
// fq arithmetic with the float operand converted exactly (I2FP.F32.U32 of
// C = 256c < 2^31, <= 23 significant bits) instead of the 2^23-biased word:
// no -2^23 q/p constant, 5 constants per function.
//   R  = fma(float(C), fl(q/p)/256, fma(c_out, fl(QLn/p), 2^-5))
//      in [u/p + 2^-5 - 0.009, u/p + 2^-5 + 0.009]  => floor(R - 1/2) in {Q-1, Q}
//   256r = C*q + Kb*(-256p) + c_out*256QLn + 256c_in   (Kb = 0x4B000000 + k)
template <int F>
struct Consts<Arith::kFq, F> {
  uint32_t q[F], qln256[F], negp256[F];
  float qp256[F], qlnp[F];
  __device__ void load(const FamPtrs& fp, int base) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      q[f] = fp.q[base + f];
      qln256[f] = fp.qln[base + f] << 8;
      negp256[f] = fp.negp[base + f] << 8;
      qp256[f] = fp.qp[base + f] * 0.00390625f;
      qlnp[f] = fp.qlnp[base + f];
    }
  }
  __device__ __forceinline__ uint32_t roll(int f, uint32_t C, uint32_t cin256, uint32_t cout,
                                           float cout_f) const {
    const float t1 = __fmaf_rn(cout_f, qlnp[f], 0.03125f);
    const float R = __fmaf_rn(__uint2float_rn(C), qp256[f], t1);
    const uint32_t kb = __float_as_uint(__fadd_rd(R, 8388607.5f));
    uint32_t x = cout * qln256[f] + cin256;
    x = C * q[f] + x;
    x = kb * negp256[f] + x;
    return min(x, x + negp256[f]);
  }
};
#else
template <int F>
struct Consts<Arith::kFq, F> {
  // integer constants pre-scaled by 256 (see step): the state is C = 256*c
  uint32_t q256[F], qln256[F], negp256[F];
  float qp[F], qlnp[F], c1e[F];
  __device__ void load(const FamPtrs& fp, int base) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      q256[f] = fp.q[base + f] << 8;
      qln256[f] = fp.qln[base + f] << 8;
      negp256[f] = fp.negp[base + f] << 8;
      qp[f] = fp.qp[base + f];
      qlnp[f] = fp.qlnp[base + f];
      c1e[f] = fp.c1e[base + f];
    }
  }
  // One rolling step for function f; returns the new scaled state 256*c.
  // With everything scaled by 256 the bias of the float bits (0x4B000000 =
  // 0x4B * 2^24) vanishes mod 2^32, so the biased words feed the IMADs
  // directly and r*256 < 2^32 comes out exact:
  //   sb   = (C >> 8) | 0x4B000000      LEA.HI       float(sb) = 2^23 + c
  //   R    = fma(sb, q/p, fma(c_out, QLn/p, c1e))   2 FFMA
  //   Kb   = bits(R + 2^23 - 1/2, rd)   FADD.RM      = 0x4B000000 + k
  //   256r = sb*256q + Kb*(-256p) + c_out*256QLn + 256c_in   3 IMAD
  //   C'   = min(256r, 256r - 256p)     VIADDMNMX    canonical, scaled
  __device__ __forceinline__ uint32_t roll(int f, uint32_t C, uint32_t cin256, uint32_t cout,
                                           float cout_f) const {
    const uint32_t sb = (C >> 8) | kMagicBits;
    const float t1 = __fmaf_rn(cout_f, qlnp[f], c1e[f]);
    const float R = __fmaf_rn(__uint_as_float(sb), qp[f], t1);
    const uint32_t kb = __float_as_uint(__fadd_rd(R, 8388607.5f));
    // the integer side only waits for kb in its last IMAD (shorter chain)
    uint32_t x = cout * qln256[f] + cin256;
    x = sb * q256[f] + x;
#if ND_K1_ASM_ORDER
    asm volatile("" : "+r"(x));  // keep the association: kb is consumed last
#endif
    x = kb * negp256[f] + x;
    return min(x, x + negp256[f]);
  }
};
#endif

// One work item (a document, or an 8192-window segment of a long one) for one
// warp; `item` is warp-uniform.
template <Arith A, int F, int Z, class T>
__device__ __forceinline__ void k1_item(
    uint64_t item, const T* __restrict__ text, const uint64_t* __restrict__ offsets,
    const uint32_t* __restrict__ item_doc, const uint64_t* __restrict__ item_off,
    const FamPtrs& fam, uint32_t L, uint32_t H, uint32_t bands, uint32_t rows, uint32_t K,
    uint32_t* __restrict__ sig, uint32_t* __restrict__ band, uint2 (*sbuf)[kLMax + chunk_for(Z)],
    uint32_t (*sbuf256)[kLMax + chunk_for(Z)], uint32_t* srow) {
  constexpr int G = 32 / Z;  // lanes per group
  constexpr int kChunk = chunk_for(Z);
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned gmask = Z == 1 ? 0xFFFFFFFFu : (((1u << G) - 1u) << (grp * G));

  uint64_t doc = item;
  uint64_t ws = 0;
  bool multi = false;
  if (item_doc) {
    doc = item_doc[item];
    uint64_t seg = item - item_off[doc];
    multi = item_off[doc + 1] - item_off[doc] > 1;
    ws = seg * kSeg;
  }
  const uint64_t off = offsets[doc];
  const uint64_t len = offsets[doc + 1] - off;
  const uint64_t nwin = len - L + 1;
  const uint64_t item_end = min(ws + kSeg, nwin);
  // this group's slice of windows [gs, ge)
  const uint64_t span = item_end - ws;
  const uint64_t gs = ws + span * grp / Z;
  const uint64_t ge = ws + span * (grp + 1) / Z;
  const uint64_t e = ge + L - 1;  // one past the last character this slice reads
  const T* base = text + off;

  Consts<A, F> k;
  k.load(fam, gl * F);
  uint32_t s[F], mn[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    s[f] = 0;
    mn[f] = 0xFFFFFFFFu;
  }

  uint2* buf = sbuf[grp];
  uint32_t* buf256 = sbuf256[grp];
  uint64_t p_hi = ge > gs ? e : gs;  // positions [p_lo, p_hi) per chunk, descending
  bool first = true;
  while (p_hi > gs) {
    const uint64_t p_lo = (p_hi - gs > kChunk) ? p_hi - kChunk : gs;
    const int cnt = static_cast<int>(p_hi - p_lo);
    // stage (char, float(char)) and 256*char for [p_lo, p_hi + L), zero beyond e
    for (int j = gl; j < cnt + static_cast<int>(L); j += G) {
      uint64_t pos = p_lo + j;
      uint32_t c = pos < e ? base[pos] : 0u;
      buf[j] = make_uint2(c, __float_as_uint(static_cast<float>(c)));
      buf256[j] = c << 8;
    }
    __syncwarp(gmask);
    int j = cnt - 1;
    if constexpr (A == Arith::kFq) {
      if (first) {
        for (int w = 0; w < static_cast<int>(L) - 1; ++w, --j) {
          const uint2 o = buf[j + L];
          const uint32_t ci = buf256[j];
#pragma unroll
          for (int f = 0; f < F; ++f) s[f] = k.roll(f, s[f], ci, o.x, __uint_as_float(o.y));
        }
        first = false;
      }
#if ND_K1_UNROLL4
      for (; j >= 3; j -= 4) {
        const uint2 o0 = buf[j + L], o1 = buf[j - 1 + L], o2 = buf[j - 2 + L], o3 = buf[j - 3 + L];
        const uint32_t c0 = buf256[j], c1 = buf256[j - 1], c2 = buf256[j - 2], c3 = buf256[j - 3];
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const uint32_t a0 = k.roll(f, s[f], c0, o0.x, __uint_as_float(o0.y));
          const uint32_t a1 = k.roll(f, a0, c1, o1.x, __uint_as_float(o1.y));
          const uint32_t a2 = k.roll(f, a1, c2, o2.x, __uint_as_float(o2.y));
          const uint32_t a3 = k.roll(f, a2, c3, o3.x, __uint_as_float(o3.y));
          s[f] = a3;
          mn[f] = __vimin3_u32(mn[f], a0, a1);
          mn[f] = __vimin3_u32(mn[f], a2, a3);
        }
      }
#endif
      // two windows per iteration: one 3-way min (VIMNMX3) folds both
      for (; j >= 1; j -= 2) {
        const uint2 o0 = buf[j + L], o1 = buf[j - 1 + L];
        const uint32_t c0 = buf256[j], c1 = buf256[j - 1];
#pragma unroll
        for (int f = 0; f < F; ++f) {
          const uint32_t a0 = k.roll(f, s[f], c0, o0.x, __uint_as_float(o0.y));
          const uint32_t a1 = k.roll(f, a0, c1, o1.x, __uint_as_float(o1.y));
          s[f] = a1;
          mn[f] = __vimin3_u32(mn[f], a0, a1);
        }
      }
      if (j == 0) {
        const uint2 o = buf[L];
        const uint32_t ci = buf256[0];
#pragma unroll
        for (int f = 0; f < F; ++f) {
          s[f] = k.roll(f, s[f], ci, o.x, __uint_as_float(o.y));
          mn[f] = min(mn[f], s[f]);
        }
      }
    } else {
      if (first) {
        // L-1 warm-up positions: partial windows, not part of the minimum
        for (int w = 0; w < static_cast<int>(L) - 1; ++w, --j) {
          const uint2 o = buf[j + L];
          k.template step<false>(buf[j].x, o.x, __uint_as_float(o.y), s, mn);
        }
        first = false;
      }
#pragma unroll 2
      for (; j >= 0; --j) {
        const uint2 o = buf[j + L];
        k.template step<true>(buf[j].x, o.x, __uint_as_float(o.y), s, mn);
      }
    }
    __syncwarp(gmask);
    p_hi = p_lo;
  }

  if (Z > 1) {  // the slices' partial minima meet
    __syncwarp();
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int o = G; o < 32; o <<= 1) mn[f] = min(mn[f], __shfl_xor_sync(0xFFFFFFFFu, mn[f], o));
    if (grp != 0) return;
  }

  if constexpr (A == Arith::kFq) {
#pragma unroll
    for (int f = 0; f < F; ++f) mn[f] >>= 8;  // scaled state -> canonical value
  }
  uint32_t* out = sig + doc * H;
  const int fbase = gl * F;
  if (multi) {
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (fbase + f < static_cast<int>(H)) atomicMin(out + fbase + f, mn[f]);
    return;
  }
  if ((H % 4) == 0 && (F % 4) == 0 && fbase + F <= static_cast<int>(H)) {
#pragma unroll
    for (int f = 0; f < F; f += 4)
      *reinterpret_cast<uint4*>(out + fbase + f) = make_uint4(mn[f], mn[f + 1], mn[f + 2], mn[f + 3]);
  } else {
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (fbase + f < static_cast<int>(H)) out[fbase + f] = mn[f];
  }
  if (band == nullptr) return;
  uint32_t* row = srow;
#pragma unroll
  for (int f = 0; f < F; ++f) row[fbase + f] = mn[f];
  __syncwarp(gmask);
  for (uint32_t jb = gl; jb < bands; jb += G) {
    uint64_t sum = 0;
    for (uint32_t r = 0; r < rows; ++r) sum += row[jb * rows + r];
    band[doc * bands + jb] = K ? static_cast<uint32_t>(sum % K) : static_cast<uint32_t>(sum);
  }
}

// Dual-slice variant (fq arithmetic, byte units, all 32 lanes on one slice
// set): lane l owns functions [l*F, l*F+F) and walks TWO slices of the
// item's windows, A = the first ceil(span/2) windows and B = the last
// ceil(span/2) (they overlap by at most one window, which the min absorbs),
// stepping both in lockstep.  The two rolls of a function read the same
// constant registers back to back (operand reuse) and are independent (ILP),
// so a lane needs F*6 constant registers for 2F chains instead of 2F*6.
template <int F, int Z>
__device__ __forceinline__ void k1_item_dual(
    uint64_t item, const uint8_t* __restrict__ text, const uint64_t* __restrict__ offsets,
    const uint32_t* __restrict__ item_doc, const uint64_t* __restrict__ item_off,
    const FamPtrs& fam, uint32_t L, uint32_t H, uint32_t bands, uint32_t rows, uint32_t K,
    uint32_t* __restrict__ sig, uint32_t* __restrict__ band, uint2 (*sbuf)[kLMax + 128],
    uint32_t (*sbuf256)[kLMax + 128], uint32_t* srow) {
  // Z groups of G lanes: group z takes the z-th of Z equal parts of the item's
  // windows and walks it as two slices (A, B); lane gl owns functions gl*F..
  constexpr int kChunk = 128;
  constexpr int G = 32 / Z;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int gl = lane % G;
  const unsigned gmask = Z == 1 ? 0xFFFFFFFFu : (((1u << G) - 1u) << (grp * G));
  uint64_t doc = item;
  uint64_t ws = 0;
  bool multi = false;
  if (item_doc) {
    doc = item_doc[item];
    const uint64_t seg = item - item_off[doc];
    multi = item_off[doc + 1] - item_off[doc] > 1;
    ws = seg * kSeg;
  }
  const uint64_t off = offsets[doc];
  const uint64_t len = offsets[doc + 1] - off;
  const uint64_t nwin = len - L + 1;
  const uint64_t item_end = min(ws + kSeg, nwin);
  const uint64_t span = item_end - ws;
  const uint64_t gs = ws + span * grp / Z;         // this group's windows [gs, ge)
  const uint64_t ge = ws + span * (grp + 1) / Z;
  const uint64_t S = (ge - gs + 1) / 2;            // windows per slice
  const uint8_t* baseA = text + off + gs;          // slice A starts at window gs
  const uint8_t* baseB = text + off + ge - S;      // slice B ends at window ge
  const uint64_t total = ge > gs ? S + L - 1 : 0;  // positions per slice

  Consts<Arith::kFq, F> k;
  k.load(fam, gl * F);
  uint32_t sa[F], sb[F], mn[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    sa[f] = 0;
    sb[f] = 0;
    mn[f] = 0xFFFFFFFFu;
  }
  uint2* bufA = sbuf[2 * grp];
  uint2* bufB = sbuf[2 * grp + 1];
  uint32_t* bufA256 = sbuf256[2 * grp];
  uint32_t* bufB256 = sbuf256[2 * grp + 1];
  uint64_t p_hi = total;
  bool first = true;
  while (p_hi > 0) {
    const uint64_t p_lo = p_hi > kChunk ? p_hi - kChunk : 0;
    const int cnt = static_cast<int>(p_hi - p_lo);
    for (int j = gl; j < cnt + static_cast<int>(L); j += G) {
      const uint64_t pos = p_lo + j;
      const uint32_t ca = pos < total ? baseA[pos] : 0u;
      const uint32_t cb = pos < total ? baseB[pos] : 0u;
      bufA[j] = make_uint2(ca, __float_as_uint(static_cast<float>(ca)));
      bufB[j] = make_uint2(cb, __float_as_uint(static_cast<float>(cb)));
      bufA256[j] = ca << 8;
      bufB256[j] = cb << 8;
    }
    __syncwarp(gmask);
    int j = cnt - 1;
    if (first) {  // L-1 warm-up positions: partial windows, not part of the minimum
      for (int w = 0; w < static_cast<int>(L) - 1; ++w, --j) {
        const uint2 oa = bufA[j + L], ob = bufB[j + L];
        const uint32_t ca = bufA256[j], cb = bufB256[j];
#pragma unroll
        for (int f = 0; f < F; ++f) {
          sa[f] = k.roll(f, sa[f], ca, oa.x, __uint_as_float(oa.y));
          sb[f] = k.roll(f, sb[f], cb, ob.x, __uint_as_float(ob.y));
        }
      }
      first = false;
    }
    for (; j >= 3; j -= 4) {  // 4 windows per slice per iteration: 32F window-function steps
      const uint2 oa0 = bufA[j + L], oa1 = bufA[j - 1 + L], oa2 = bufA[j - 2 + L],
                  oa3 = bufA[j - 3 + L];
      const uint2 ob0 = bufB[j + L], ob1 = bufB[j - 1 + L], ob2 = bufB[j - 2 + L],
                  ob3 = bufB[j - 3 + L];
      const uint32_t ca0 = bufA256[j], ca1 = bufA256[j - 1], ca2 = bufA256[j - 2],
                     ca3 = bufA256[j - 3];
      const uint32_t cb0 = bufB256[j], cb1 = bufB256[j - 1], cb2 = bufB256[j - 2],
                     cb3 = bufB256[j - 3];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const uint32_t a0 = k.roll(f, sa[f], ca0, oa0.x, __uint_as_float(oa0.y));
        const uint32_t b0 = k.roll(f, sb[f], cb0, ob0.x, __uint_as_float(ob0.y));
        const uint32_t a1 = k.roll(f, a0, ca1, oa1.x, __uint_as_float(oa1.y));
        const uint32_t b1 = k.roll(f, b0, cb1, ob1.x, __uint_as_float(ob1.y));
        const uint32_t a2 = k.roll(f, a1, ca2, oa2.x, __uint_as_float(oa2.y));
        const uint32_t b2 = k.roll(f, b1, cb2, ob2.x, __uint_as_float(ob2.y));
        const uint32_t a3 = k.roll(f, a2, ca3, oa3.x, __uint_as_float(oa3.y));
        const uint32_t b3 = k.roll(f, b2, cb3, ob3.x, __uint_as_float(ob3.y));
        sa[f] = a3;
        sb[f] = b3;
        mn[f] = __vimin3_u32(mn[f], a0, a1);
        mn[f] = __vimin3_u32(mn[f], b0, b1);
        mn[f] = __vimin3_u32(mn[f], a2, a3);
        mn[f] = __vimin3_u32(mn[f], b2, b3);
      }
    }
    for (; j >= 1; j -= 2) {
      const uint2 oa0 = bufA[j + L], oa1 = bufA[j - 1 + L];
      const uint2 ob0 = bufB[j + L], ob1 = bufB[j - 1 + L];
      const uint32_t ca0 = bufA256[j], ca1 = bufA256[j - 1];
      const uint32_t cb0 = bufB256[j], cb1 = bufB256[j - 1];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const uint32_t a0 = k.roll(f, sa[f], ca0, oa0.x, __uint_as_float(oa0.y));
        const uint32_t b0 = k.roll(f, sb[f], cb0, ob0.x, __uint_as_float(ob0.y));
        const uint32_t a1 = k.roll(f, a0, ca1, oa1.x, __uint_as_float(oa1.y));
        const uint32_t b1 = k.roll(f, b0, cb1, ob1.x, __uint_as_float(ob1.y));
        sa[f] = a1;
        sb[f] = b1;
        mn[f] = __vimin3_u32(mn[f], a0, a1);
        mn[f] = __vimin3_u32(mn[f], b0, b1);
      }
    }
    if (j == 0) {
      const uint2 oa = bufA[L], ob = bufB[L];
      const uint32_t ca = bufA256[0], cb = bufB256[0];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        sa[f] = k.roll(f, sa[f], ca, oa.x, __uint_as_float(oa.y));
        sb[f] = k.roll(f, sb[f], cb, ob.x, __uint_as_float(ob.y));
        mn[f] = __vimin3_u32(mn[f], sa[f], sb[f]);
      }
    }
    __syncwarp(gmask);
    p_hi = p_lo;
  }
  if (Z > 1) {  // the groups' partial minima meet
    __syncwarp();
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int o = G; o < 32; o <<= 1) mn[f] = min(mn[f], __shfl_xor_sync(0xFFFFFFFFu, mn[f], o));
    if (grp != 0) return;
  }
#pragma unroll
  for (int f = 0; f < F; ++f) mn[f] >>= 8;  // scaled state -> canonical value
  uint32_t* out = sig + doc * H;
  const int fbase = gl * F;
  if (multi) {
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (fbase + f < static_cast<int>(H)) atomicMin(out + fbase + f, mn[f]);
    return;
  }
  if ((H % 4) == 0 && (F % 4) == 0 && fbase + F <= static_cast<int>(H)) {
#pragma unroll
    for (int f = 0; f < F; f += 4)
      *reinterpret_cast<uint4*>(out + fbase + f) = make_uint4(mn[f], mn[f + 1], mn[f + 2], mn[f + 3]);
  } else {
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (fbase + f < static_cast<int>(H)) out[fbase + f] = mn[f];
  }
  if (band == nullptr) return;
#pragma unroll
  for (int f = 0; f < F; ++f) srow[fbase + f] = mn[f];
  __syncwarp(gmask);
  for (uint32_t jb = gl; jb < bands; jb += G) {
    uint64_t sum = 0;
    for (uint32_t r = 0; r < rows; ++r) sum += srow[jb * rows + r];
    band[doc * bands + jb] = K ? static_cast<uint32_t>(sum % K) : static_cast<uint32_t>(sum);
  }
}

// row length of a warp's staging buffers
__host__ __device__ constexpr int k1_buf_rows(int Z, int SL) {
  return (SL == 2 ? 128 : chunk_for(Z)) + kLMax;
}

template <Arith A, int F, int Z, class T, int SL>
struct K1Item {
  static __device__ __forceinline__ void run(
      uint64_t item, const T* text, const uint64_t* offsets, const uint32_t* item_doc,
      const uint64_t* item_off, const FamPtrs& fam, uint32_t L, uint32_t H, uint32_t bands,
      uint32_t rows, uint32_t K, uint32_t* sig, uint32_t* band, uint2* sbuf, uint32_t* sbuf256,
      uint32_t* srow) {
    constexpr int R = k1_buf_rows(Z, SL);
    if constexpr (SL == 2) {
      static_assert(A == Arith::kFq && R == kLMax + 128, "dual-slice layout");
      k1_item_dual<F, Z>(item, text, offsets, item_doc, item_off, fam, L, H, bands, rows, K, sig,
                         band, reinterpret_cast<uint2(*)[R]>(sbuf),
                         reinterpret_cast<uint32_t(*)[R]>(sbuf256), srow);
    } else {
      k1_item<A, F, Z, T>(item, text, offsets, item_doc, item_off, fam, L, H, bands, rows, K, sig,
                          band, reinterpret_cast<uint2(*)[R]>(sbuf),
                          reinterpret_cast<uint32_t(*)[R]>(sbuf256), srow);
    }
  }
};

// next_item == nullptr: one item per warp (grid = items / kWarps).  Otherwise
// persistent: a grid of resident blocks whose warps pull items from a global
// counter, so a block is never held by one long item while its other warps
// idle (lognormal lengths) and no block slot waits for a straggler.
template <Arith A, int F, int Z, class T, int SL>
__global__ void ND_K1_BOUNDS
    k_signature(const T* __restrict__ text, const uint64_t* __restrict__ offsets,
                const uint32_t* __restrict__ item_doc, const uint64_t* __restrict__ item_off,
                uint64_t n_items, FamPtrs fam, uint32_t L, uint32_t H, uint32_t bands,
                uint32_t rows, uint32_t K, uint32_t* __restrict__ sig,
                uint32_t* __restrict__ band, unsigned long long* __restrict__ next_item) {
  constexpr int G = 32 / Z;  // lanes per group
  constexpr int Hp = G * F;
  constexpr int kBuf = k1_buf_rows(Z, SL);
  constexpr int kSlots = Z * SL;  // staging buffers per warp
  __shared__ __align__(16) uint2 sbuf[kWarps][kSlots][kBuf];
  __shared__ __align__(16) uint32_t sbuf256[kWarps][kSlots][kBuf];
  __shared__ __align__(16) uint32_t srow[kWarps][Hp];
  const int warp = threadIdx.x >> 5;
  if (next_item == nullptr) {
    const uint64_t item = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
    if (item < n_items)
      K1Item<A, F, Z, T, SL>::run(item, text, offsets, item_doc, item_off, fam, L, H, bands, rows,
                                  K, sig, band, &sbuf[warp][0][0], &sbuf256[warp][0][0], srow[warp]);
    return;
  }
  const int lane = threadIdx.x & 31;
  unsigned long long item = 0;
  if (lane == 0) item = atomicAdd(next_item, 1ull);
  item = __shfl_sync(0xFFFFFFFFu, item, 0);
  while (item < n_items) {
    // claim the next item before working on this one: the atomic's round trip
    // overlaps the item instead of idling the warp between items
    unsigned long long next = 0;
    if (lane == 0) next = atomicAdd(next_item, 1ull);
    K1Item<A, F, Z, T, SL>::run(item, text, offsets, item_doc, item_off, fam, L, H, bands, rows, K,
                                sig, band, &sbuf[warp][0][0], &sbuf256[warp][0][0], srow[warp]);
    __syncwarp();
    item = __shfl_sync(0xFFFFFFFFu, next, 0);
  }
}

template <Arith A, int F, int Z, class T = uint8_t, int SL = 1>
void launch_k1(const DevFamily& fam, const void* d_text, const uint64_t* d_offsets,
               const uint32_t* item_doc, const uint64_t* item_off, uint64_t items, uint32_t bands,
               uint32_t rows, uint32_t K, uint32_t* d_sig, uint32_t* d_band,
               unsigned long long* counter, cudaStream_t s) {
  FamPtrs p{fam.q,   fam.qln,  fam.m,   fam.negp, fam.c3, fam.qp,
            fam.qlnp, fam.c1e, fam.m45, fam.p,    fam.rf};
  uint64_t blocks = (items + kWarps - 1) / kWarps;
  if (counter) {  // persistent: resident blocks only
    static int per_sm = -1;
    if (per_sm < 0) {
      ND_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_signature<A, F, Z, T, SL>,
                                                            kWarps * 32, 0));
      per_sm = std::max(per_sm, 1);
    }
    const uint64_t resident = static_cast<uint64_t>(per_sm) * sm_count();
    if (blocks > resident) {
      blocks = resident;
      ND_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    } else {
      counter = nullptr;  // one wave anyway
    }
  }
  k_signature<A, F, Z, T, SL><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
      static_cast<const T*>(d_text), d_offsets, item_doc, item_off, items, p, fam.L, fam.H, bands,
      rows, K, d_sig, d_band, counter);
  ND_CHECK_LAUNCH();
}

using Launcher = void (*)(const DevFamily&, const void*, const uint64_t*, const uint32_t*,
                          const uint64_t*, uint64_t, uint32_t, uint32_t, uint32_t, uint32_t*,
                          uint32_t*, unsigned long long*, cudaStream_t);

// (arith, Hp) -> instantiation; F = functions per lane, Z = window slices per
// warp.  ND_K1_FZ="F,Z" overrides the default shape (tuning experiments).
Launcher pick_launcher(bool int_arith, uint32_t Hp, bool codepoint, bool exact) {
  if (exact) {  // families outside the fast domains (nd_family_upload)
    switch (Hp) {
      case 32: return codepoint ? launch_k1<Arith::kExact, 1, 1, uint32_t> : launch_k1<Arith::kExact, 1, 1>;
      case 64: return codepoint ? launch_k1<Arith::kExact, 2, 1, uint32_t> : launch_k1<Arith::kExact, 2, 1>;
      case 128: return codepoint ? launch_k1<Arith::kExact, 4, 1, uint32_t> : launch_k1<Arith::kExact, 4, 1>;
      case 256: return codepoint ? launch_k1<Arith::kExact, 8, 1, uint32_t> : launch_k1<Arith::kExact, 8, 1>;
      case 512: return codepoint ? launch_k1<Arith::kExact, 16, 1, uint32_t> : launch_k1<Arith::kExact, 16, 1>;
    }
    return nullptr;
  }
  if (codepoint) {  // u32 units: wide arithmetic
    switch (Hp) {
      case 32: return launch_k1<Arith::kWide, 1, 1, uint32_t>;
      case 64: return launch_k1<Arith::kWide, 2, 1, uint32_t>;
      case 128: return launch_k1<Arith::kWide, 4, 1, uint32_t>;
      case 256: return launch_k1<Arith::kWide, 8, 1, uint32_t>;
      case 512: return launch_k1<Arith::kWide, 16, 1, uint32_t>;
    }
    return nullptr;
  }
  if (int_arith) {
    switch (Hp) {
      case 32: return launch_k1<Arith::kInt, 1, 1>;
      case 64: return launch_k1<Arith::kInt, 2, 1>;
      case 128: return launch_k1<Arith::kInt, 4, 1>;
      case 256: return launch_k1<Arith::kInt, 8, 1>;
      case 512: return launch_k1<Arith::kInt, 16, 1>;
    }
    return nullptr;
  }
  const char* dual = getenv("ND_K1_DUAL");
  const bool dual_on = !(dual && std::string(dual) == "0");
  // H=128: 2 groups x 16 lanes x 8 functions x 2 slices (3.15 T HWE/s on C2;
  // ND_K1_DUALZ=1: 32 lanes x 4 functions x 2 slices, 3.07 T)
  const char* dz = getenv("ND_K1_DUALZ");
  if (dual_on && Hp == 128 && dz && std::string(dz) == "1")
    return launch_k1<Arith::kFq, 4, 1, uint8_t, 2>;
  if (dual_on && Hp == 128) return launch_k1<Arith::kFq, 8, 2, uint8_t, 2>;
  if (dual_on && Hp == 256) return launch_k1<Arith::kFq, 8, 1, uint8_t, 2>;
  const char* fz = getenv("ND_K1_FZ");
  if (fz && Hp == 128) {
    std::string v(fz);
    if (v == "4,1") return launch_k1<Arith::kFq, 4, 1>;
    if (v == "8,2") return launch_k1<Arith::kFq, 8, 2>;
    if (v == "16,4") return launch_k1<Arith::kFq, 16, 4>;
  }
  switch (Hp) {
    case 32: return launch_k1<Arith::kFq, 4, 4>;
    case 64: return launch_k1<Arith::kFq, 8, 4>;
    case 128: return launch_k1<Arith::kFq, 8, 2>;
    case 256: return launch_k1<Arith::kFq, 8, 1>;
    case 512: return launch_k1<Arith::kFq, 16, 1>;
  }
  return nullptr;
}

}  // namespace


void k1_gate_wait(const unsigned int* flag, unsigned int epoch, cudaStream_t s) {
  k_gate_wait<<<1, 1, 0, s>>>(flag, epoch);
  ND_CHECK_LAUNCH();
}

void launch_signatures(const DevFamily& fam, const uint8_t* d_bytes, const uint64_t* d_offsets,
                       uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                       uint32_t* d_band, SigScratch& sc, cudaStream_t s, bool check_short,
                       const uint64_t* h_offsets, const K1Gate* gate,
                       const uint32_t* doc_class, uint32_t class_lo, uint32_t class_hi) {
  if (n == 0) return;
  if (fam.L == 0 || fam.L > static_cast<uint32_t>(kLMax))
    fail(ND_ERR_CONFIG, "shingle length must be in [1, 64] on the GPU path");
  if (n > 0xFFFFFFFFull) fail(ND_ERR_CONFIG, "batch exceeds 2^32 documents");
  unsigned tb = 256;
  const void* d_text = d_bytes;
  // only the documents whose class lies in [class_lo, class_hi] (codepoint
  // batches: the u16 pass and K1w each take their own documents)
  const uint32_t* wide_mask = doc_class;
  if (fam.unit == 1 && fam.narrow_ok) {
    // pure ASCII batch: units are the bytes -- the byte path on the text as it
    // is (no decode); one pass over the text decides
    const char* nv = getenv("ND_K1_NARROW");
    if (!(nv && nv[0] == '0')) {
      uint64_t ends[2];
      if (h_offsets) {
        ends[0] = h_offsets[0];
        ends[1] = h_offsets[n];
      } else {
        ND_CUDA(cudaMemcpyAsync(&ends[0], d_offsets, 8, cudaMemcpyDeviceToHost, s));
        ND_CUDA(cudaMemcpyAsync(&ends[1], d_offsets + n, 8, cudaMemcpyDeviceToHost, s));
      }
      unsigned int* flag = sc.flags.as<unsigned int>(4);
      ND_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned int), s));
      ND_CUDA(cudaStreamSynchronize(s));
      unsigned int high = 1;
      if (ends[1] > ends[0]) {
        k_any_high<<<8 * sm_count(), 256, 0, s>>>(d_bytes, ends[0], ends[1], flag);
        ND_CHECK_LAUNCH();
        ND_CUDA(cudaMemcpyAsync(&high, flag, sizeof high, cudaMemcpyDeviceToHost, s));
        ND_CUDA(cudaStreamSynchronize(s));
      }
      if (!high) {
        DevFamily byte_view = fam;
        byte_view.unit = 0;
        byte_view.narrow_ok = false;
        launch_signatures(byte_view, d_bytes, d_offsets, n, bands, rows, K, d_sig, d_band, sc, s,
                          /*check_short=*/true, h_offsets, gate, doc_class, class_lo, class_hi);
        return;
      }
    }
  }
  if (fam.unit == 1) {
    // codepoint units: decode, then plan and sign over the u32 unit arrays;
    // unit counts are only known on the device, so the short check runs there
    const char* nv = getenv("ND_K1_NARROW");  // 0: every codepoint document through K1w
    const bool narrow = fam.narrow_ok && !(nv && nv[0] == '0');
    // Documents whose code points are all < 256 hash exactly like bytes (the
    // fq arithmetic's domain: units < 256, 2^21 <= p < 2^23) and run the byte
    // kernels; those below 2^16 run K1j over 16-bit units; the rest K1w.  The
    // decode classifies every document (count pass) and writes 16-bit units
    // for the narrow classes, u32 units only for the documents K1w takes.
    CodepointClasses cc;
    cc.cls_buf = &sc.wide;
    cc.cnt_buf = &sc.cls_cnt;
    cc.u16_buf = &sc.units16;
    cc.wide_from = fam.jit16 ? 2u : 1u;
    const uint32_t* units = nullptr;
    const uint64_t* uoff = nullptr;
    decode_codepoints_device(d_bytes, d_offsets, n, sc.units, sc.unit_off, sc.unit_cnt,
                             sc.scan_tmp, s, &units, &uoff, narrow ? &cc : nullptr);
    d_text = units;
    d_offsets = uoff;
    h_offsets = nullptr;
    check_short = true;
    if (narrow) {
      const uint32_t* wide = cc.cls;
      const uint32_t nwide = cc.n_wide, nastral = cc.n_astral;
      const uint64_t total = cc.total;
      // K1w below: the documents with a code point >= 2^16 when the u16 pass
      // runs, else every document with one >= 256
      class_lo = cc.wide_from;
      class_hi = 2u;
      if (nwide < n) {
        uint8_t* u8 = sc.units8.as<uint8_t>(total + 16);
        if (total) {
          k_u16_to_u8<<<4 * sm_count(), 256, 0, s>>>(cc.u16, total, u8);
          ND_CHECK_LAUNCH();
        }
        DevFamily byte_view = fam;
        byte_view.unit = 0;
        byte_view.narrow_ok = false;
        // only the documents of class 0 when others exist (their rows come
        // from the u16 pass or K1w); every document is still checked for length
        launch_signatures(byte_view, u8, uoff, n, bands, rows, K, d_sig, d_band, sc, s,
                          /*check_short=*/true, nullptr, nullptr, nwide ? wide : nullptr, 0u, 0u);
        if (nwide == 0) return;
      }
      if (fam.jit16 && nwide > nastral) {
        // K1j over 16-bit units for the documents of class 1 (code points
        // < 2^16, some >= 256)
        DevFamily v16 = fam;
        v16.unit = 2;
        v16.narrow_ok = false;
        launch_signatures(v16, reinterpret_cast<const uint8_t*>(cc.u16), uoff, n, bands, rows, K,
                          d_sig, d_band, sc, s, /*check_short=*/true, nullptr, nullptr, wide, 1u, 1u);
        if (nastral == 0) return;
      }
      wide_mask = wide;  // K1w below: the documents of classes [class_lo, 2]
    }
  }
  // K1j splits documents into items of seg_len windows; a small batch gets
  // shorter items so that the pass-major grid still fills the GPU (~1.5
  // items per resident lane; the register kernels keep kSeg)
  uint32_t seg_len = kSeg;
  const void* jit_handle = fam.unit == 0 ? fam.jit : fam.unit == 2 ? fam.jit16 : nullptr;
  const bool jit_path = jit_handle != nullptr;
  if (jit_path) {
    // target items: 1.5 per resident lane (ND_K1J_HALF_ITEMS=h: h/2 per lane; tuning)
    static const uint64_t half_items = [] {
      const char* v = getenv("ND_K1J_HALF_ITEMS");
      return static_cast<uint64_t>(v ? std::max(1, std::min(16, atoi(v))) : 3);
    }();
    const uint64_t target = half_items * 32 / 2 * k1_jit_resident_warps(jit_handle);
    if (n < target) {
      uint64_t bytes = 0;
      if (h_offsets) {
        bytes = h_offsets[n] - h_offsets[0];
      } else {
        uint64_t ends[2] = {0, 0};
        ND_CUDA(cudaMemcpyAsync(&ends[0], d_offsets, 8, cudaMemcpyDeviceToHost, s));
        ND_CUDA(cudaMemcpyAsync(&ends[1], d_offsets + n, 8, cudaMemcpyDeviceToHost, s));
        ND_CUDA(cudaStreamSynchronize(s));
        bytes = ends[1] - ends[0];
      }
      const uint64_t per = (bytes + target - 1) / target;  // ~windows per item
      const char* ms = getenv("ND_K1J_MIN_SEG");           // tuning
      const uint64_t lo = ms ? std::max(64, atoi(ms)) : 512;
      seg_len = static_cast<uint32_t>(std::min<uint64_t>(kSeg, std::max<uint64_t>(lo, (per + 63) / 64 * 64)));
    }
  }
  uint32_t hflags[4] = {0, 0, 0, 0};
  uint64_t host_items = n;  // work items, known on the host when h_offsets is
  if (h_offsets) {  // host planning: no device round trip (the pipelines keep running)
    host_items = 0;
    for (uint64_t d = 0; d < n; ++d) {
      uint64_t len = h_offsets[d + 1] - h_offsets[d];
      if (len < fam.L) {
        hflags[0] = 1;
        ++host_items;
        continue;
      }
      const uint64_t segs = (len - fam.L + 1 + seg_len - 1) / seg_len;
      host_items += segs;
      if (segs > 1) ++hflags[1];
    }
    if (check_short && hflags[0]) fail(ND_ERR_SHORT, "a document has fewer units than the shingle length");
  }
  uint32_t* seg_count = nullptr;
  uint32_t* flags = nullptr;
  if (!h_offsets || hflags[1] || wide_mask) {
    seg_count = sc.seg_count.as<uint32_t>(n);
    flags = sc.flags.as<uint32_t>(4);
    ND_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(uint32_t), s));
    k_plan<<<static_cast<unsigned>((n + tb - 1) / tb), tb, 0, s>>>(d_offsets, n, fam.L, seg_count,
                                                                    flags, seg_len);
    ND_CHECK_LAUNCH();
    if (!h_offsets) {
      ND_CUDA(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
      if (check_short && hflags[0]) fail(ND_ERR_SHORT, "a document has fewer units than the shingle length");
    }
    if (wide_mask) {
      k_keep_class<<<static_cast<unsigned>((n + tb - 1) / tb), tb, 0, s>>>(wide_mask, n, class_lo,
                                                                          class_hi, seg_count);
      ND_CHECK_LAUNCH();
    }
  }

  const uint32_t* item_doc = nullptr;
  const uint64_t* item_off = nullptr;
  uint64_t items = n;
  uint32_t nmulti = hflags[1];
  uint32_t* multi_docs = nullptr;
  if (nmulti || wide_mask) {
    uint64_t* off = sc.item_off.as<uint64_t>(n + 1);
    scan_u32_to_u64(seg_count, off, n, sc.scan_tmp, s);
    if (h_offsets) {
      items = host_items;
    } else {
      ND_CUDA(cudaMemcpyAsync(&items, off + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
    }
    uint32_t* idoc = sc.item_doc.as<uint32_t>(items);
    multi_docs = sc.multi_docs.as<uint32_t>(nmulti + 1);
    uint32_t* counter = flags + 2;
    ND_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    k_item_scatter<<<static_cast<unsigned>((n + tb - 1) / tb), tb, 0, s>>>(off, n, idoc, multi_docs,
                                                                           counter);
    ND_CHECK_LAUNCH();
    if (wide_mask) {  // the multi-item documents among the wide ones
      ND_CUDA(cudaMemcpyAsync(&nmulti, counter, 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
    }
    k_fill_multi<<<1024, 256, 0, s>>>(multi_docs, nmulti, fam.H, d_sig);
    ND_CHECK_LAUNCH();
    item_doc = idoc;
    item_off = off;
  }
  static const bool int_arith = [] {
    const char* v = getenv("ND_K1_KERNEL");
    return v && std::string(v) == "int";
  }();
  Launcher go = pick_launcher(int_arith, fam.Hp, fam.unit == 1, fam.exact);
  if (!go) fail(ND_ERR_CONFIG, "hash count must be at most 512 on the GPU path");
  static const bool persistent = [] {
    const char* v = getenv("ND_K1_PERSISTENT");
    return !(v && std::string(v) == "0");
  }();
  unsigned long long* counter =
      persistent ? sc.item_counter.as<unsigned long long>(1) : nullptr;
  if (jit_path) {
    // K1j: items sorted by length, then the family-specialised kernel
    uint32_t* keys = sc.order_keys.as<uint32_t>(items);
    uint32_t* order = sc.order_vals.as<uint32_t>(items);
    k_item_len_keys<<<static_cast<unsigned>((items + tb - 1) / tb), tb, 0, s>>>(
        d_offsets, item_doc, item_off, items, fam.L, seg_len, keys, order);
    ND_CHECK_LAUNCH();
    radix_sort_u32(keys, order, items, 14, sc.sort, s);
    k1_jit_launch(jit_handle, static_cast<const uint8_t*>(d_text), d_offsets, order, item_doc,
                  item_off, static_cast<uint32_t>(items), seg_len, d_sig,
                  sc.item_counter.as<unsigned long long>(k1_jit_passes(jit_handle)), s, gate);
    // band keys of every document from its finished row (keys is free again)
    if (d_band) launch_band_keys(d_sig, n, fam.H, bands, rows, K, d_band, keys, s);
    return;
  } else {
    go(fam, d_text, d_offsets, item_doc, item_off, items, bands, rows, K, d_sig, d_band, counter,
       s);
  }
  if (nmulti && d_band) {
    uint64_t total = static_cast<uint64_t>(nmulti) * bands;
    k_bands_from_rows<<<static_cast<unsigned>((total + tb - 1) / tb), tb, 0, s>>>(
        multi_docs, nmulti, d_sig, fam.H, bands, rows, K, d_band);
    ND_CHECK_LAUNCH();
  }
}

void launch_band_keys(const uint32_t* d_sig, uint64_t n, uint32_t H, uint32_t bands, uint32_t rows,
                      uint32_t K, uint32_t* d_band, uint32_t* d_docs, cudaStream_t s) {
  if (n == 0) return;
  if (n > 0xFFFFFFFFull) fail(ND_ERR_CONFIG, "batch exceeds 2^32 documents");
  const unsigned tb = 256;
  k_iota_docs<<<static_cast<unsigned>((n + tb - 1) / tb), tb, 0, s>>>(d_docs, n);
  ND_CHECK_LAUNCH();
  uint64_t total = n * bands;
  k_bands_from_rows<<<static_cast<unsigned>((total + tb - 1) / tb), tb, 0, s>>>(
      d_docs, static_cast<uint32_t>(n), d_sig, H, bands, rows, K, d_band);
  ND_CHECK_LAUNCH();
}

}  // namespace ndb
