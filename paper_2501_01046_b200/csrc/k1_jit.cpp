// K1j: family-specialised signature kernel, generated and compiled at
// nd_family_upload time (NVRTC, sm_100a) -- the same exact fq arithmetic as
// K1 (k_signature.cu, ND_K1_I2F form), with every per-function constant an
// instruction immediate.
//
// Why.  K1 is integer/FP issue bound at ~9 SASS per hash-window evaluation
// (HWE); with per-lane constants most of those instructions read three
// registers and the measured issue rate stalls on register-bank dispatch
// (profiles/r1_k1_ncu_full_1M.txt: dispatch + math-pipe throttle).  With the
// constants in the instruction stream the same roll sequence issues at 12.75
// HWE/clk/SM against 9.7 (scripts/k1_imm_microbench.cu).  Immediates are
// warp-uniform, so the layout flips: a warp runs 32 work items (one per lane,
// sorted by length so the lanes finish together) through the same block of F
// functions, then the next block.
//
// Walk per lane (one item = a document or an 8192-window segment of one;
// windows [wlo, we), characters [wlo, e), e = we + L - 1):
//   * state 0 at position e, warm-up over the L-1 partial windows (chars >= e
//     read as 0) -- identical to K1 (minhash.cpp:133-162 semantics: min over
//     the windows [wlo, we));
//   * single steps until position p+1 is 4-byte aligned in memory;
//   * whole aligned words: 4 windows per 32-bit load, c_in / c_out bytes
//     extracted with PRMT from the current word and a ring of the words above
//     (c_out = the character L positions up, already loaded);
//   * single steps down to wlo.
// Multi-item documents meet through atomicMin, as in K1.  Band keys
// (lsh.cpp:42-60) are summed from the finished rows by k_bands_from_rows.
// Scheduling is pass-major (one work counter per block of F functions), so
// all SMs run the same pass's code and the instruction cache holds it.
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "nd_internal.cuh"

namespace ndb {
namespace {

constexpr int kJitThreads = 128;

// Tuning knobs of the generated kernel (part of the cache key): functions per
// pass F (their states + minima stay in registers), the minimum resident
// blocks per SM handed to ptxas, and how many words ahead the text is loaded.
// Defaults per arithmetic, measured on the C2 shard (1M docs, H=128, B200,
// profiles/r2_k1j_variants.txt):
//   fq: F=16 / 6 blocks 66.9 ms (F=32 / 4 blocks 67.6, F=24 / 5 blocks 67.7,
//       F=32 / 5 blocks 74.4 (spills), F=16 / 8 blocks 73.4; prefetch 2: same)
//   dn: F=32 / 4 blocks / 2 words prefetched 63.7 ms (F=16 / 6 blocks 65.9,
//       F=20 / 5 64.8, F=32 / 4 / prefetch 1 64.1, F=40 / 4 65.1, F=48 / 4
//       67.8, F=64 / 2 67.0): with 7.5 instructions per HWE the per-pass
//       extraction and loop overhead and the exposed text load matter more
struct JitShape {
  int F = 32;
  int min_blocks = 4;
  int prefetch = 2;
  int unroll = 1;  // whole words per loop iteration (2: ND_K1J_UNROLL=2, slower)
  int arith = 1;   // 1: denormal-state arithmetic (dn, default); 0: the fq state of K1 (ND_K1J_ARITH=fq)
  int classes = 4; // dn: most w classes (c_in extractions per window) in one pass
  int pfw = 0;     // > 0: prefetch the text pfw words below the current one at every
                   // word (ND_K1J_PFW; ND_K1J_PFL2=1: into L2 instead of L1)
  int pfl2 = 0;
  int sring = 0;   // 1: text lines staged per lane in a 2-line shared-memory ring by
                   // cp.async one line ahead (ND_K1J_SRING=1)
  int uw = 1;      // bytes per text unit: 1 (bytes), 2 (code points < 2^16, fq only)
  int gptr = 0;    // 1: word pointer derived from the text pointer (LDG) instead of
                   // an integer address (generic LD); ND_K1J_GPTR=1
};

JitShape jit_shape() {
  JitShape j;
  if (const char* v = getenv("ND_K1J_ARITH")) j.arith = std::strcmp(v, "fq") == 0 ? 0 : 1;
  if (j.arith == 0) {
    j.F = 16;
    j.min_blocks = 6;
    j.prefetch = 1;
  }
  if (const char* v = getenv("ND_K1J_F")) j.F = std::max(4, std::min(64, atoi(v)));
  if (const char* v = getenv("ND_K1J_MINB")) j.min_blocks = std::max(1, std::min(16, atoi(v)));
  if (const char* v = getenv("ND_K1J_PREFETCH")) j.prefetch = std::max(1, std::min(2, atoi(v)));
  if (const char* v = getenv("ND_K1J_UNROLL")) j.unroll = std::max(1, std::min(2, atoi(v)));
  if (const char* v = getenv("ND_K1J_CLASSES")) j.classes = std::max(1, std::min(8, atoi(v)));
  if (const char* v = getenv("ND_K1J_GPTR")) j.gptr = atoi(v) ? 1 : 0;
  if (const char* v = getenv("ND_K1J_PFW")) j.pfw = std::max(0, std::min(4096, atoi(v)));
  if (const char* v = getenv("ND_K1J_PFL2")) j.pfl2 = atoi(v) ? 1 : 0;
  if (const char* v = getenv("ND_K1J_SRING")) j.sring = atoi(v) ? 1 : 0;
  if (j.unroll != 1) j.sring = 0;
  return j;
}

// ---- NVRTC, loaded on first use (the library does not link it) ----------
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  std::string error;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      r.error = std::string("libnvrtc not found: ") + dlerror();
      return r;
    }
#define ND_SYM(field, name)                                                 \
  r.field = reinterpret_cast<decltype(r.field)>(dlsym(h, name));            \
  if (!r.field) {                                                           \
    r.error = std::string("libnvrtc lacks ") + name;                        \
    return r;                                                               \
  }
    ND_SYM(create, "nvrtcCreateProgram")
    ND_SYM(compile, "nvrtcCompileProgram")
    ND_SYM(cubin_size, "nvrtcGetCUBINSize")
    ND_SYM(cubin, "nvrtcGetCUBIN")
    ND_SYM(log_size, "nvrtcGetProgramLogSize")
    ND_SYM(log, "nvrtcGetProgramLog")
    ND_SYM(destroy, "nvrtcDestroyProgram")
#undef ND_SYM
    r.ok = true;
    return r;
  }();
  return n;
}

// ---- source generation -------------------------------------------------------
struct FnConst {
  uint32_t q, qln256, negp256;
  uint32_t qp256_bits, qlnp_bits;
};

FnConst fn_const(const nd_hash_fn& f, uint32_t L) {
  const uint64_t p = f.modulus, q = f.base;
  uint64_t qL = 1;
  for (uint32_t i = 0; i < L; ++i) qL = qL * q % p;  // q^L mod p
  const uint32_t qln = static_cast<uint32_t>((p - qL) % p);
  const float qp = static_cast<float>(static_cast<double>(q) / static_cast<double>(p));
  const float qp256 = qp * 0.00390625f;  // exact (power-of-two scaling)
  const float qlnp = static_cast<float>(static_cast<double>(qln) / static_cast<double>(p));
  FnConst c;
  c.q = static_cast<uint32_t>(q);
  c.qln256 = qln << 8;
  c.negp256 = static_cast<uint32_t>(0u - static_cast<uint32_t>(p)) << 8;
  std::memcpy(&c.qp256_bits, &qp256, 4);
  std::memcpy(&c.qlnp_bits, &qlnp, 4);
  return c;
}

std::string hex(uint32_t v) {
  char b[16];
  std::snprintf(b, sizeof b, "0x%08xu", v);
  return b;
}

// rol(state, <window i>) with function f's constants as literals
std::string rol_call(const std::string& st, int i, const FnConst& c) {
  std::ostringstream o;
  o << "rol(" << st << ", ci" << i << ", co" << i << ", cf" << i << ", " << hex(c.q) << ", "
    << hex(c.qln256) << ", " << hex(c.negp256) << ", __uint_as_float(" << hex(c.qp256_bits)
    << "), __uint_as_float(" << hex(c.qlnp_bits) << "), c5)";
  return o.str();
}

// ---- dn arithmetic: the state as a negative denormal -------------------------
// The fq roll spends one instruction per HWE converting the state to float
// (I2FP) for the quotient estimate.  dn keeps the state as the bit pattern
// z = 0x80000000 + c (c < p < 2^23), which *is* the float -c * 2^-149 (sign
// set, exponent field 0: a denormal), so the estimate FFMA reads the state
// register directly:
//
//   t1 = (c_out + 256 g) * B                       FMUL  (shared float c_out)
//   R  = z_f * A + t1      = (c q/p + t1) U        FFMA  (A = -fl(q/p) 2^(e-1))
//   Kb = bits(R + M, round-down) = v +- floor(R/U) FADD.RM
//   z' = c_out*QLn + (c_in + w) + z*q + Kb*(-+p)   3 IMAD (0x80000000*q == 0x80000000)
//   z' = min_s32(z' + p, z')                       VIADDMNMX.S32 (the wrap at INT_MIN
//                                                  canonicalises r in [-p, p))
//
// U = 2^(e-150) is the ulp of M's binade e, so the FADD leaves k' = floor(R/U)
// in the low bits of Kb.  The float sees c_out + 256g where the integers see
// c_out: R/U = u/p + n + f + eps with n + f = 256 g QLn / p (n integer,
// f in [1/64, 63/64], g <= 64) and |eps| < 0.0094 (rounding of fl(q/p) and of
// R < 2^17: 2^-8 each; t1 < 2^15: 2^-10; fl(QLn/p): 2^-11; the dropped
// c_in/p < 2^-13), so
// floor(R/U) - n = k' in {Q, Q+1} and r = u - k' p in [-p, p).  The integer
// chain cancels both Kb's bias and the offset n through w: Kb = t + k' with
// t = w p^-1 (mod 2^32), so Kb*(-p) = -w - k' p against the +w the c_in
// extraction (one PRMT: c_in in byte 0, w's bytes 1..3) adds.  For each
// function, v = t - n (M > 0) or v = n - t (M < 0, multiplier +p) must be a
// normal float with e in [30, ehi] and room for floor(R/U) in its mantissa;
// that holds for ~38% of random w, so the functions of a pass are grouped
// into a few classes sharing w (one c_in PRMT per class and window) by a
// seeded search.  Per HWE: FMUL, FFMA, FADD, 3 IMAD, VIADDMNMX + half a
// VIMNMX3 = 7.5 (fq: 8.5).  The running minima are min_s32 of the z's; the
// signature value is m ^ 0x80000000.
struct DnFn {
  uint32_t fn, cls;
  uint32_t q, qln, kp, p;
  uint32_t a_bits, b_bits, m_bits;
};

struct DnPass {
  uint32_t g = 1;
  std::vector<uint32_t> w;
  std::vector<DnFn> fns;
};

struct DnInfo {
  uint32_t p, q, qln, pinv;
  float qp, qlnp;
  int ehi;
};

constexpr int kDnElo = 30;
constexpr uint32_t kDnMaxG = 64;  // offsets 256g: t1 < 2^15 units keeps |eps| < 0.0094

DnInfo dn_info(const nd_hash_fn& f, uint32_t L) {
  DnInfo d;
  d.p = f.modulus;
  d.q = f.base;
  uint64_t qL = 1;
  for (uint32_t i = 0; i < L; ++i) qL = qL * d.q % d.p;
  d.qln = static_cast<uint32_t>((d.p - qL) % d.p);
  uint32_t inv = d.p;  // p^-1 mod 2^32 by Newton (3 -> 6 -> 12 -> 24 -> 48 bits)
  for (int i = 0; i < 5; ++i) inv *= 2u - d.p * inv;
  d.pinv = inv;
  d.qp = static_cast<float>(static_cast<double>(d.q) / d.p);
  d.qlnp = static_cast<float>(static_cast<double>(d.qln) / d.p);
  int ex = 0;
  std::frexp(d.qp, &ex);  // qp < 2^ex
  d.ehi = 128 - ex;       // |A| = qp 2^(e-1) < 2^127
  return d;
}

bool dn_offset_ok(const DnInfo& d, uint32_t g) {
  const uint64_t rem = (256ull * g * d.qln) % d.p;
  return rem * 64 >= d.p && rem * 64 <= 63ull * d.p;  // f in [1/64, 63/64]
}

bool dn_fit(const DnInfo& d, uint32_t g, uint32_t w, DnFn* out) {
  const uint64_t n = 256ull * g * d.qln / d.p;
  const uint32_t qb = d.q + 257u + 256u * g;  // floor(R/U) <= q + 256 + n + 1
  const uint32_t t = w * d.pinv;
  const uint32_t vp = t - static_cast<uint32_t>(n), vn = static_cast<uint32_t>(n) - t;
  auto ok_e = [&](uint32_t x) {
    const int e = static_cast<int>((x >> 23) & 0xFF);
    return e >= kDnElo && e <= d.ehi;
  };
  uint32_t v;
  bool neg;
  if (vp < 0x80000000u && ok_e(vp) && (vp & 0x7FFFFFu) + qb <= 0x7FFFFFu) {
    v = vp;
    neg = false;
  } else if (vn >= 0x80000000u && ok_e(vn) && (vn & 0x7FFFFFu) >= qb) {
    v = vn;
    neg = true;
  } else {
    return false;
  }
  if (out) {
    const int e = static_cast<int>((v >> 23) & 0xFF);
    const float A = -std::ldexp(d.qp, e - 1);   // exact (power-of-two scaling, normal)
    const float B = std::ldexp(d.qlnp, e - 150);
    out->q = d.q;
    out->qln = d.qln;
    out->p = d.p;
    out->kp = neg ? d.p : 0u - d.p;
    std::memcpy(&out->a_bits, &A, 4);
    std::memcpy(&out->b_bits, &B, 4);
    out->m_bits = v;
  }
  return true;
}

// Groups the family's functions into passes of at most F functions, each pass
// with one offset g and at most `classes` values of w.  Deterministic for a
// family (seeded).  Functions that fit no offset g <= 64 (256 g QLn within
// p/64 of a multiple of p for every g -- rare) or no w go to `fq`: they run
// fq passes of the same kernel.
struct DnPlan {
  std::vector<DnPass> passes;
  std::vector<uint32_t> fq;
};

DnPlan dn_plan(const nd_hash_fn* fns, uint32_t H, uint32_t L, int F, int classes) {
  DnPlan plan;
  std::vector<DnInfo> info(H);
  for (uint32_t i = 0; i < H; ++i) info[i] = dn_info(fns[i], L);
  std::vector<uint32_t> rest;
  for (uint32_t i = 0; i < H; ++i) {
    bool any = false;
    for (uint32_t g = 1; g <= kDnMaxG && !any; ++g) any = dn_offset_ok(info[i], g);
    (any ? rest : plan.fq).push_back(i);
  }
  uint64_t rng = 0x9E3779B97F4A7C15ull;
  auto next = [&] {  // splitmix64
    uint64_t z = (rng += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return static_cast<uint32_t>((z ^ (z >> 31)) >> 16);
  };
  while (!rest.empty()) {
    const size_t want = std::min<size_t>(static_cast<size_t>(F), rest.size());
    DnPass pass;
    size_t best_elig = 0;
    for (uint32_t g = 1; g <= kDnMaxG && best_elig < rest.size(); ++g) {
      size_t c = 0;
      for (uint32_t j : rest) c += dn_offset_ok(info[j], g);
      if (c > best_elig) {
        best_elig = c;
        pass.g = g;
      }
    }
    std::vector<char> taken(H, 0);
    std::vector<uint32_t> cand;
    for (uint32_t j : rest)
      if (dn_offset_ok(info[j], pass.g)) cand.push_back(j);
    while (pass.fns.size() < want && static_cast<int>(pass.w.size()) < classes) {
      const size_t need = want - pass.fns.size();
      uint32_t best_w = 0;
      size_t best = 0;
      for (int trial = 0; trial < 8192 && best < need; ++trial) {
        const uint32_t w = next() << 8;  // low byte 0: c_in goes there
        size_t c = 0;
        for (uint32_t j : cand)
          if (!taken[j] && dn_fit(info[j], pass.g, w, nullptr)) ++c;
        if (c > best) {
          best = c;
          best_w = w;
        }
      }
      if (best == 0) break;
      const uint32_t cls = static_cast<uint32_t>(pass.w.size());
      pass.w.push_back(best_w);
      for (uint32_t j : cand) {
        if (pass.fns.size() >= want) break;
        DnFn f;
        if (taken[j] || !dn_fit(info[j], pass.g, best_w, &f)) continue;
        f.fn = j;
        f.cls = cls;
        taken[j] = 1;
        pass.fns.push_back(f);
      }
    }
    if (pass.fns.empty()) {  // nothing of the rest fits this pass's g
      bool moved = false;
      std::vector<uint32_t> left;
      for (uint32_t j : rest) {
        if (!moved && dn_offset_ok(info[j], pass.g)) {
          plan.fq.push_back(j);  // one function at a time keeps the loop finite
          moved = true;
        } else {
          left.push_back(j);
        }
      }
      if (!moved) {
        plan.fq.insert(plan.fq.end(), left.begin(), left.end());
        left.clear();
      }
      rest.swap(left);
      continue;
    }
    std::sort(pass.fns.begin(), pass.fns.end(),
              [](const DnFn& a, const DnFn& b) { return a.fn < b.fn; });
    std::vector<uint32_t> left;
    for (uint32_t j : rest)
      if (!taken[j]) left.push_back(j);
    rest.swap(left);
    plan.passes.push_back(std::move(pass));
  }
  std::sort(plan.fq.begin(), plan.fq.end());
  return plan;
}

std::string fbits(uint32_t v) { return "__uint_as_float(" + hex(v) + ")"; }

std::string rold_call(const std::string& st, int i, const DnFn& c) {
  std::ostringstream o;
  o << "rold(" << st << ", x" << c.cls << "_" << i << ", co" << i << ", cf" << i << ", "
    << hex(c.q) << ", " << hex(c.qln) << ", " << hex(c.kp) << ", " << hex(c.p) << ", "
    << fbits(c.a_bits) << ", " << fbits(c.b_bits) << ", " << fbits(c.m_bits) << ")";
  return o.str();
}

// One pass's functions in either arithmetic (fq: fb.., dn: an explicit list).
struct PassFns {
  std::vector<uint32_t> fn;   // signature positions
  std::vector<FnConst> fq;    // arith 0
  const DnPass* dn = nullptr; // arith 1
};

std::string generate(const nd_hash_fn* fns, uint32_t H, uint32_t L, const JitShape& js,
                     uint32_t* passes_out = nullptr) {
  const uint32_t kJitF = static_cast<uint32_t>(js.F);
  const int min_blocks = js.min_blocks;
  DnPlan dn;
  if (js.arith == 1) {
    dn = dn_plan(fns, H, L, js.F, js.classes);
  } else {
    for (uint32_t f = 0; f < H; ++f) dn.fq.push_back(f);
  }
  std::vector<PassFns> passes;
  for (const DnPass& dp : dn.passes) {
    PassFns pf;
    for (const DnFn& f : dp.fns) pf.fn.push_back(f.fn);
    pf.dn = &dp;
    passes.push_back(std::move(pf));
  }
  for (size_t i = 0; i < dn.fq.size(); i += kJitF) {  // fq passes
    PassFns pf;
    for (size_t k = i; k < std::min(dn.fq.size(), i + kJitF); ++k) {
      pf.fn.push_back(dn.fq[k]);
      pf.fq.push_back(fn_const(fns[dn.fq[k]], L));
    }
    passes.push_back(std::move(pf));
  }
  if (passes_out) *passes_out = static_cast<uint32_t>(passes.size());
  const int UW = js.uw;                           // bytes per unit
  const int WU = 4 / UW;                          // units per 4-byte word
  const int R = (WU - 1 + static_cast<int>(L)) / WU;  // ring words above the current one
  std::ostringstream s;
  s << "typedef unsigned int u32; typedef unsigned long long u64; typedef unsigned char u8;\n"
       "typedef long long i64;\n"
       "#define L " << L << "\n#define H " << H << "\n"
       "#define NPASS " << passes.size() << "\n"
       "#define UW " << UW << "  // bytes per unit\n"
    << (UW == 2 ? "#define UNIT(i) ((u32)((const unsigned short*)bp)[i])\n"
                : "#define UNIT(i) ((u32)bp[i])\n")
    << ""
    << (js.gptr ? "#define LW(a) __ldg(a)  // text words through the read-only path (LDG)\n"
                : "#define LW(a) (*(a))\n")
    << "// arithmetic: " << dn.passes.size() << " dn passes, " << dn.fq.size()
    << " fq functions\n"
       "static __device__ __forceinline__ u32 umin(u32 a, u32 b) { return a < b ? a : b; }\n"
       "static __device__ __forceinline__ u32 smin(u32 a, u32 b) {\n"
       "  return (u32)min((int)a, (int)b);\n"
       "}\n"
       "static __device__ __forceinline__ u32 rol(u32 C, u32 ci, u32 co, float cf, u32 q,\n"
       "    u32 qln256, u32 negp256, float qp256, float qlnp, float c5) {\n"
       "  const float t1 = __fmaf_rn(cf, qlnp, c5);\n"
       "  const float R = __fmaf_rn(__uint2float_rn(C), qp256, t1);\n"
       "  const u32 kb = __float_as_uint(__fadd_rd(R, 8388607.5f));\n"
       "  u32 x = co * qln256 + ci;\n"
       "  x = C * q + x;\n"
       "  x = kb * negp256 + x;\n"
       "  return umin(x, x + negp256);\n"
       "}\n"
       "// dn: z = 0x80000000 + c is the float -c*2^-149 (see k1_jit.cpp)\n"
       "static __device__ __forceinline__ u32 rold(u32 z, u32 X, u32 co, float cf, u32 q,\n"
       "    u32 qln, u32 kp, u32 p, float A, float B, float M) {\n"
       "  const float t1 = __fmul_rn(cf, B);\n"
       "  const float R = __fmaf_rn(__uint_as_float(z), A, t1);\n"
       "  const u32 kb = __float_as_uint(__fadd_rd(R, M));\n"
       "  u32 x = co * qln + X;\n"
       "  x = z * q + x;\n"
       "  x = kb * kp + x;\n"
       "  return (u32)__viaddmin_s32((int)x, (int)p, (int)x);\n"
       "}\n"
       "// sring: the 128-byte line at g (aligned) into shared memory at s\n"
       "static __device__ __forceinline__ void fetch_line(u32 s, const void* g) {\n"
       "#pragma unroll\n"
       "  for (int i = 0; i < 8; ++i)\n"
       "    asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\" :: \"r\"(s + 16 * i),\n"
       "                 \"l\"((const char*)g + 16 * i) : \"memory\");\n"
       "}\n"
       "static __device__ __forceinline__ void ring_commit() {\n"
       "  asm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n"
       "}\n"
       "// all but the most recent group (the line fetched at the last line entry,\n"
       "// first read >= 1 iteration later)\n"
       "static __device__ __forceinline__ void ring_wait() {\n"
       "  asm volatile(\"cp.async.wait_group 1;\" ::: \"memory\");\n"
       "}\n"
       "extern \"C\" __global__ void __launch_bounds__(" << kJitThreads << ", " << min_blocks << ")\n"
       "k1j(const u8* __restrict__ text, const u64* __restrict__ offsets,\n"
       "    const u32* __restrict__ order, const u32* __restrict__ item_doc,\n"
       "    const u64* __restrict__ item_off, u32 n_items, u32 seg_len,\n"
       "    u32* __restrict__ sig, u64* __restrict__ counter, float c5,\n"
       "    u32* __restrict__ pass_flag, u32 epoch) {\n"
       "  const i64 KSEG = seg_len;  // windows per work item\n"
       "  // c5 = 2^-5 arrives as a parameter so that it sits in a register and\n"
       "  // every FFMA keeps its function constant as the immediate (fq)\n"
       "  const u32 lane = threadIdx.x & 31;\n"
    << (js.sring ? "  // sring: per lane a 2-line ring (256 B) of its text, indexed by address & 255\n"
                   "  __shared__ __align__(128) u32 sring_buf[" + std::to_string(kJitThreads * 64) + "];\n"
                   "  const u32* myr = sring_buf + threadIdx.x * 64;\n"
                   "  const u32 myr_s = (u32)__cvta_generic_to_shared(myr);\n"
                 : std::string())
    << ""
       "  // pass-major: every warp of the grid works on pass P until pass P's\n"
       "  // items are exhausted, so the SMs execute one pass's code at a time\n"
       "  // (the instruction cache holds one pass, not all of them)\n"
       "  for (u32 P = 0; P < NPASS; ++P) {\n"
       "  // the chunk gate (K1Gate): the next launch may start filling SMs\n"
       "  if (P == NPASS - 1 && lane == 0 && pass_flag) atomicMax(pass_flag, epoch);\n"
       "  u64 base = 0;\n"
       "  if (lane == 0) base = atomicAdd(counter + P, 32ull);\n"
       "  base = __shfl_sync(0xffffffffu, base, 0);\n"
       "  while (base < n_items) {\n"
       "    u32 nxt = 0;  // < 2^32 (n_items is u32): one register across the pass\n"
       "    if (lane == 0) nxt = (u32)atomicAdd(counter + P, 32ull);\n"
       "    const bool active = base + lane < n_items;\n"
       "    const u32 item = active ? order[base + lane] : 0u;\n"
       "    u64 doc = item; i64 ws = 0; bool multi = false;\n"
       "    if (item_doc && active) {\n"
       "      doc = item_doc[item];\n"
       "      const u64 s0 = item_off[doc];\n"
       "      ws = (i64)(item - s0) * KSEG;\n"
       "      multi = item_off[doc + 1] - s0 > 1;\n"
       "    }\n"
       "    const u64 off = offsets[doc];\n"
       "    const i64 len = active ? (i64)(offsets[doc + 1] - off) : 0;\n"
       "    const i64 nwin = len - L + 1;\n"
       "    const i64 we = active ? (ws + KSEG < nwin ? ws + KSEG : nwin) : 0;\n"
       "    const i64 wlo = active ? ws : 0;\n"
       "    const i64 e = active ? we + L - 1 : 0;\n"
       "    const u8* bp = text + off * UW;\n"
       "    const u64 abase = (u64)bp;\n"
       "    u32* row = sig + doc * H;\n"
       "    switch (P) {\n";
  for (size_t pass = 0; pass < passes.size(); ++pass) {
    const PassFns& pf = passes[pass];
    const bool isdn = pf.dn != nullptr;
    const int n = static_cast<int>(pf.fn.size());
    const int ncls = isdn ? static_cast<int>(pf.dn->w.size()) : 0;
    s << "    case " << pass << ": { // functions";
    for (int f = 0; f < n; ++f) s << " " << pf.fn[f];
    s << "\n";
    if (isdn) {
      s << "      const u32 GG = " << hex(pf.dn->g << 8) << ";  // float c_out offset 256g\n";
      for (int c = 0; c < ncls; ++c) s << "      const u32 W" << c << " = " << hex(pf.dn->w[c]) << ";\n";
      for (int f = 0; f < n; ++f)
        s << "      u32 s" << f << " = 0x80000000u, m" << f << " = 0x7fffffffu;\n";
    } else {
      for (int f = 0; f < n; ++f) s << "      u32 s" << f << " = 0u, m" << f << " = 0xffffffffu;\n";
    }
    auto call = [&](const std::string& st, int i, int f) {
      return isdn ? rold_call(st, i, pf.dn->fns[f]) : rol_call(st, i, pf.fq[f]);
    };
    const char* mn = isdn ? "smin" : "umin";
    // one single-step loop, run twice: phase 0 = warm-up (no min) + steps to
    // a 4-byte-aligned word boundary; phase 1 = the tail below the words
    s << "      i64 p = e - 1;\n"
         "      for (int phase = 0; phase < 2; ++phase) {\n"
         "        while (p >= wlo && (phase == 1 || p > e - L || ((abase + (u64)(p + 1) * UW) & 3))) {\n";
    if (isdn) {
      s << "          const u32 ci0 = UNIT(p);\n";
      for (int c = 0; c < ncls; ++c) s << "          const u32 x" << c << "_0 = ci0 | W" << c << ";\n";
      s << "          const u32 co0 = (p + L < e) ? UNIT(p + L) : 0u;\n"
           "          const float cf0 = __uint2float_rn(co0 + GG);\n";
    } else {
      s << "          const u32 ci0 = UNIT(p) << 8;\n"
           "          const u32 co0 = (p + L < e) ? UNIT(p + L) : 0u;\n"
           "          const float cf0 = __uint2float_rn(co0);\n";
    }
    s << "          const bool cnt = p <= e - L;\n";
    for (int f = 0; f < n; ++f) {
      s << "          s" << f << " = " << call("s" + std::to_string(f), 0, f) << ";\n"
        << "          if (cnt) m" << f << " = " << mn << "(m" << f << ", s" << f << ");\n";
    }
    s << "          --p;\n"
         "        }\n"
         "        if (phase == 1) break;\n";
    // whole aligned words
    s << "        if (p - " << (js.unroll == 2 ? 2 * WU - 1 : WU - 1) << " >= wlo) {\n"
      << "          const u32* wp = (const u32*)(abase + (u64)(p - " << WU - 1 << ") * UW);\n"
      << "          i64 q = p - " << WU - 1 << ";\n"
         "          u32 cur = LW(wp);\n";
    for (int k = 1; k <= R; ++k) {
      // the ring holds words q+4 .. q+4R (each shifts up one slot per word,
      // so every slot is loaded, not only those the first word reads); bytes
      // at positions >= e read as 0 (the first word's c_out can be position
      // e), and a word with no position below e is not loaded at all
      s << "          u32 r" << k << " = 0u;\n"
        << "          { const i64 nv = e - (q + " << WU * k << ");\n"
        << "            if (nv > 0) r" << k << " = LW(wp + " << k
        << ") & (nv >= " << WU << " ? 0xffffffffu : ((1u << (8 * UW * (u32)nv)) - 1u)); }\n";
    }
    if (js.sring && js.unroll == 1)
      s << "          { // prime: the current word's line and the one below, then an empty\n"
           "            // group so that the first ring_wait() waits for them\n"
           "            const u64 lb = ((u64)wp) & ~127ull;\n"
           "            fetch_line(myr_s + ((u32)lb & 255u), (const void*)lb);\n"
           "            if (lb > abase + (u64)wlo) fetch_line(myr_s + ((u32)(lb - 128) & 255u), (const void*)(lb - 128));\n"
           "            ring_commit(); ring_commit(); }\n";
    // one word: 4 windows of every function of the pass, then the ring
    // shifts down one word and `next` becomes the current word
    auto word = [&](const std::string& next) {
      for (int i = WU - 1; i >= 0; --i) {
        const int pos = i + static_cast<int>(L), k = pos / WU, j = pos % WU;
        const std::string src = k == 0 ? "cur" : "r" + std::to_string(k);
        char sel_in[8], sel_out[8], sel_x[8], sel_f[8];
        if (UW == 2) {  // half-words: c_in << 8 from bytes 2i, 2i+1; c_out from 2j, 2j+1
          std::snprintf(sel_in, sizeof sel_in, "0x4%d%d4", 2 * i + 1, 2 * i);
          std::snprintf(sel_out, sizeof sel_out, "0x44%d%d", 2 * j + 1, 2 * j);
        } else {
          std::snprintf(sel_in, sizeof sel_in, "0x44%d4", i);
          std::snprintf(sel_out, sizeof sel_out, "0x444%d", j);
        }
        std::snprintf(sel_x, sizeof sel_x, "0x765%d", i);  // c_in + (w & ~0xff)
        std::snprintf(sel_f, sizeof sel_f, "0x445%d", j);  // c_out + 256g
        s << "            {";
        if (isdn) {
          for (int c = 0; c < ncls; ++c)
            s << " const u32 x" << c << "_" << i << " = __byte_perm(cur, W" << c << ", " << sel_x
              << ");\n";
          s << "            const u32 co" << i << " = __byte_perm(" << src << ", 0u, " << sel_out
            << ");\n"
            << "            const float cf" << i << " = __uint2float_rn(__byte_perm(" << src
            << ", GG, " << sel_f << "));\n";
        } else {
          s << " const u32 ci" << i << " = __byte_perm(cur, 0u, " << sel_in << ");\n"
            << "            const u32 co" << i << " = __byte_perm(" << src << ", 0u, " << sel_out
            << ");\n"
            << "            const float cf" << i << " = __uint2float_rn(co" << i << ");\n";
        }
      }
      const char* mn3 = isdn ? "(u32)__vimin3_s32((int)" : "__vimin3_u32(";
      const char* cst = isdn ? "(int)" : "";
      for (int f = 0; f < n; ++f) {
        const std::string sf = "s" + std::to_string(f), mf = "m" + std::to_string(f);
        if (WU == 4) {
          s << "            { const u32 a3 = " << call(sf, 3, f) << ";\n"
            << "              const u32 a2 = " << call("a3", 2, f) << ";\n"
            << "              const u32 a1 = " << call("a2", 1, f) << ";\n"
            << "              const u32 a0 = " << call("a1", 0, f) << ";\n"
            << "              " << sf << " = a0; " << mf << " = " << mn3 << mf << ", " << cst
            << "a3, " << cst << "a2); " << mf << " = " << mn3 << mf << ", " << cst << "a1, " << cst
            << "a0); }\n";
        } else {  // two windows per word
          s << "            { const u32 a1 = " << call(sf, 1, f) << ";\n"
            << "              const u32 a0 = " << call("a1", 0, f) << ";\n"
            << "              " << sf << " = a0; " << mf << " = " << mn3 << mf << ", " << cst
            << "a1, " << cst << "a0); }\n";
        }
      }
      s << "            " << std::string(WU, '}') << "\n";
      for (int k = R; k >= 2; --k) s << "            r" << k << " = r" << k - 1 << ";\n";
      if (R >= 1) s << "            r1 = cur;\n";
      s << "            cur = " << next << ";\n";
    };
    if (js.unroll == 2) {
      // pairs of words while two remain (a 32-bit pair count); an odd last
      // word goes to the single steps below
      s << "          u32 npair = (u32)((q - wlo + 4) >> 3);\n"
           "          do {\n"
           "            const u32 nx = LW(wp - 1);\n";
      word("nx");
      s << "            const u32 nx2 = (q - 8 >= wlo) ? LW(wp - 2) : 0u;\n";
      word("nx2");
      s << "            wp -= 2; q -= 8;\n"
           "          } while (--npair);\n"
           "          p = q + 3;\n"
           "        }\n"
           "      }\n";
    } else {
      const bool pf2 = js.prefetch >= 2 && !js.sring;
      if (pf2)
        s << "          u32 nx1 = (q - " << WU << " >= wlo) ? LW(wp - 1) : 0u;\n";
      s << "          for (;;) {\n"
           "            const bool more = q - " << WU << " >= wlo;\n";
      if (js.pfw > 0)
        s << "            if (q - " << WU * js.pfw << " >= wlo) asm volatile(\"prefetch.global."
          << (js.pfl2 ? "L2" : "L1") << " [%0];\" :: \"l\"(wp - " << js.pfw << "));\n";
      if (js.sring)
        s << "            ring_wait();\n"
             "            const u32 nx = myr[((u32)(u64)(wp - 1) & 255u) >> 2];\n";
      else if (pf2)
        s << "            const u32 nx = nx1;\n"
             "            nx1 = (q - " << 2 * WU << " >= wlo) ? LW(wp - 2) : 0u;\n";
      else
        s << "            const u32 nx = more ? LW(wp - 1) : 0u;\n";
      word("nx");
      s << "            --wp; q -= " << WU << ";\n"
           "            if (!more) break;\n";
      if (js.sring)
        s << "            if (((u32)(u64)wp & 127u) == 124u) {  // entered a new line: fetch the one below\n"
             "              const u64 lb = (((u64)wp) & ~127ull) - 128;\n"
             "              if (lb + 128 > abase + (u64)wlo) fetch_line(myr_s + ((u32)lb & 255u), (const void*)lb);\n"
             "            }\n"
             "            ring_commit();\n";
      s << "          }\n"
           "          p = q + " << WU - 1 << ";\n"
           "        }\n"
           "      }\n";
    }
    // store the canonical minima (fq: state scaled by 256; dn: biased by 2^31)
    auto val = [&](int f) {
      return isdn ? "(m" + std::to_string(f) + " ^ 0x80000000u)" : "(m" + std::to_string(f) + " >> 8)";
    };
    s << "      if (active) {\n        if (multi) {\n";
    for (int f = 0; f < n; ++f) s << "          atomicMin(row + " << pf.fn[f] << ", " << val(f) << ");\n";
    s << "        } else {\n";
    for (int f = 0; f < n;) {
      const bool vec = f + 4 <= n && pf.fn[f] % 4 == 0 && pf.fn[f + 1] == pf.fn[f] + 1 &&
                       pf.fn[f + 2] == pf.fn[f] + 2 && pf.fn[f + 3] == pf.fn[f] + 3 && H % 4 == 0;
      if (vec) {
        s << "          *(uint4*)(row + " << pf.fn[f] << ") = make_uint4(" << val(f) << ", "
          << val(f + 1) << ", " << val(f + 2) << ", " << val(f + 3) << ");\n";
        f += 4;
      } else {
        s << "          row[" << pf.fn[f] << "] = " << val(f) << ";\n";
        ++f;
      }
    }
    s << "        }\n      }\n      break;\n    }\n";
  }
  s << "    }\n"
       "    base = __shfl_sync(0xffffffffu, nxt, 0);\n"
       "  }\n"
       "  }\n"
       "}\n";
  return s.str();
}


struct JitKernel {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
  int per_sm = 0;
  uint32_t passes = 0;
  double compile_seconds = 0;
  float c5 = 0.03125f;  // fq's quotient offset: 2^-5 for bytes, 2^-3 for 16-bit units
};

std::mutex g_jit_mu;
std::map<std::string, std::shared_ptr<JitKernel>> g_jit_cache;

std::shared_ptr<JitKernel> compile(const nd_hash_fn* fns, uint32_t H, uint32_t L,
                                   const JitShape& js) {
  const Nvrtc& nv = nvrtc();
  if (!nv.ok) fail(ND_ERR_DEVICE, "K1j: " + nv.error);
  uint32_t passes = 0;
  const std::string src = generate(fns, H, L, js, &passes);
  auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "k1j.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    fail(ND_ERR_DEVICE, "K1j: nvrtcCreateProgram failed");
  // denormals must survive: the dn state is a denormal float (no FTZ)
  const char* opts[] = {"--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17", "--ftz=false"};
  const nvrtcResult rc = nv.compile(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    nv.log(prog, log.data());
    nv.destroy(&prog);
    fail(ND_ERR_DEVICE, "K1j: NVRTC compile failed: " + log.substr(0, 2000));
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  std::vector<char> cubin(n);
  nv.cubin(prog, cubin.data());
  nv.destroy(&prog);
  auto k = std::make_shared<JitKernel>();
  ND_CUDA(cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
  ND_CUDA(cudaLibraryGetKernel(&k->fn, k->lib, "k1j"));
  ND_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &k->per_sm, reinterpret_cast<const void*>(k->fn), kJitThreads, 0));
  k->per_sm = std::max(k->per_sm, 1);
  k->passes = passes;
  k->c5 = js.uw == 2 ? 0.125f : 0.03125f;
  k->compile_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return k;
}

}  // namespace

bool k1_jit_eligible(const DevFamily& fam) {
  const char* v = getenv("ND_K1_JIT");  // 0: the register-constant K1
  if (v && v[0] == '0') return false;
  // codepoint families compile too when narrow documents can use them
  return (fam.unit == 0 || fam.narrow_ok) && !fam.exact && fam.L >= 1 && fam.L <= 16 &&
         fam.H >= 1 && fam.H <= 1024;
}

// Compiles (or finds) the family's kernel; the cache outlives contexts so a
// family is compiled once per process.
// uw = 2: text of 16-bit units (code points < 2^16), the fq arithmetic with
// c5 = 2^-3 (the error bound of DESIGN §3 with c_in, c_out < 2^16)
JitShape unit_shape(JitShape js, int uw) {
  if (uw == 2) {
    js.uw = 2;
    js.arith = 0;
    // 32 functions per pass, 4 CTAs, the word after next prefetched: two
    // windows per word leave more per-word overhead to amortise (BMP text,
    // 500k docs, whole call: F=16/6 CTAs 23.02 ms, F=20/5 22.68, F=24/5
    // 22.77, F=32/4 22.65, F=32/4 + prefetch 2 22.34; profiles/r2_codepoint.txt)
    js.F = 32;
    js.min_blocks = 4;
    js.prefetch = 2;
    js.unroll = 1;
    js.sring = 0;
    js.pfw = 0;
    if (const char* v = getenv("ND_K1J16_F")) js.F = std::max(4, std::min(64, atoi(v)));  // tuning
    if (const char* v = getenv("ND_K1J16_MINB")) js.min_blocks = std::max(1, std::min(16, atoi(v)));
    if (const char* v = getenv("ND_K1J16_PREFETCH")) js.prefetch = std::max(1, std::min(2, atoi(v)));
  }
  return js;
}

void* k1_jit_prepare(const nd_hash_fn* fns, uint32_t H, uint32_t L, int uw) {
  std::string key(reinterpret_cast<const char*>(fns), sizeof(nd_hash_fn) * H);
  const JitShape js = unit_shape(jit_shape(), uw);
  key += "|" + std::to_string(H) + "|" + std::to_string(L) + "|" + std::to_string(js.F) + "|" +
         std::to_string(js.min_blocks) + "|" + std::to_string(js.prefetch) + "|" +
         std::to_string(js.unroll) + "|" + std::to_string(js.arith) + "|" +
         std::to_string(js.classes) + "|" + std::to_string(js.gptr) + "|" +
         std::to_string(js.pfw) + "|" + std::to_string(js.pfl2) + "|" + std::to_string(js.sring) +
         "|u" + std::to_string(js.uw);
  int dev = 0;
  cudaGetDevice(&dev);
  key += "|" + std::to_string(dev);
  std::lock_guard<std::mutex> g(g_jit_mu);
  auto it = g_jit_cache.find(key);
  if (it != g_jit_cache.end()) return it->second.get();
  auto k = compile(fns, H, L, js);
  g_jit_cache[key] = k;
  return k.get();
}

uint32_t k1_jit_passes(const void* handle) {
  return static_cast<const JitKernel*>(handle)->passes;
}

double k1_jit_compile_seconds(const void* handle) {
  return handle ? static_cast<const JitKernel*>(handle)->compile_seconds : 0.0;
}

uint64_t k1_jit_resident_warps(const void* handle) {
  return static_cast<uint64_t>(static_cast<const JitKernel*>(handle)->per_sm) * sm_count() *
         (kJitThreads / 32);
}

void k1_jit_launch(const void* handle, const uint8_t* d_text, const uint64_t* d_offsets,
                   const uint32_t* order, const uint32_t* item_doc, const uint64_t* item_off,
                   uint32_t n_items, uint32_t seg_len, uint32_t* d_sig,
                   unsigned long long* counter, cudaStream_t s, const K1Gate* gate) {
  const JitKernel* k = static_cast<const JitKernel*>(handle);
  const uint64_t warps = (static_cast<uint64_t>(n_items) + 31) / 32;
  uint64_t blocks = (warps + kJitThreads / 32 - 1) / (kJitThreads / 32);
  blocks = std::min<uint64_t>(blocks, static_cast<uint64_t>(k->per_sm) * sm_count());
  ND_CUDA(cudaMemsetAsync(counter, 0, k->passes * sizeof(unsigned long long), s));  // one per pass
  float c5 = k->c5;
  unsigned int* pass_flag = gate ? gate->flag : nullptr;
  unsigned int epoch = gate ? gate->epoch : 0u;
  void* args[] = {&d_text, &d_offsets, &order, &item_doc, &item_off, &n_items, &seg_len, &d_sig,
                  &counter, &c5, &pass_flag, &epoch};
  ND_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(k->fn), dim3(static_cast<unsigned>(blocks)),
                           dim3(kJitThreads), args, 0, s));
  ND_CHECK_LAUNCH();
}

std::string k1_jit_source(const nd_hash_fn* fns, uint32_t H, uint32_t L, int uw) {
  return generate(fns, H, L, unit_shape(jit_shape(), uw));
}

}  // namespace ndb

extern "C" int64_t nd_k1j_source_units(const nd_hash_fn* fns, uint32_t H, uint32_t L,
                                       uint32_t unit_bytes, char* out, uint64_t cap) {
  if (!fns || H == 0 || H > 1024 || L == 0 || L > 16 || (unit_bytes != 1 && unit_bytes != 2))
    return -1;
  for (uint32_t i = 0; i < H; ++i)  // the fq domain (derive_family's)
    if (fns[i].modulus < (1u << 21) || fns[i].modulus >= (1u << 23) || fns[i].base == 0 ||
        fns[i].base >= (1u << 16))
      return -1;
  const std::string s = ndb::k1_jit_source(fns, H, L, static_cast<int>(unit_bytes));
  if (out && cap) {
    const uint64_t n = std::min<uint64_t>(cap - 1, s.size());
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
  return static_cast<int64_t>(s.size());
}

extern "C" int64_t nd_k1j_source(const nd_hash_fn* fns, uint32_t H, uint32_t L, char* out,
                                 uint64_t cap) {
  return nd_k1j_source_units(fns, H, L, 1, out, cap);
}

extern "C" int64_t nd_k1j_plan(const nd_hash_fn* fns, uint32_t H, uint32_t L, uint32_t* out,
                               uint64_t cap_rows) {
  if (!fns || H == 0 || H > 1024 || L == 0 || L > 16) return -1;
  for (uint32_t i = 0; i < H; ++i)  // the fq domain (derive_family's)
    if (fns[i].modulus < (1u << 21) || fns[i].modulus >= (1u << 23) || fns[i].base == 0 ||
        fns[i].base >= (1u << 16))
      return -1;
  const ndb::JitShape js = ndb::jit_shape();
  if (js.arith != 1) return -1;
  const ndb::DnPlan plan = ndb::dn_plan(fns, H, L, js.F, js.classes);
  uint64_t row = 0;
  auto put = [&](const uint32_t* v) {
    if (out && row < cap_rows) std::memcpy(out + 12 * row, v, 12 * sizeof(uint32_t));
    ++row;
  };
  for (size_t P = 0; P < plan.passes.size(); ++P)
    for (const ndb::DnFn& f : plan.passes[P].fns) {
      const ndb::DnPass& dp = plan.passes[P];
      const uint32_t v[12] = {static_cast<uint32_t>(P), f.cls, dp.g, dp.w[f.cls], f.fn,
                              f.q, f.qln, f.kp, f.p, f.a_bits, f.b_bits, f.m_bits};
      put(v);
    }
  const uint32_t F = static_cast<uint32_t>(js.F);
  for (size_t i = 0; i < plan.fq.size(); ++i) {  // fq passes: g = 0
    const uint32_t v[12] = {static_cast<uint32_t>(plan.passes.size() + i / F), 0, 0, 0,
                            plan.fq[i], fns[plan.fq[i]].base, 0, 0, fns[plan.fq[i]].modulus, 0, 0, 0};
    put(v);
  }
  return static_cast<int64_t>(row);
}
