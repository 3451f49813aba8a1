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
// (C2 shard, H=128: F=16 / 6 blocks 66.9 ms, F=32 / 4 blocks 67.6 ms,
// F=24 / 5 blocks 67.7 ms, F=32 / 5 blocks 74.4 ms (spills), F=16 / 8 blocks
// 73.4 ms; a second prefetched word changes nothing -- profiles/r2_k1j_variants.txt)
struct JitShape {
  int F = 16;
  int min_blocks = 6;
  int prefetch = 1;
  int unroll = 1;  // whole words per loop iteration (2: ND_K1J_UNROLL=2, slower)
};

JitShape jit_shape() {
  JitShape j;
  if (const char* v = getenv("ND_K1J_F")) j.F = std::max(4, std::min(64, atoi(v)));
  if (const char* v = getenv("ND_K1J_MINB")) j.min_blocks = std::max(1, std::min(16, atoi(v)));
  if (const char* v = getenv("ND_K1J_PREFETCH")) j.prefetch = std::max(1, std::min(2, atoi(v)));
  if (const char* v = getenv("ND_K1J_UNROLL")) j.unroll = std::max(1, std::min(2, atoi(v)));
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

std::string generate(const nd_hash_fn* fns, uint32_t H, uint32_t L, const JitShape& js) {
  const uint32_t kJitF = static_cast<uint32_t>(js.F);
  const int min_blocks = js.min_blocks;
  std::vector<FnConst> cs(H);
  for (uint32_t f = 0; f < H; ++f) cs[f] = fn_const(fns[f], L);
  const int R = (3 + static_cast<int>(L)) >> 2;  // ring words above the current one
  std::ostringstream s;
  s << "typedef unsigned int u32; typedef unsigned long long u64; typedef unsigned char u8;\n"
       "typedef long long i64;\n"
       "#define L " << L << "\n#define H " << H << "\n"
       "#define NPASS " << (H + kJitF - 1) / kJitF << "\n"
       "static __device__ __forceinline__ u32 umin(u32 a, u32 b) { return a < b ? a : b; }\n"
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
       "extern \"C\" __global__ void __launch_bounds__(" << kJitThreads << ", " << min_blocks << ")\n"
       "k1j(const u8* __restrict__ text, const u64* __restrict__ offsets,\n"
       "    const u32* __restrict__ order, const u32* __restrict__ item_doc,\n"
       "    const u64* __restrict__ item_off, u32 n_items, u32 seg_len,\n"
       "    u32* __restrict__ sig, u64* __restrict__ counter, float c5,\n"
       "    u32* __restrict__ pass_flag, u32 epoch) {\n"
       "  const i64 KSEG = seg_len;  // windows per work item\n"
       "  // c5 = 2^-5 arrives as a parameter so that it sits in a register and\n"
       "  // every FFMA keeps its function constant as the immediate\n"
       "  const u32 lane = threadIdx.x & 31;\n"
       "  // pass-major: every warp of the grid works on pass P (functions\n"
       "  // P*F .. P*F+F-1) until pass P's items are exhausted, so the SMs\n"
       "  // execute one pass's code at a time (the instruction cache holds one\n"
       "  // pass, not all of them)\n"
       "  for (u32 P = 0; P < NPASS; ++P) {\n"
       "  // the chunk gate (K1Gate): the next launch may start filling SMs\n"
       "  if (P == NPASS - 1 && lane == 0 && pass_flag) atomicMax(pass_flag, epoch);\n"
       "  u64 base = 0;\n"
       "  if (lane == 0) base = atomicAdd(counter + P, 32ull);\n"
       "  base = __shfl_sync(0xffffffffu, base, 0);\n"
       "  while (base < n_items) {\n"
       "    u64 nxt = 0;\n"
       "    if (lane == 0) nxt = atomicAdd(counter + P, 32ull);\n"
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
       "    const u8* bp = text + off;\n"
       "    const u64 abase = (u64)bp;\n"
       "    u32* row = sig + doc * H;\n"
       "    switch (P) {\n";
  int pass = 0;
  for (uint32_t fb = 0; fb < H; fb += kJitF, ++pass) {
    const int n = static_cast<int>(std::min<uint32_t>(kJitF, H - fb));
    s << "    case " << pass << ": { // functions " << fb << " .. " << fb + n - 1 << "\n";
    for (int f = 0; f < n; ++f) s << "      u32 s" << f << " = 0u, m" << f << " = 0xffffffffu;\n";
    // one single-step loop, run twice: phase 0 = warm-up (no min) + steps to
    // a 4-byte-aligned word boundary; phase 1 = the tail below the words
    s << "      i64 p = e - 1;\n"
         "      for (int phase = 0; phase < 2; ++phase) {\n"
         "        while (p >= wlo && (phase == 1 || p > e - L || ((abase + (u64)p + 1) & 3))) {\n"
         "          const u32 ci0 = ((u32)bp[p]) << 8;\n"
         "          const u32 co0 = (p + L < e) ? (u32)bp[p + L] : 0u;\n"
         "          const float cf0 = __uint2float_rn(co0);\n"
         "          const bool cnt = p <= e - L;\n";
    for (int f = 0; f < n; ++f) {
      s << "          s" << f << " = " << rol_call("s" + std::to_string(f), 0, cs[fb + f]) << ";\n"
        << "          if (cnt) m" << f << " = umin(m" << f << ", s" << f << ");\n";
    }
    s << "          --p;\n"
         "        }\n"
         "        if (phase == 1) break;\n";
    // whole aligned words
    s << "        if (p - " << (js.unroll == 2 ? 7 : 3) << " >= wlo) {\n"
         "          const u32* wp = (const u32*)(abase + (u64)(p - 3));\n"
         "          i64 q = p - 3;\n"
         "          u32 cur = wp[0];\n";
    for (int k = 1; k <= R; ++k) {
      // the ring holds words q+4 .. q+4R (each shifts up one slot per word,
      // so every slot is loaded, not only those the first word reads); bytes
      // at positions >= e read as 0 (the first word's c_out can be position
      // e), and a word with no position below e is not loaded at all
      s << "          u32 r" << k << " = 0u;\n"
        << "          { const i64 nv = e - (q + " << 4 * k << ");\n"
        << "            if (nv > 0) r" << k << " = wp[" << k
        << "] & (nv >= 4 ? 0xffffffffu : ((1u << (8 * (u32)nv)) - 1u)); }\n";
    }
    // one word: 4 windows of every function of the pass, then the ring
    // shifts down one word and `next` becomes the current word
    auto word = [&](const std::string& next) {
      for (int i = 3; i >= 0; --i) {
        const int pos = i + static_cast<int>(L), k = pos >> 2, j = pos & 3;
        const std::string src = k == 0 ? "cur" : "r" + std::to_string(k);
        char sel_in[8], sel_out[8];
        std::snprintf(sel_in, sizeof sel_in, "0x44%d4", i);
        std::snprintf(sel_out, sizeof sel_out, "0x444%d", j);
        s << "            { const u32 ci" << i << " = __byte_perm(cur, 0u, " << sel_in << ");\n"
          << "            const u32 co" << i << " = __byte_perm(" << src << ", 0u, " << sel_out
          << ");\n"
          << "            const float cf" << i << " = __uint2float_rn(co" << i << ");\n";
      }
      for (int f = 0; f < n; ++f) {
        const std::string sf = "s" + std::to_string(f), mf = "m" + std::to_string(f);
        s << "            { const u32 a3 = " << rol_call(sf, 3, cs[fb + f]) << ";\n"
          << "              const u32 a2 = " << rol_call("a3", 2, cs[fb + f]) << ";\n"
          << "              const u32 a1 = " << rol_call("a2", 1, cs[fb + f]) << ";\n"
          << "              const u32 a0 = " << rol_call("a1", 0, cs[fb + f]) << ";\n"
          << "              " << sf << " = a0; " << mf << " = __vimin3_u32(" << mf << ", a3, a2); "
          << mf << " = __vimin3_u32(" << mf << ", a1, a0); }\n";
      }
      s << "            }}}}\n";
      for (int k = R; k >= 2; --k) s << "            r" << k << " = r" << k - 1 << ";\n";
      if (R >= 1) s << "            r1 = cur;\n";
      s << "            cur = " << next << ";\n";
    };
    if (js.unroll == 2) {
      // pairs of words while two remain (a 32-bit pair count); an odd last
      // word goes to the single steps below
      s << "          u32 npair = (u32)((q - wlo + 4) >> 3);\n"
           "          do {\n"
           "            const u32 nx = wp[-1];\n";
      word("nx");
      s << "            const u32 nx2 = (q - 8 >= wlo) ? wp[-2] : 0u;\n";
      word("nx2");
      s << "            wp -= 2; q -= 8;\n"
           "          } while (--npair);\n"
           "          p = q + 3;\n"
           "        }\n"
           "      }\n";
    } else {
      if (js.prefetch >= 2)
        s << "          u32 nx1 = (q - 4 >= wlo) ? wp[-1] : 0u;\n";
      s << "          for (;;) {\n"
           "            const bool more = q - 4 >= wlo;\n";
      if (js.prefetch >= 2)
        s << "            const u32 nx = nx1;\n"
             "            nx1 = (q - 8 >= wlo) ? wp[-2] : 0u;\n";
      else
        s << "            const u32 nx = more ? wp[-1] : 0u;\n";
      word("nx");
      s << "            --wp; q -= 4;\n"
           "            if (!more) break;\n"
           "          }\n"
           "          p = q + 3;\n"
           "        }\n"
           "      }\n";
    }
    // store the canonical minima (state scaled by 256)
    s << "      if (active) {\n        if (multi) {\n";
    for (int f = 0; f < n; ++f)
      s << "          atomicMin(row + " << fb + f << ", m" << f << " >> 8);\n";
    s << "        } else {\n";
    if (H % 4 == 0 && n % 4 == 0) {
      for (int f = 0; f < n; f += 4)
        s << "          *(uint4*)(row + " << fb + f << ") = make_uint4(m" << f << " >> 8, m" << f + 1
          << " >> 8, m" << f + 2 << " >> 8, m" << f + 3 << " >> 8);\n";
    } else {
      for (int f = 0; f < n; ++f) s << "          row[" << fb + f << "] = m" << f << " >> 8;\n";
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
};

std::mutex g_jit_mu;
std::map<std::string, std::shared_ptr<JitKernel>> g_jit_cache;

std::shared_ptr<JitKernel> compile(const nd_hash_fn* fns, uint32_t H, uint32_t L,
                                   const JitShape& js) {
  const Nvrtc& nv = nvrtc();
  if (!nv.ok) fail(ND_ERR_DEVICE, "K1j: " + nv.error);
  const std::string src = generate(fns, H, L, js);
  auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  if (nv.create(&prog, src.c_str(), "k1j.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    fail(ND_ERR_DEVICE, "K1j: nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17"};
  const nvrtcResult rc = nv.compile(prog, 3, opts);
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
  k->passes = (H + js.F - 1) / js.F;
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
void* k1_jit_prepare(const nd_hash_fn* fns, uint32_t H, uint32_t L) {
  std::string key(reinterpret_cast<const char*>(fns), sizeof(nd_hash_fn) * H);
  const JitShape js = jit_shape();
  key += "|" + std::to_string(H) + "|" + std::to_string(L) + "|" + std::to_string(js.F) + "|" +
         std::to_string(js.min_blocks) + "|" + std::to_string(js.prefetch) + "|" +
         std::to_string(js.unroll);
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
  float c5 = 0.03125f;
  unsigned int* pass_flag = gate ? gate->flag : nullptr;
  unsigned int epoch = gate ? gate->epoch : 0u;
  void* args[] = {&d_text, &d_offsets, &order, &item_doc, &item_off, &n_items, &seg_len, &d_sig,
                  &counter, &c5, &pass_flag, &epoch};
  ND_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(k->fn), dim3(static_cast<unsigned>(blocks)),
                           dim3(kJitThreads), args, 0, s));
  ND_CHECK_LAUNCH();
}

std::string k1_jit_source(const nd_hash_fn* fns, uint32_t H, uint32_t L) {
  return generate(fns, H, L, jit_shape());
}

}  // namespace ndb

extern "C" int64_t nd_k1j_source(const nd_hash_fn* fns, uint32_t H, uint32_t L, char* out,
                                 uint64_t cap) {
  if (!fns || H == 0 || H > 1024 || L == 0 || L > 16) return -1;
  for (uint32_t i = 0; i < H; ++i)  // the fq domain (derive_family's)
    if (fns[i].modulus < (1u << 21) || fns[i].modulus >= (1u << 23) || fns[i].base == 0 ||
        fns[i].base >= (1u << 16))
      return -1;
  const std::string s = ndb::k1_jit_source(fns, H, L);
  if (out && cap) {
    const uint64_t n = std::min<uint64_t>(cap - 1, s.size());
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
  return static_cast<int64_t>(s.size());
}
