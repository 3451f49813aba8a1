// Synthetic planted-duplicate corpora in the reference generator's shape
// (synthetic.cpp:39-110): 37-character alphabet (synthetic.cpp:15), group
// members = base text + substitution edits (synthetic.cpp:25-35), members and
// singletons scattered over output positions (synthetic.cpp:81-88).
//
// mode 0: generate_synthetic bit for bit (one mt19937_64 stream, single
//         thread) -- used for the C1 parity corpus.
// mode 1: streaming, multi-threaded variant for corpora of 10^6..10^7+ docs:
//         each document draws from its own counter-based stream, positions
//         come from a Feistel bijection, so the output is a pure function of
//         the spec (independent of the thread count).  Lengths follow a
//         uniform or clipped lognormal law (C3/C5 shapes).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "nd_internal.cuh"

#define ND_HD __host__ __device__

namespace ndb {
namespace {

constexpr char kAlphabet[] = "abcdefghijklmnopqrstuvwxyz0123456789 ";
__device__ __constant__ char kAlphaDev[] = "abcdefghijklmnopqrstuvwxyz0123456789 ";
constexpr uint64_t kAlpha = 37;
#ifdef __CUDA_ARCH__
#define kAlphaChars kAlphaDev
#else
#define kAlphaChars kAlphabet
#endif

uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

void validate(const nd_synth_spec& s) {
  if (s.group_size_min < 2 || s.group_size_max < s.group_size_min)
    fail(ND_ERR_CONFIG, "group sizes must satisfy 2 <= min <= max");
  if (s.len_min < 1 || s.len_max < s.len_min)
    fail(ND_ERR_CONFIG, "base length range is empty");
  if (s.edit_den == 0 || s.edit_num > s.edit_den) fail(ND_ERR_CONFIG, "edit rate must be in [0, 1]");
}

// ---------------------------------------------------------------- mode 0
struct Mode0Cache {
  std::mutex mu;
  std::vector<uint8_t> key;
  std::vector<std::string> texts;
} g_cache;

std::string random_text(std::mt19937_64& rng, uint32_t lo, uint32_t hi) {
  uint64_t len = lo + bounded_random(rng, static_cast<uint64_t>(hi) - lo + 1);
  std::string t(len, ' ');
  for (auto& c : t) c = kAlphabet[bounded_random(rng, kAlpha)];
  return t;
}

std::string perturb(const std::string& base, uint64_t num, uint64_t den, std::mt19937_64& rng) {
  std::string t = base;
  if (num == 0) return t;
  for (auto& c : t) {
    if (bounded_random(rng, den) >= num) continue;
    char r = kAlphabet[bounded_random(rng, kAlpha)];
    while (r == c) r = kAlphabet[bounded_random(rng, kAlpha)];
    c = r;
  }
  return t;
}

std::vector<std::string> generate_mode0(const nd_synth_spec& s) {
  uint64_t g = gcd_u64(s.edit_num, s.edit_den);
  uint64_t num = s.edit_num / g, den = s.edit_den / g;  // Ratio reduces (util.cpp:19-27)
  if (num == 0) den = 1;
  std::mt19937_64 rng(s.seed);
  std::vector<uint32_t> sizes(s.group_count);
  uint64_t grouped = 0;
  for (auto& sz : sizes) {
    sz = s.group_size_min + static_cast<uint32_t>(bounded_random(
                                rng, static_cast<uint64_t>(s.group_size_max) - s.group_size_min + 1));
    grouped += sz;
  }
  if (grouped > s.doc_count) fail(ND_ERR_CONFIG, "doc count cannot hold the grouped documents");
  std::vector<std::string> texts;
  texts.reserve(s.doc_count);
  for (size_t gi = 0; gi < sizes.size(); ++gi) {
    std::string base = random_text(rng, s.len_min, s.len_max);
    for (uint32_t m = 0; m < sizes[gi]; ++m) texts.push_back(m == 0 ? base : perturb(base, num, den, rng));
  }
  while (texts.size() < s.doc_count) texts.push_back(random_text(rng, s.len_min, s.len_max));
  std::vector<uint64_t> pos(texts.size());
  std::iota(pos.begin(), pos.end(), 0);
  for (uint64_t i = pos.size(); i > 1; --i) std::swap(pos[i - 1], pos[bounded_random(rng, i)]);
  std::vector<std::string> placed(texts.size());
  for (uint64_t i = 0; i < texts.size(); ++i) placed[pos[i]] = std::move(texts[i]);
  return placed;
}

// ---------------------------------------------------------------- mode 1
// Counter-based and random-access: draw(key, i) = mix64(mix64(key) + i*C), so
// any character of any document can be produced independently -- on the host
// (threads) or on the device (k_synth_text, one warp per document), with
// identical bytes.  Lengths (which use libm for the lognormal law) are always
// computed on the host.
ND_HD inline uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
ND_HD inline uint64_t draw(uint64_t mixed_key, uint64_t i) {
  return mix64(mixed_key + i * 0xD1B54A32D192ED03ull);
}

struct Stream {  // sequential view of the same counter-based draws
  uint64_t key, ctr = 0;
  explicit Stream(uint64_t k) : key(mix64(k)) {}
  uint64_t next() { return draw(key, ctr++); }
  uint64_t below(uint64_t b) { return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * b) >> 64); }
  double unit() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
};

// POD view shared by host and device
struct M1 {
  uint64_t n, seed, grouped, ngroups, perm_key, half_mask;
  int half_bits;
  uint32_t edit_thresh;  // P(edit) * 2^32
  uint32_t len_draws;    // draws consumed by the length law (1 uniform, 2 lognormal)
};

ND_HD inline uint64_t perm_dec(const M1& m, uint64_t y) {
  uint64_t l = y >> m.half_bits, rr = y & m.half_mask;
  for (int r = 3; r >= 0; --r) {
    uint64_t t = rr ^ (mix64(l ^ (m.perm_key + 0x100000001B3ull * r)) & m.half_mask);
    rr = l;
    l = t;
  }
  return (l << m.half_bits) | rr;
}
ND_HD inline uint64_t perm_inv(const M1& m, uint64_t y) {  // Feistel + cycle walking
  do y = perm_dec(m, y);
  while (y >= m.n);
  return y;
}

// logical index -> (text stream key, edit stream key or 0)
ND_HD inline void m1_source(const M1& m, const uint64_t* group_first, uint64_t logical,
                            uint64_t& text_key, uint64_t& edit_key) {
  if (logical < m.grouped) {
    uint64_t lo = 0, hi = m.ngroups;  // last g with group_first[g] <= logical
    while (hi - lo > 1) {
      uint64_t mid = (lo + hi) / 2;
      if (group_first[mid] <= logical) lo = mid; else hi = mid;
    }
    const uint64_t g = lo, k = logical - group_first[g];
    text_key = m.seed * 0x632BE59BD9B4E019ull + 0x7777 + g;
    edit_key = k == 0 ? 0 : (m.seed * 0x8CB92BA72F3D8DD7ull + (g << 8) + k + 1);
  } else {
    text_key = m.seed * 0x632BE59BD9B4E019ull + 0x3333333333ull + logical;
    edit_key = 0;
  }
}

// character i of a document (text stream mixed key tkm, edit stream mixed keys
// ekm / ekm2 or 0)
ND_HD inline uint8_t m1_char(const M1& m, uint64_t tkm, uint64_t ekm, uint64_t ekm2, uint64_t i) {
  const uint64_t x = draw(tkm, m.len_draws + i / 2);
  const uint32_t h = static_cast<uint32_t>(x >> (32 * (i & 1)));
  uint32_t idx = static_cast<uint32_t>((static_cast<uint64_t>(h) * kAlpha) >> 32);
  if (ekm) {
    const uint32_t e = static_cast<uint32_t>(draw(ekm, i / 2) >> (32 * (i & 1)));
    if (e < m.edit_thresh)  // substitution by a different letter
      idx = (idx + 1 + static_cast<uint32_t>(draw(ekm2, i) % (kAlpha - 1))) % kAlpha;
  }
  return static_cast<uint8_t>(kAlphaChars[idx]);
}

struct Mode1 {
  const nd_synth_spec& s;
  std::vector<uint64_t> group_first;  // logical index of each group's first member (+ total)
  M1 m;
  explicit Mode1(const nd_synth_spec& spec) : s(spec) {
    group_first.resize(s.group_count + 1);
    uint64_t acc = 0;
    for (uint64_t g = 0; g < s.group_count; ++g) {
      group_first[g] = acc;
      Stream st(s.seed * 0x9E3779B97F4A7C15ull + 0x5151 + g * 7);
      acc += s.group_size_min + st.below(static_cast<uint64_t>(s.group_size_max) - s.group_size_min + 1);
    }
    group_first[s.group_count] = acc;
    if (acc > s.doc_count) fail(ND_ERR_CONFIG, "doc count cannot hold the grouped documents");
    m.n = s.doc_count;
    m.seed = s.seed;
    m.grouped = acc;
    m.ngroups = s.group_count;
    m.perm_key = mix64(s.seed ^ 0xABCDEF);
    int bits = 2;
    while ((1ull << bits) < m.n) bits += 2;
    m.half_bits = bits / 2;
    m.half_mask = (1ull << m.half_bits) - 1;
    m.edit_thresh = s.edit_num == 0 ? 0u : static_cast<uint32_t>(std::min<long double>(
        4294967295.0L, (static_cast<long double>(s.edit_num) / s.edit_den) * 4294967296.0L));
    m.len_draws = s.len_law == 0 ? 1 : 2;
  }
  uint64_t length(Stream& st) const {
    if (s.len_law == 0) return s.len_min + st.below(static_cast<uint64_t>(s.len_max) - s.len_min + 1);
    // lognormal: median len_min, sigma = sigma_milli/1000, clipped to [200, len_max]
    double u1 = st.unit(), u2 = st.unit();
    if (u1 < 1e-300) u1 = 1e-300;
    double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    double len = std::round(s.len_min * std::exp(z * s.sigma_milli / 1000.0));
    len = std::min<double>(std::max<double>(len, 200.0), s.len_max);
    return static_cast<uint64_t>(len);
  }
  uint64_t doc_len(uint64_t position) const {
    uint64_t tk, ek;
    m1_source(m, group_first.data(), perm_inv(m, position), tk, ek);
    Stream st(tk);
    return length(st);
  }
  void doc_text(uint64_t position, uint8_t* out, uint64_t len) const {
    uint64_t tk, ek;
    m1_source(m, group_first.data(), perm_inv(m, position), tk, ek);
    const uint64_t tkm = mix64(tk);
    const uint64_t ekm = (ek && m.edit_thresh) ? mix64(ek) : 0;
    const uint64_t ekm2 = ekm ? mix64(ek ^ 0x5A5A5A5A5A5A5A5Aull) : 0;
    for (uint64_t i = 0; i < len; ++i) out[i] = m1_char(m, tkm, ekm, ekm2, i);
  }
};

__global__ void k_synth_text(M1 m, const uint64_t* __restrict__ group_first,
                             const uint64_t* __restrict__ offsets, uint8_t* __restrict__ out) {
  const uint64_t doc = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (doc >= m.n) return;
  uint64_t tk, ek;
  m1_source(m, group_first, perm_inv(m, doc), tk, ek);
  const uint64_t tkm = mix64(tk);
  const uint64_t ekm = (ek && m.edit_thresh) ? mix64(ek) : 0;
  const uint64_t ekm2 = ekm ? mix64(ek ^ 0x5A5A5A5A5A5A5A5Aull) : 0;
  const uint64_t b = offsets[doc], len = offsets[doc + 1] - b;
  for (uint64_t i = lane; i < len; i += 32) out[b + i] = m1_char(m, tkm, ekm, ekm2, i);
}

template <class F>
void parallel_range(uint64_t n, unsigned threads, F&& fn) {
  if (threads <= 1 || n < 4096) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> pool;
  uint64_t chunk = (n + threads - 1) / threads;
  for (unsigned t = 0; t < threads; ++t) {
    uint64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

void synth_generate(const nd_synth_spec& s, uint8_t* bytes, uint64_t* offsets,
                    uint64_t* nbytes_out) {
  validate(s);
  if (s.mode == 0) {
    std::lock_guard<std::mutex> lock(g_cache.mu);
    std::vector<uint8_t> key(reinterpret_cast<const uint8_t*>(&s),
                             reinterpret_cast<const uint8_t*>(&s) + sizeof s);
    if (key != g_cache.key) {
      g_cache.texts = generate_mode0(s);
      g_cache.key = key;
    }
    uint64_t off = 0;
    for (size_t i = 0; i < g_cache.texts.size(); ++i) {
      if (offsets) offsets[i] = off;
      if (bytes) std::memcpy(bytes + off, g_cache.texts[i].data(), g_cache.texts[i].size());
      off += g_cache.texts[i].size();
    }
    if (offsets) offsets[g_cache.texts.size()] = off;
    *nbytes_out = off;
    if (bytes) {  // second phase done: drop the cache
      g_cache.texts.clear();
      g_cache.texts.shrink_to_fit();
      g_cache.key.clear();
    }
    return;
  }
  if (s.mode != 1) fail(ND_ERR_CONFIG, "unknown synthetic mode");
  if (s.len_min < 5) fail(ND_ERR_CONFIG, "len_min must be at least 5");
  Mode1 gen(s);
  unsigned threads = s.threads ? s.threads : std::max(1u, std::thread::hardware_concurrency());
  std::vector<uint64_t> local;
  uint64_t* offs = offsets;
  if (!offs) {
    local.resize(s.doc_count + 1);
    offs = local.data();
  }
  parallel_range(s.doc_count, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) offs[i + 1] = gen.doc_len(i);
  });
  offs[0] = 0;
  for (uint64_t i = 0; i < s.doc_count; ++i) offs[i + 1] += offs[i];
  *nbytes_out = offs[s.doc_count];
  if (!bytes) return;
  parallel_range(s.doc_count, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) gen.doc_text(i, bytes + offs[i], offs[i + 1] - offs[i]);
  });
}

void synth_text_device(const nd_synth_spec& s, const uint64_t* d_offsets, uint8_t* d_bytes,
                       DevBuf& scratch, cudaStream_t stream) {
  validate(s);
  if (s.mode != 1) fail(ND_ERR_CONFIG, "device generation supports mode 1 only");
  Mode1 gen(s);
  uint64_t* d_gf = scratch.as<uint64_t>(gen.group_first.size());
  ND_CUDA(cudaMemcpyAsync(d_gf, gen.group_first.data(), gen.group_first.size() * sizeof(uint64_t),
                          cudaMemcpyHostToDevice, stream));
  const uint64_t threads = s.doc_count * 32;
  if (threads == 0) return;
  k_synth_text<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(gen.m, d_gf, d_offsets,
                                                                              d_bytes);
  ND_CHECK_LAUNCH();
  ND_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace ndb
