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

#include "host_internal.hpp"

namespace ndb {
namespace {

constexpr char kAlphabet[] = "abcdefghijklmnopqrstuvwxyz0123456789 ";
constexpr uint64_t kAlpha = 37;

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
inline uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Stream {  // counter-based stream: x_i = mix64(key + i * golden)
  uint64_t key, ctr = 0;
  explicit Stream(uint64_t k) : key(mix64(k)) {}
  uint64_t next() { return mix64(key + (ctr++) * 0xD1B54A32D192ED03ull); }
  uint64_t below(uint64_t b) { return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * b) >> 64); }
  double unit() { return (next() >> 11) * (1.0 / 9007199254740992.0); }
};

// bijection on [0, n) (Feistel on 2*half bits + cycle walking)
struct Perm {
  uint64_t n, half_mask;
  int half_bits;
  uint64_t key;
  Perm(uint64_t n_, uint64_t seed) : n(n_), key(seed) {
    int bits = 2;
    while ((1ull << bits) < n) bits += 2;
    half_bits = bits / 2;
    half_mask = (1ull << half_bits) - 1;
  }
  uint64_t round_f(uint64_t x, int r) const { return mix64(x ^ (key + 0x100000001B3ull * r)) & half_mask; }
  uint64_t enc(uint64_t x) const {
    uint64_t l = x >> half_bits, rr = x & half_mask;
    for (int r = 0; r < 4; ++r) {
      uint64_t t = l ^ round_f(rr, r);
      l = rr;
      rr = t;
    }
    return (l << half_bits) | rr;
  }
  uint64_t dec(uint64_t y) const {
    uint64_t l = y >> half_bits, rr = y & half_mask;
    for (int r = 3; r >= 0; --r) {
      uint64_t t = rr ^ round_f(l, r);
      rr = l;
      l = t;
    }
    return (l << half_bits) | rr;
  }
  uint64_t fwd(uint64_t x) const {
    do x = enc(x);
    while (x >= n);
    return x;
  }
  uint64_t inv(uint64_t y) const {
    do y = dec(y);
    while (y >= n);
    return y;
  }
};

struct Mode1 {
  const nd_synth_spec& s;
  std::vector<uint64_t> group_first;  // logical index of each group's first member (+ total)
  Perm perm;
  uint64_t edit_thresh;  // P(edit) * 2^32
  explicit Mode1(const nd_synth_spec& spec) : s(spec), perm(spec.doc_count, mix64(spec.seed ^ 0xABCDEF)) {
    group_first.resize(s.group_count + 1);
    uint64_t acc = 0;
    for (uint64_t g = 0; g < s.group_count; ++g) {
      group_first[g] = acc;
      Stream st(s.seed * 0x9E3779B97F4A7C15ull + 0x5151 + g * 7);
      acc += s.group_size_min + st.below(static_cast<uint64_t>(s.group_size_max) - s.group_size_min + 1);
    }
    group_first[s.group_count] = acc;
    if (acc > s.doc_count) fail(ND_ERR_CONFIG, "doc count cannot hold the grouped documents");
    edit_thresh = static_cast<uint64_t>((static_cast<long double>(s.edit_num) / s.edit_den) * 4294967296.0L);
  }
  // logical index -> (text stream key, edit stream key or 0)
  void source(uint64_t logical, uint64_t& text_key, uint64_t& edit_key) const {
    if (logical < group_first[s.group_count]) {
      uint64_t g = std::upper_bound(group_first.begin(), group_first.end(), logical) - group_first.begin() - 1;
      uint64_t m = logical - group_first[g];
      text_key = s.seed * 0x632BE59BD9B4E019ull + 0x7777 + g;
      edit_key = m == 0 ? 0 : (s.seed * 0x8CB92BA72F3D8DD7ull + (g << 8) + m + 1);
    } else {
      text_key = s.seed * 0x632BE59BD9B4E019ull + 0x3333333333ull + logical;
      edit_key = 0;
    }
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
    source(perm.inv(position), tk, ek);
    Stream st(tk);
    return length(st);
  }
  void doc_text(uint64_t position, uint8_t* out) const {
    uint64_t tk, ek;
    source(perm.inv(position), tk, ek);
    Stream st(tk);
    uint64_t len = length(st);
    uint64_t i = 0;
    while (i < len) {
      uint64_t x = st.next();
      for (int k = 0; k < 2 && i < len; ++k, ++i) {
        uint32_t h = static_cast<uint32_t>(x >> (32 * k));
        out[i] = static_cast<uint8_t>(kAlphabet[(static_cast<uint64_t>(h) * kAlpha) >> 32]);
      }
    }
    if (ek && s.edit_num) {
      Stream ed(ek);
      for (uint64_t j = 0; j < len; j += 2) {
        uint64_t x = ed.next();
        for (int k = 0; k < 2 && j + k < len; ++k) {
          uint32_t h = static_cast<uint32_t>(x >> (32 * k));
          if (h < edit_thresh) {
            uint8_t c = out[j + k];
            uint8_t r;
            do r = static_cast<uint8_t>(kAlphabet[ed.below(kAlpha)]);
            while (r == c);
            out[j + k] = r;
          }
        }
      }
    }
  }
};

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
    for (uint64_t i = b; i < e; ++i) gen.doc_text(i, bytes + offs[i]);
  });
}

}  // namespace ndb
