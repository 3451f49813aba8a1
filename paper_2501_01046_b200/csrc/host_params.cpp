// Host-side parameter logic of the hot path (no device work):
//   derive_family        minhash.cpp:71-105 (Miller-Rabin minhash.cpp:22-50,
//                        bounded_random util.cpp:70-79)
//   choose_bucket_count  lsh.cpp:26-40
//   min_matches          compare.cpp:17-22
//   band_partition       lsh.cpp:62-72
// These must be bit-identical with the reference: the family is pinned by the
// FNV checksums of SURVEY App. A (tests/test_host.py).
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <set>
#include <string>
#include <utility>

#include "host_internal.hpp"

namespace ndb {

namespace {
using u128 = unsigned __int128;

uint64_t mod_pow(uint64_t base, uint64_t exp, uint64_t mod) {
  uint64_t result = 1 % mod;
  base %= mod;
  while (exp > 0) {
    if (exp & 1) result = static_cast<uint64_t>(static_cast<u128>(result) * base % mod);
    base = static_cast<uint64_t>(static_cast<u128>(base) * base % mod);
    exp >>= 1;
  }
  return result;
}

bool is_prime_u32(uint32_t n) {
  if (n < 2) return false;
  for (uint32_t p : {2u, 3u, 5u, 7u}) {
    if (n == p) return true;
    if (n % p == 0) return false;
  }
  uint32_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++s;
  }
  for (uint32_t a : {2u, 3u, 5u, 7u}) {  // exact below 3,215,031,751
    uint64_t x = mod_pow(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool composite = true;
    for (int i = 1; i < s && composite; ++i) {
      x = x * x % n;
      if (x == n - 1) composite = false;
    }
    if (composite) return false;
  }
  return true;
}

uint64_t isqrt_u128(u128 x) {
  if (x == 0) return 0;
  u128 r = static_cast<u128>(std::sqrt(static_cast<long double>(x)));
  if (r == 0) r = 1;
  for (int i = 0; i < 4; ++i) r = (r + x / r) / 2;
  const u128 cap = std::numeric_limits<uint64_t>::max();
  if (r > cap) r = cap;
  while (r * r > x) --r;
  while (r < cap && (r + 1) * (r + 1) <= x) ++r;
  return static_cast<uint64_t>(r);
}

uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}
}  // namespace

uint64_t bounded_random(std::mt19937_64& rng, uint64_t bound) {
  if (bound == 0) fail(ND_ERR_CONFIG, "bounded_random: bound must be positive");
  uint64_t rem = (0 - bound) % bound;
  uint64_t limit = 0 - rem;
  for (;;) {
    uint64_t x = rng();
    if (x < limit || rem == 0) return x % bound;
  }
}

std::vector<nd_hash_fn> derive_family(uint64_t seed, uint32_t H, uint32_t L, uint32_t unit) {
  if (H < 1) fail(ND_ERR_CONFIG, "hash count must be at least 1");
  if (L < 1) fail(ND_ERR_CONFIG, "shingle length must be at least 1");
  if (unit > 1) fail(ND_ERR_CONFIG, "unknown shingle unit");
  std::vector<nd_hash_fn> out;
  out.reserve(H);
  std::mt19937_64 rng(seed);
  std::set<std::pair<uint32_t, uint32_t>> used;
  uint64_t attempts = 0;
  constexpr uint32_t kPLo = 1u << 21, kPHi = 1u << 23, kQLo = 257, kQHi = 1u << 16;
  while (out.size() < H) {
    if (++attempts > 10'000'000ull)
      fail(ND_ERR_CONFIG, "could not derive " + std::to_string(H) +
                              " distinct hash functions; lower the hash count");
    auto p = static_cast<uint32_t>(kPLo + bounded_random(rng, kPHi - kPLo));
    auto q = static_cast<uint32_t>(kQLo + bounded_random(rng, kQHi - kQLo));
    if (!is_prime_u32(p) || !is_prime_u32(q)) continue;
    if (!used.insert({p, q}).second) continue;
    nd_hash_fn f;
    f.modulus = p;
    f.base = q;
    f.base_inverse = static_cast<uint32_t>(mod_pow(q, p - 2, p));
    f.base_power = static_cast<uint32_t>(mod_pow(q, L - 1, p));
    f.reduce_factor = static_cast<uint64_t>((static_cast<u128>(1) << 64) / p);
    out.push_back(f);
  }
  return out;
}

uint32_t choose_bucket_count(uint64_t n, uint64_t num, uint64_t den) {
  if (den == 0) fail(ND_ERR_CONFIG, "ratio denominator must be positive");
  if (num == 0) fail(ND_ERR_CONFIG, "bucket scale must be positive");
  uint64_t g = gcd_u64(num, den);
  num /= g;
  den /= g;
  if (n == 0) return 1;
  u128 m = static_cast<u128>(num) * num * n;
  uint64_t root = isqrt_u128(m);
  bool exact = static_cast<u128>(root) * root == m && root % den == 0;
  uint64_t k = exact ? root / den : root / den + 1;
  if (k < 1) k = 1;
  if (k > std::numeric_limits<uint32_t>::max())
    fail(ND_ERR_CONFIG, "bucket count " + std::to_string(k) + " exceeds 32 bits; lower the bucket scale");
  return static_cast<uint32_t>(k);
}

uint32_t min_matches(uint32_t H, uint64_t num, uint64_t den) {
  if (den == 0) return H + 1;
  u128 lhs = static_cast<u128>(num) * H;
  uint64_t m = static_cast<uint64_t>(lhs / den) + 1;
  return m > H ? H + 1 : static_cast<uint32_t>(m);
}

// ---- public scalar primitives of minhash.hpp (host) ------------------------
uint64_t mod_pow_checked(uint64_t base, uint64_t exp, uint64_t mod) {  // minhash.cpp:10-20
  if (mod == 0) fail(ND_ERR_CONFIG, "mod_pow: zero modulus");
  return mod_pow(base, exp, mod);
}

bool is_prime(uint32_t n) { return is_prime_u32(n); }  // minhash.cpp:22-50

namespace {
// minhash.cpp:61-67: x mod p for x < 2^48 through floor(2^64 / p)
uint32_t barrett(uint64_t x, const nd_hash_fn& f) {
  const uint64_t q = static_cast<uint64_t>((static_cast<u128>(x) * f.reduce_factor) >> 64);
  uint64_t r = x - q * f.modulus;
  while (r >= f.modulus) r -= f.modulus;
  return static_cast<uint32_t>(r);
}
}  // namespace

// minhash.cpp:111-119 (Horner from the last unit)
uint32_t hash_window_direct(const uint32_t* w, uint32_t len, const nd_hash_fn& f) {
  if (len == 0) fail(ND_ERR_CONFIG, "hash_window_direct: empty window");
  uint64_t acc = 0;
  for (uint32_t i = len; i-- > 0;) acc = barrett(acc * f.base + w[i], f);
  return static_cast<uint32_t>(acc);
}

// minhash.cpp:121-131 (Eq. 5 update)
uint32_t roll_next(uint32_t state, uint32_t outgoing, uint32_t incoming, const nd_hash_fn& f) {
  const uint64_t dropped = static_cast<uint64_t>(state) + f.modulus - outgoing;
  const uint64_t shifted = barrett(dropped * f.base_inverse, f);
  const uint64_t appended = barrett(static_cast<uint64_t>(incoming) * f.base_power, f);
  uint64_t sum = shifted + appended;
  if (sum >= f.modulus) sum -= f.modulus;
  return static_cast<uint32_t>(sum);
}

}  // namespace ndb
