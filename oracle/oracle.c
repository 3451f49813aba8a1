/* CPU restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.
 * See oracle.h for the parity-pinning statement.  Every function cites the
 * reference file:line (under /root/reference/proj/src) it restates.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* std::mt19937_64 (the engine derive_family and the synthetic generator draw
 * from, minhash.cpp:79 / synthetic.cpp:48) */
void or_mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

uint64_t or_mt64_next(or_mt64* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= A;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* util.cpp:70-79: rejection sampling above the largest multiple of bound */
uint64_t or_bounded_random(or_mt64* g, uint64_t bound) {
  uint64_t rem = (0 - bound) % bound;
  uint64_t limit = 0 - rem;
  for (;;) {
    uint64_t x = or_mt64_next(g);
    if (x < limit || rem == 0) return x % bound;
  }
}

/* n successive bounded_random(rng, bound) draws of mt19937_64(seed): the
 * random streams the reference's acceptance criteria draw their inputs from
 * (acceptance_main.cpp:123-124, :534-545) */
void or_bounded_stream(uint64_t seed, uint64_t bound, uint64_t n, uint32_t* out) {
  or_mt64 g;
  or_mt64_seed(&g, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)or_bounded_random(&g, bound);
}

/* minhash.cpp:10-20 */
uint64_t or_mod_pow(uint64_t base, uint64_t exp, uint64_t mod) {
  uint64_t result = 1 % mod;
  base %= mod;
  while (exp > 0) {
    if (exp & 1) result = (uint64_t)(((u128)result * base) % mod);
    base = (uint64_t)(((u128)base * base) % mod);
    exp >>= 1;
  }
  return result;
}

/* minhash.cpp:22-50: deterministic Miller-Rabin, bases {2,3,5,7} */
int or_is_prime_u32(uint32_t n) {
  static const uint32_t small[4] = {2, 3, 5, 7};
  if (n < 2) return 0;
  for (int k = 0; k < 4; ++k) {
    if (n == small[k]) return 1;
    if (n % small[k] == 0) return 0;
  }
  uint32_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++s;
  }
  for (int k = 0; k < 4; ++k) {
    uint64_t x = or_mod_pow(small[k], d, n);
    if (x == 1 || x == n - 1) continue;
    int witness = 1;
    for (int i = 1; i < s; ++i) {
      x = (x * x) % n;
      if (x == n - 1) {
        witness = 0;
        break;
      }
    }
    if (witness) return 0;
  }
  return 1;
}

/* minhash.cpp:71-105: p in [2^21, 2^23), q in [257, 2^16), both prime, pair
 * distinct, drawn in that order from mt19937_64(seed) */
int or_derive_family(uint64_t seed, uint32_t H, uint32_t L, or_hash_fn* out) {
  if (H < 1 || L < 1) return -1;
  or_mt64* g = (or_mt64*)malloc(sizeof(or_mt64));
  or_mt64_seed(g, seed);
  uint32_t have = 0;
  uint64_t attempts = 0;
  while (have < H) {
    if (++attempts > 10000000ULL) {
      free(g);
      return -1;
    }
    uint32_t modulus = (uint32_t)((1u << 21) + or_bounded_random(g, (1u << 23) - (1u << 21)));
    uint32_t base = (uint32_t)(257 + or_bounded_random(g, (1u << 16) - 257));
    if (!or_is_prime_u32(modulus) || !or_is_prime_u32(base)) continue;
    int dup = 0;
    for (uint32_t i = 0; i < have; ++i)
      if (out[i].modulus == modulus && out[i].base == base) dup = 1;
    if (dup) continue;
    or_hash_fn f;
    f.modulus = modulus;
    f.base = base;
    f.base_inverse = (uint32_t)or_mod_pow(base, modulus - 2, modulus);
    f.base_power = (uint32_t)or_mod_pow(base, L - 1, modulus);
    f.reduce_factor = (uint64_t)((((u128)1) << 64) / modulus);
    out[have++] = f;
  }
  free(g);
  return 0;
}

/* minhash.cpp:61-67 */
static inline uint32_t barrett(uint64_t x, const or_hash_fn* f) {
  uint64_t q = (uint64_t)(((u128)x * f->reduce_factor) >> 64);
  uint64_t r = x - q * f->modulus;
  while (r >= f->modulus) r -= f->modulus;
  return (uint32_t)r;
}

/* minhash.cpp:111-119: Horner from the last unit */
uint32_t or_hash_window_direct(const uint32_t* w, uint32_t L, const or_hash_fn* f) {
  uint64_t acc = 0;
  for (uint32_t i = L; i-- > 0;) acc = barrett(acc * f->base + w[i], f);
  return (uint32_t)acc;
}

/* minhash.cpp:121-131: Eq. 5 update */
uint32_t or_roll_next(uint32_t state, uint32_t out, uint32_t in, const or_hash_fn* f) {
  uint64_t dropped = (uint64_t)state + f->modulus - out;
  uint64_t shifted = barrett(dropped * f->base_inverse, f);
  uint64_t appended = barrett((uint64_t)in * f->base_power, f);
  uint64_t sum = shifted + appended;
  if (sum >= f->modulus) sum -= f->modulus;
  return (uint32_t)sum;
}

/* minhash.cpp:133-162 with byte units (text.cpp:115-122) */
int or_signature_bytes(const uint8_t* text, uint64_t len, const or_hash_fn* fns, uint32_t H,
                       uint32_t L, uint32_t* out) {
  if (len < L) return -1;
  uint32_t window[64];
  if (L > 64) return -2;
  for (uint32_t i = 0; i < L; ++i) window[i] = text[i];
  for (uint32_t h = 0; h < H; ++h) {
    const or_hash_fn* f = &fns[h];
    uint32_t state = or_hash_window_direct(window, L, f);
    uint32_t best = state;
    for (uint64_t w = 1; w + L <= len; ++w) {
      state = or_roll_next(state, text[w - 1], text[w + L - 1], f);
      if (state < best) best = state;
    }
    out[h] = best;
  }
  return 0;
}

/* text.cpp:101-113 decode_codepoints: U8_NEXT walk (Unicode Table 3-7 ranges),
 * one U+FFFD per maximal ill-formed subpart.  Returns the unit count; writes
 * at most cap units. */
uint64_t or_decode_codepoints(const uint8_t* s, uint64_t len, uint32_t* out, uint64_t cap) {
  uint64_t i = 0, n = 0;
  while (i < len) {
    uint32_t b0 = s[i++], cp = 0xFFFD, c = 0, lo = 0x80, hi = 0xBF;
    int need = -1, k;
    if (b0 < 0x80) {
      cp = b0;
      need = 0;
    } else if (b0 >= 0xC2 && b0 <= 0xDF) {
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
    }
    if (need > 0) {
      for (k = 0; k < need; ++k) {
        uint32_t b;
        if (i >= len) break;
        b = s[i];
        if (b < lo || b > hi) break;
        lo = 0x80;
        hi = 0xBF;
        c = (c << 6) | (b & 0x3F);
        ++i;
      }
      cp = k == need ? c : 0xFFFD;
    }
    if (n < cap) out[n] = cp;
    ++n;
  }
  return n;
}

/* minhash.cpp:133-162 over u32 units (text_units output); returns -1 if short */
int or_signature_units(const uint32_t* u, uint64_t len, const or_hash_fn* fns, uint32_t H,
                       uint32_t L, uint32_t* out) {
  if (len < L) return -1;
  for (uint32_t h = 0; h < H; ++h) {
    const or_hash_fn* f = &fns[h];
    uint32_t state = or_hash_window_direct(u, L, f);
    uint32_t best = state;
    for (uint64_t w = 1; w + L <= len; ++w) {
      state = or_roll_next(state, u[w - 1], u[w + L - 1], f);
      if (state < best) best = state;
    }
    out[h] = best;
  }
  return 0;
}

/* batch with a shingle unit (0 byte, 1 codepoint) */
int or_signature_batch_unit(const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                            const or_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit,
                            uint32_t* out) {
  uint64_t i, j;
  for (i = 0; i < n; ++i) {
    const uint8_t* t = bytes + offsets[i];
    uint64_t len = offsets[i + 1] - offsets[i];
    uint32_t* units = (uint32_t*)malloc((len ? len : 1) * sizeof(uint32_t));
    uint64_t m;
    int rc;
    if (!units) return -3;
    if (unit == 1) {
      m = or_decode_codepoints(t, len, units, len);
    } else {
      for (j = 0; j < len; ++j) units[j] = t[j];
      m = len;
    }
    rc = or_signature_units(units, m, fns, H, L, out + i * H);
    free(units);
    if (rc != 0) return rc;
  }
  return 0;
}

int or_signature_batch(const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                       const or_hash_fn* fns, uint32_t H, uint32_t L, uint32_t* out) {
  for (uint64_t i = 0; i < n; ++i) {
    int rc = or_signature_bytes(bytes + offsets[i], offsets[i + 1] - offsets[i], fns, H, L,
                                out + i * H);
    if (rc != 0) return rc;
  }
  return 0;
}

/* lsh.cpp:12-22 */
static uint64_t isqrt_u128(u128 x) {
  if (x == 0) return 0;
  u128 r = (u128)__builtin_sqrtl((long double)x);
  if (r == 0) r = 1;
  for (int i = 0; i < 4; ++i) r = (r + x / r) / 2;
  if (r > (u128)UINT64_MAX) r = UINT64_MAX;
  while (r * r > x) --r;
  while (r < UINT64_MAX && (r + 1) * (r + 1) <= x) ++r;
  return (uint64_t)r;
}

/* lsh.cpp:26-40: K = max(1, ceil(num*sqrt(N)/den)); Ratio reduces num/den
 * by their gcd first (util.cpp:19-27), which does not change the value. */
uint32_t or_choose_bucket_count(uint64_t n, uint64_t num, uint64_t den) {
  if (num == 0 || den == 0) return 0;
  { /* Ratio(n, d) reduces (util.cpp:19-27) */
    uint64_t a = num, b = den;
    while (b) {
      uint64_t t = a % b;
      a = b;
      b = t;
    }
    num /= a;
    den /= a;
  }
  if (n == 0) return 1;
  u128 m = (u128)num * num * n;
  uint64_t root = isqrt_u128(m);
  int exact = (u128)root * root == m && root % den == 0;
  uint64_t k = exact ? root / den : root / den + 1;
  if (k < 1) k = 1;
  if (k > UINT32_MAX) return 0;
  return (uint32_t)k;
}

/* lsh.cpp:42-60 */
void or_band_bucket_ids(const uint32_t* sig, uint32_t bands, uint32_t rows, uint32_t K,
                        uint32_t* out) {
  for (uint32_t j = 0; j < bands; ++j) {
    uint64_t sum = 0;
    for (uint32_t i = 0; i < rows; ++i) sum += sig[j * rows + i];
    out[j] = (uint32_t)(sum % K);
  }
}

/* compare.cpp:17-22 */
uint32_t or_min_matches(uint32_t H, uint64_t num, uint64_t den) {
  u128 lhs = (u128)num * H;
  uint64_t m = (uint64_t)(lhs / den) + 1;
  return m > H ? H + 1 : (uint32_t)m;
}

/* compare.hpp:31-34: strict m*den > num*H */
int or_accepts(uint32_t m, uint32_t H, uint64_t num, uint64_t den) {
  return (u128)m * den > (u128)num * H;
}

/* compare.cpp:24-67, written as the naive double loop (test_compare.cpp:16-30);
 * the tiled order visits the same pair set. */
uint64_t or_compare_cell(const uint32_t* sigs, uint32_t H, const uint32_t* rows, uint64_t n,
                         uint64_t num, uint64_t den, uint32_t* lo, uint32_t* hi, uint32_t* m,
                         uint64_t cap) {
  uint64_t found = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t* a = sigs + (uint64_t)rows[i] * H;
    for (uint64_t j = i + 1; j < n; ++j) {
      const uint32_t* b = sigs + (uint64_t)rows[j] * H;
      uint32_t matches = 0;
      for (uint32_t h = 0; h < H; ++h) matches += a[h] == b[h];
      if (or_accepts(matches, H, num, den)) {
        if (found < cap) {
          lo[found] = rows[i];
          hi[found] = rows[j];
          m[found] = matches;
        }
        ++found;
      }
    }
  }
  return found;
}

/* dedup_graph.cpp:28-46: path compression + union by rank */
static uint32_t uf_find(uint32_t* parent, uint32_t x) {
  uint32_t r = x;
  while (parent[r] != r) r = parent[r];
  while (parent[x] != r) {
    uint32_t nx = parent[x];
    parent[x] = r;
    x = nx;
  }
  return r;
}

/* dedup_graph.cpp:48-81: components; the representative is the minimum member */
void or_components(const uint32_t* lo, const uint32_t* hi, uint64_t npairs, uint32_t nnodes,
                   uint32_t* label_out) {
  uint32_t* parent = (uint32_t*)malloc(sizeof(uint32_t) * (nnodes ? nnodes : 1));
  uint8_t* rank = (uint8_t*)calloc(nnodes ? nnodes : 1, 1);
  uint8_t* seen = (uint8_t*)calloc(nnodes ? nnodes : 1, 1);
  for (uint32_t i = 0; i < nnodes; ++i) parent[i] = i;
  for (uint64_t e = 0; e < npairs; ++e) {
    seen[lo[e]] = seen[hi[e]] = 1;
    uint32_t ra = uf_find(parent, lo[e]), rb = uf_find(parent, hi[e]);
    if (ra == rb) continue;
    if (rank[ra] < rank[rb]) {
      uint32_t t = ra;
      ra = rb;
      rb = t;
    }
    parent[rb] = ra;
    if (rank[ra] == rank[rb]) ++rank[ra];
  }
  uint32_t* minof = (uint32_t*)malloc(sizeof(uint32_t) * (nnodes ? nnodes : 1));
  for (uint32_t i = 0; i < nnodes; ++i) minof[i] = UINT32_MAX;
  for (uint32_t i = 0; i < nnodes; ++i) {
    if (!seen[i]) continue;
    uint32_t r = uf_find(parent, i);
    if (i < minof[r]) minof[r] = i;
  }
  for (uint32_t i = 0; i < nnodes; ++i) label_out[i] = seen[i] ? minof[uf_find(parent, i)] : UINT32_MAX;
  free(parent);
  free(rank);
  free(seen);
  free(minof);
}
