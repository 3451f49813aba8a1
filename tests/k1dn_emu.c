/* Host emulation of K1j's dn arithmetic (paper_2501_01046_b200/csrc/k1_jit.cpp,
 * rold()), for the CPU tests: one roll per call with the plan row's constants
 * (nd_k1j_plan), IEEE single precision with the same rounding as the device
 * instructions (FMUL.RN, FFMA.RN with denormal inputs, FADD.RM).  Test
 * infrastructure only -- the product runs the generated CUDA kernel. */
#include <fenv.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#pragma STDC FENV_ACCESS ON

static float f_of(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t b_of(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* row: {pass, class, g, w, fn, q, QLn, kp, p, A, B, M} */
uint32_t dn_rol(const uint32_t* r, uint32_t z, uint32_t c_in, uint32_t c_out) {
  const uint32_t g = r[2], w = r[3], q = r[5], qln = r[6], kp = r[7], p = r[8];
  volatile float cf = (float)(c_out + 256u * g);
  volatile float t1 = cf * f_of(r[10]);
  volatile float R = fmaf(f_of(z), f_of(r[9]), t1);
  fesetround(FE_DOWNWARD);
  volatile float S = R + f_of(r[11]);
  fesetround(FE_TONEAREST);
  const uint32_t kb = b_of(S);
  uint32_t x = c_out * qln + (c_in | (w & 0xFFFFFF00u));
  x = z * q + x;
  x = kb * kp + x;
  const int32_t a = (int32_t)(x + p), b = (int32_t)x;
  return (uint32_t)(a < b ? a : b);
}

static uint64_t mod_inv(uint64_t a, uint64_t p) { /* a^(p-2) mod p, p prime */
  uint64_t r = 1, e = p - 2;
  a %= p;
  while (e) {
    if (e & 1) r = r * a % p;
    a = a * a % p;
    e >>= 1;
  }
  return r;
}

/* Every (c_out, c_in) byte pair with the states whose next residue is one of
 * 0, 1, 2, p-3, p-2, p-1 (u/p next to an integer: where the quotient estimate
 * is decided), plus c = 0 and c = p-1; returns the mismatches against
 * (q c + c_out QLn + c_in) mod p. */
uint64_t dn_check_edges(const uint32_t* r) {
  const uint64_t q = r[5], qln = r[6], p = r[8], qinv = mod_inv(q, p);
  uint64_t bad = 0;
  for (uint32_t co = 0; co < 256; ++co)
    for (uint32_t ci = 0; ci < 256; ++ci) {
      const uint64_t base = (co * qln + ci) % p;
      uint64_t cs[8];
      const uint64_t tg[6] = {0, 1, 2, p - 3, p - 2, p - 1};
      for (int i = 0; i < 6; ++i) cs[i] = (tg[i] + p - base) % p * qinv % p;
      cs[6] = 0;
      cs[7] = p - 1;
      for (int i = 0; i < 8; ++i) {
        const uint64_t c = cs[i];
        const uint32_t want = 0x80000000u + (uint32_t)((q * c + co * qln + ci) % p);
        if (dn_rol(r, 0x80000000u + (uint32_t)c, ci, co) != want) ++bad;
      }
    }
  return bad;
}

/* n random (c, c_in, c_out) draws (xorshift) */
uint64_t dn_check_random(const uint32_t* r, uint64_t n, uint64_t seed) {
  const uint64_t q = r[5], qln = r[6], p = r[8];
  uint64_t s = seed | 1, bad = 0;
  for (uint64_t i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const uint64_t c = (s >> 16) % p;
    const uint32_t ci = (uint32_t)(s & 0xFF), co = (uint32_t)((s >> 8) & 0xFF);
    const uint32_t want = 0x80000000u + (uint32_t)((q * c + co * qln + ci) % p);
    if (dn_rol(r, 0x80000000u + (uint32_t)c, ci, co) != want) ++bad;
  }
  return bad;
}

/* signature_of_document with the dn roll: backward over the whole document
 * from state 0 at its end (the L-1 partial windows warm up), min over the
 * full windows; rows = the plan (nrows = H), sig[fn] = m ^ 0x80000000 */
void dn_signatures(const uint32_t* rows, uint32_t nrows, uint32_t L, const uint8_t* text,
                   const uint64_t* offsets, uint64_t ndocs, uint32_t H, uint32_t* sig) {
  for (uint64_t d = 0; d < ndocs; ++d) {
    const uint8_t* t = text + offsets[d];
    const int64_t len = (int64_t)(offsets[d + 1] - offsets[d]);
    for (uint32_t k = 0; k < nrows; ++k) {
      const uint32_t* r = rows + 12 * k;
      uint32_t z = 0x80000000u;
      int32_t m = 0x7fffffff;
      for (int64_t pos = len - 1; pos >= 0; --pos) {
        const uint32_t co = pos + (int64_t)L < len ? t[pos + L] : 0u;
        z = dn_rol(r, z, t[pos], co);
        if (pos + (int64_t)L <= len && (int32_t)z < m) m = (int32_t)z;
      }
      sig[d * H + r[4]] = (uint32_t)m ^ 0x80000000u;
    }
  }
}
