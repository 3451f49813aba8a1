/* CPU restatement of the reference's MinHash-LSH hot path (TEST INFRASTRUCTURE ONLY).
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * against (a) the reference's own unit-test vectors (test_minhash.cpp,
 * test_lsh.cpp, test_compare.cpp, test_dedup_graph.cpp), (b) SURVEY App. A
 * known-answer values produced by the reference, and (c) oracle/_ref (the
 * reference's own sources compiled in place) on seeded random inputs.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so, and only as the checker.  The product never links it.
 */
#ifndef ND_ORACLE_H
#define ND_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t modulus, base, base_inverse, base_power;
  uint64_t reduce_factor;
} or_hash_fn; /* minhash.hpp:17-25 HashFunctionParams */

typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64; /* std::mt19937_64 */

void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);
uint64_t or_bounded_random(or_mt64* g, uint64_t bound);               /* util.cpp:70-79 */
void or_bounded_stream(uint64_t seed, uint64_t bound, uint64_t n, uint32_t* out);
uint64_t or_mod_pow(uint64_t base, uint64_t exp, uint64_t mod);       /* minhash.cpp:10-20 */
int or_is_prime_u32(uint32_t n);                                      /* minhash.cpp:22-50 */
int or_derive_family(uint64_t seed, uint32_t H, uint32_t L, or_hash_fn* out); /* minhash.cpp:71-105 */
uint32_t or_hash_window_direct(const uint32_t* w, uint32_t L, const or_hash_fn* f); /* :111-119 */
uint32_t or_roll_next(uint32_t state, uint32_t out, uint32_t in, const or_hash_fn* f); /* :121-131 */
/* signature_of_document over byte units (minhash.cpp:133-162); returns -1 if short */
int or_signature_bytes(const uint8_t* text, uint64_t len, const or_hash_fn* fns, uint32_t H,
                       uint32_t L, uint32_t* out);
/* batch form over a packed buffer, rows written at out + i*H */
int or_signature_batch(const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                       const or_hash_fn* fns, uint32_t H, uint32_t L, uint32_t* out);
/* text.cpp:101-113 decode_codepoints; returns the unit count (writes <= cap) */
uint64_t or_decode_codepoints(const uint8_t* s, uint64_t len, uint32_t* out, uint64_t cap);
/* signature_of_document over u32 units; returns -1 if short */
int or_signature_units(const uint32_t* units, uint64_t len, const or_hash_fn* fns, uint32_t H,
                       uint32_t L, uint32_t* out);
/* batch form with a shingle unit (0 byte, 1 codepoint) */
int or_signature_batch_unit(const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                            const or_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit,
                            uint32_t* out);
uint32_t or_choose_bucket_count(uint64_t n, uint64_t num, uint64_t den); /* lsh.cpp:26-40, 0 = error */
void or_band_bucket_ids(const uint32_t* sig, uint32_t bands, uint32_t rows, uint32_t K,
                        uint32_t* out); /* lsh.cpp:42-60 */
uint32_t or_min_matches(uint32_t H, uint64_t num, uint64_t den); /* compare.cpp:17-22 */
int or_accepts(uint32_t m, uint32_t H, uint64_t num, uint64_t den); /* compare.hpp:31-34 */
/* naive all-pairs of one cell (compare.cpp:24-67 / test_compare.cpp:16-30).
 * rows: cell members (indices into sigs, ascending doc order). Appends to
 * lo/hi/m (capacity cap); returns number of pairs found (may exceed cap). */
uint64_t or_compare_cell(const uint32_t* sigs, uint32_t H, const uint32_t* rows, uint64_t n,
                         uint64_t num, uint64_t den, uint32_t* lo, uint32_t* hi, uint32_t* m,
                         uint64_t cap);
/* Union-find components over dense node ids < nnodes (dedup_graph.cpp:9-81).
 * label_out[i] = smallest node id in i's component, or UINT32_MAX when i is
 * in no pair. */
void or_components(const uint32_t* lo, const uint32_t* hi, uint64_t npairs, uint32_t nnodes,
                   uint32_t* label_out);

#ifdef __cplusplus
}
#endif
#endif
