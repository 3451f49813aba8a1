// K3: all-pairs comparison inside LSH cells -- compare_bucket
// (compare.cpp:24-67) over every non-singleton cell.
//
// The reference counts all H positions of every pair (i < j) and accepts iff
// m*den > num*H (compare.hpp:31-34), i.e. m >= min_matches.  A pair can only
// be accepted if it has at most A = H - min_matches mismatches, so a pair
// with NO match among any fixed P >= A+1 positions is provably rejected (the
// exact early-termination rule of the reference's own oracle,
// oracle.cpp:81-92, proven equal to the full scan by test_oracle.cpp:96-112).
//
// Layout: one 128-thread CTA per (cell, tile of kCmpRows = 256 rows).  Thread t
// owns rows tile*256 + t and + 128 and keeps the first Pf values of both
// signatures in registers.  Columns j > i stream through shared memory in batches of 64
// (Pf values each) and are read back as broadcast LDS.128; the prefilter is
// an OR-chain of equality tests (ISETP.EQ.OR).  Survivors are queued in
// shared memory and, after each column batch, counted exactly by whole warps
// (32 positions per step, ballot/popc, the same early exit) so a rare
// survivor does not stall its warp; accepted pairs are appended with one
// atomic per pair.  Pairs are canonical (lo < hi) row
// indices packed as lo << nb | hi so that sort + unique (compare.cpp:77-84)
// is a single radix sort over 2*nb bits.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "nd_internal.cuh"
#include "k_compare_util.cuh"

namespace ndb {
namespace {

constexpr int kCols = 64;  // columns staged per batch

// Warp-cooperative exact count of one candidate pair: lanes compare 32
// consecutive positions per step (coalesced 128-byte row reads) and a
// ballot/popc reduces them; the early exit of oracle.cpp:81-92 is applied per
// 32-position chunk.  Returns true when accepted (m >= min_match).
__device__ __forceinline__ bool warp_count(const uint32_t* __restrict__ a,
                                           const uint32_t* __restrict__ b, uint32_t H,
                                           uint32_t allowed, uint32_t min_match, uint32_t& m) {
  const int lane = threadIdx.x & 31;
  uint32_t matches = 0;
  for (uint32_t h0 = 0; h0 < H; h0 += 32) {
    const uint32_t h = h0 + lane;
    const bool eq = h < H && __ldg(a + h) == __ldg(b + h);
    matches += __popc(__ballot_sync(0xFFFFFFFFu, eq));
    const uint32_t seen = min(H, h0 + 32);
    if (seen - matches > allowed) return false;
  }
  m = matches;
  return matches >= min_match;
}

// Pf > 0: prefilter over the first Pf positions (Pf >= H - min_matches + 1);
// prefilter survivors are queued in shared memory and counted exactly by
// whole warps after each column batch, so one survivor no longer stalls its
// warp's 31 other lanes (a full queue falls back to an inline count).
// Pf == 0: no prefilter (every pair is a survivor).  Each thread owns kR rows
// (i and i + kThreads), so every broadcast LDS.128 feeds 4*kR comparisons.
constexpr int kThreads = 128;
constexpr int kR = kCmpRows / kThreads;  // rows per thread
constexpr int kQueue = 1024;             // survivor slots per CTA (drained every batch)

template <int Pf>
__global__ void __launch_bounds__(kThreads)
    k_compare(const SigView sv, uint32_t H, const uint32_t* __restrict__ rows,
              const uint64_t* __restrict__ cell_start, const uint32_t* __restrict__ cell_len,
              const uint32_t* __restrict__ item_cell, const uint64_t* __restrict__ item_off,
              uint32_t min_match, int nb, uint64_t* __restrict__ out_key,
              uint32_t* __restrict__ out_m, unsigned long long* __restrict__ count, uint64_t cap) {
  constexpr int PS = Pf > 0 ? ((Pf + 3) / 4) * 4 : 4;
  __shared__ __align__(16) uint32_t cols[kCols][PS];
  __shared__ uint32_t col_row[kCols];
  __shared__ uint2 queue[kQueue];
  __shared__ uint32_t qn;
  const uint32_t item = blockIdx.x;
  const uint32_t cell = item_cell[item];
  const uint32_t tile = static_cast<uint32_t>(item - item_off[cell]);
  const uint64_t s = cell_start[cell];
  const uint32_t n = cell_len[cell];
  const uint32_t allowed = H - min_match;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kWarpsPerBlock = kThreads / 32;

  uint32_t ri[kR], row[kR];
  bool valid[kR];
  uint32_t pre[kR][Pf > 0 ? Pf : 1];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    ri[r] = tile * kCmpRows + r * kThreads + threadIdx.x;
    valid[r] = ri[r] < n;
    row[r] = valid[r] ? rows[s + ri[r]] : 0;
    if constexpr (Pf > 0) {
      const uint32_t* my_sig = sv.row(row[r]);
#pragma unroll
      for (int k = 0; k < Pf; ++k) pre[r][k] = valid[r] ? __ldg(my_sig + k) : 0xFFFFFFFFu;
    }
  }
  if (threadIdx.x == 0) qn = 0;

  for (uint32_t j0 = tile * kCmpRows + 1; j0 < n; j0 += kCols) {
    const uint32_t cmax = min(static_cast<uint32_t>(kCols), n - j0);
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < cmax; c += kThreads) col_row[c] = rows[s + j0 + c];
    if constexpr (Pf > 0) {
      __syncthreads();
      for (uint32_t idx = threadIdx.x; idx < cmax * Pf; idx += kThreads) {
        const uint32_t c = idx / Pf, k = idx % Pf;
        cols[c][k] = __ldg(sv.row(col_row[c]) + k);
      }
    }
    __syncthreads();
    // columns j <= i are not row i's (upper triangle, compare.cpp:46)
    const uint32_t c0 = valid[0] ? ((ri[0] + 1 > j0) ? ri[0] + 1 - j0 : 0) : cmax;
    for (uint32_t c = c0; c < cmax; ++c) {
      const uint32_t j = j0 + c;
      bool cand[kR];
      if constexpr (Pf > 0) {
        bool any[kR];
#pragma unroll
        for (int r = 0; r < kR; ++r) any[r] = false;
        const uint4* col = reinterpret_cast<const uint4*>(cols[c]);
#pragma unroll
        for (int q = 0; q < PS / 4; ++q) {
          const uint4 v = col[q];
#pragma unroll
          for (int r = 0; r < kR; ++r) {
            if (4 * q + 0 < Pf) any[r] |= pre[r][4 * q + 0] == v.x;
            if (4 * q + 1 < Pf) any[r] |= pre[r][4 * q + 1] == v.y;
            if (4 * q + 2 < Pf) any[r] |= pre[r][4 * q + 2] == v.z;
            if (4 * q + 3 < Pf) any[r] |= pre[r][4 * q + 3] == v.w;
          }
        }
#pragma unroll
        for (int r = 0; r < kR; ++r) cand[r] = any[r];
      } else {
#pragma unroll
        for (int r = 0; r < kR; ++r) cand[r] = true;
      }
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        if (cand[r] && valid[r] && j > ri[r]) {
          const uint32_t other = col_row[c];
          const uint32_t slot = atomicAdd(&qn, 1u);
          if (slot < kQueue) {
            queue[slot] = make_uint2(row[r], other);
          } else {  // queue full: count inline
            bool alive;
            const uint32_t m = full_matches(sv.row(row[r]),
                                            sv.row(other), H, allowed, alive);
            if (alive && m >= min_match) emit(row[r], other, m, nb, out_key, out_m, count, cap);
          }
        }
      }
    }
    __syncthreads();
    // drain the survivors: one warp per candidate pair
    const uint32_t lim = min(qn, static_cast<uint32_t>(kQueue));
    for (uint32_t t = warp; t < lim; t += kWarpsPerBlock) {
      const uint2 pr = queue[t];
      uint32_t m;
      if (warp_count(sv.row(pr.x), sv.row(pr.y), H,
                     allowed, min_match, m) && lane == 0)
        emit(pr.x, pr.y, m, nb, out_key, out_m, count, cap);
    }
    __syncthreads();
    if (threadIdx.x == 0) qn = 0;
  }
}

// ---------------------------------------------------------------------------
// Exact hash-join candidate generation for cells of up to kJoinMax documents.
//
// A pair with no match among positions [0, P) (P = H - min_matches + 1) is
// provably rejected (see the header), so the pairs worth counting are exactly
// the pairs that share a value at some position k < P.  Instead of testing
// all n(n-1)/2 pairs, one CTA per cell builds, for each k, a hash table of
// value -> chain of documents in shared memory (tagged entries, so tables are
// never cleared between positions) and enumerates the pairs inside each
// chain: O(n*P) work per cell instead of O(n^2*P).  Each candidate (d, e)
// found at position k is checked by one thread: the first P' = min(H, 32)
// positions of both rows are compared, the candidate is dropped unless k is
// its FIRST matching position (each pair is checked once per cell) and unless
// it has at most H - min_matches mismatches so far; survivors get the full
// early-exit count (oracle.cpp:81-92) and accepted pairs are emitted.
constexpr int kJoinThreads = 256;

__device__ __forceinline__ void join_check(const SigView sv, uint32_t H,
                                           uint32_t ra, uint32_t rb, uint32_t k, uint32_t P,
                                           uint32_t min_match, int nb,
                                           uint64_t* __restrict__ out_key,
                                           uint32_t* __restrict__ out_m,
                                           unsigned long long* __restrict__ count, uint64_t cap) {
  const uint32_t* a = sv.row(ra);
  const uint32_t* b = sv.row(rb);
  const uint32_t allowed = H - min_match;
  uint32_t matches = 0, first = 0xFFFFFFFFu, pc;
  if (H >= 32 && (H & 3) == 0) {
    pc = 32;  // 16 independent 16-byte loads in flight
    uint4 x[8], y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      x[q] = __ldg(reinterpret_cast<const uint4*>(a) + q);
      y[q] = __ldg(reinterpret_cast<const uint4*>(b) + q);
    }
#pragma unroll
    for (int q = 7; q >= 0; --q) {  // descending, so `first` ends at the lowest match
      const bool e0 = x[q].x == y[q].x, e1 = x[q].y == y[q].y, e2 = x[q].z == y[q].z,
                 e3 = x[q].w == y[q].w;
      matches += e0 + e1 + e2 + e3;
      if (e3) first = 4 * q + 3;
      if (e2) first = 4 * q + 2;
      if (e1) first = 4 * q + 1;
      if (e0) first = 4 * q;
    }
  } else {
    pc = min(H, 32u);
    for (uint32_t h = 0; h < pc; ++h) {
      const bool e = __ldg(a + h) == __ldg(b + h);
      matches += e;
      if (e && first == 0xFFFFFFFFu) first = h;
    }
  }
  if (pc - matches > allowed) return;     // accepting count already unreachable
  // check each pair once per cell: at its FIRST matching position (this also
  // rejects fingerprint collisions: a pair chained at k without a[k] == b[k])
  if (k < pc) {
    if (first != k) return;
  } else {
    if (first != 0xFFFFFFFFu) return;     // matched inside the prefix already
    if (__ldg(a + k) != __ldg(b + k)) return;  // fingerprint collision
    for (uint32_t h = pc; h < k; ++h)
      if (__ldg(a + h) == __ldg(b + h)) return;
  }
  bool alive;
  const uint32_t m = full_matches(a, b, H, allowed, alive);
  if (alive && m >= min_match) emit(ra, rb, m, nb, out_key, out_m, count, cap);
  (void)P;
}

// DPT = documents per thread (join_max <= DPT * kJoinThreads)
template <int DPT>
__global__ void __launch_bounds__(kJoinThreads)
    k_join(const SigView sv, uint32_t H, const uint32_t* __restrict__ rows,
           const uint64_t* __restrict__ cell_start, const uint32_t* __restrict__ cell_len,
           uint32_t join_max, uint32_t tbits, uint32_t P, uint32_t min_match, int nb,
           uint64_t* __restrict__ out_key, uint32_t* __restrict__ out_m,
           unsigned long long* __restrict__ count, uint64_t cap) {
  extern __shared__ uint32_t jsm[];
  const uint32_t n = cell_len[blockIdx.x];
  if (n > join_max) return;  // big cells go to k_compare
  const uint32_t T = 1u << tbits;
  uint32_t* keys = jsm;                // T   (tag << 23 | value), tag 0 = empty
  uint32_t* head = keys + T;           // T   (tag << 16 | doc)
  uint32_t* next = head + T;           // join_max
  uint32_t* rowsm = next + join_max;   // join_max
  const uint64_t s = cell_start[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < n; i += kJoinThreads) rowsm[i] = rows[s + i];
  for (uint32_t i = threadIdx.x; i < T; i += kJoinThreads) {
    keys[i] = 0;
    head[i] = 0;
  }
  __syncthreads();
  const uint32_t mask = T - 1;
  const bool vec = (H & 3) == 0;
  for (uint32_t k0 = 0; k0 < P; k0 += 4) {
    // this thread's documents' values at positions k0..k0+3, loaded up front
    uint4 val[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const uint32_t d = threadIdx.x + j * kJoinThreads;
      if (d < n) {
        const uint32_t* r = sv.row(rowsm[d]) + k0;
        if (vec && k0 + 4 <= H)
          val[j] = __ldg(reinterpret_cast<const uint4*>(r));
        else
          val[j] = make_uint4(__ldg(r), k0 + 1 < H ? __ldg(r + 1) : 0u,
                              k0 + 2 < H ? __ldg(r + 2) : 0u, k0 + 3 < H ? __ldg(r + 3) : 0u);
      }
    }
#pragma unroll
    for (uint32_t dk = 0; dk < 4; ++dk) {
      const uint32_t k = k0 + dk;
      if (k >= P) break;
      const uint32_t tag = k + 1;
#pragma unroll
      for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x + j * kJoinThreads;
        if (d >= n) break;
        const uint32_t v = dk == 0 ? val[j].x : dk == 1 ? val[j].y : dk == 2 ? val[j].z : val[j].w;
        // keyed by a 23-bit fingerprint of the value (values are arbitrary
        // u32, compare.cpp:24-67); join_check re-verifies a[k] == b[k]
        const uint32_t fpv = (v * 0x9E3779B1u) ^ ((v * 0x85EBCA6Bu) >> 9);
        const uint32_t key = (tag << 23) | (fpv & 0x7FFFFFu);
        uint32_t h = (v * 0x9E3779B1u) >> (32 - tbits);
        for (;;) {
          const uint32_t cur = keys[h];
          if (cur == key) break;
          if ((cur >> 23) == tag) {  // another value of this position: probe on
            h = (h + 1) & mask;
            continue;
          }
          const uint32_t old = atomicCAS(&keys[h], cur, key);
          if (old == cur || old == key) break;
          // lost a race for this slot: look at it again
        }
        const uint32_t prev = atomicExch(&head[h], (tag << 16) | d);
        next[d] = (prev >> 16) == tag ? (prev & 0xFFFFu) : 0xFFFFFFFFu;
      }
      __syncthreads();
      for (uint32_t d = threadIdx.x; d < n; d += kJoinThreads)
        for (uint32_t e = next[d]; e != 0xFFFFFFFFu; e = next[e])
          join_check(sv, H, rowsm[d], rowsm[e], k, P, min_match, nb, out_key, out_m, count, cap);
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Pigeonhole hash join (the default for cells of up to kJoinMax documents).
//
// With A = H - min_matches allowed mismatches, take NB = A + 1 disjoint blocks
// of BW consecutive positions (NB * BW <= H).  An acceptable pair spoils at
// most A blocks, so it agrees on EVERY position of at least one block: the
// pairs worth counting are the pairs with an identical block k < NB.  Per
// block, one hash table keyed by a 23-bit fingerprint of the block's BW values
// chains the documents of the cell; each chained pair is checked by one
// thread -- block k really identical (fingerprints may collide), no identical
// block before k (so each pair is counted once per cell), then the exact
// early-exit count (oracle.cpp:81-92).  With BW = 1 this is the per-position
// join above; with BW = 4 a random pair shares a block with probability ~q^4
// instead of ~q per position (q = chance two minima coincide, ~1/3000 here),
// which removes almost all spurious candidates.
template <int BW>
__device__ __forceinline__ uint32_t block_fp(const uint32_t (&v)[BW]) {
  uint32_t h = 0x9E3779B9u;
#pragma unroll
  for (int t = 0; t < BW; ++t) {
    h = (h ^ v[t]) * 0x85EBCA6Bu;
    h ^= h >> 15;
  }
  return h & 0x7FFFFFu;
}

// Block fingerprints of every signature row, computed once per compare:
// fps[row * NB + k] = block_fp of block k.  The join then reads 4 bytes per
// (document, cell, block) instead of the block's BW values -- each document is
// in one cell per band, so its row would otherwise be gathered b times.
template <int BW>
__global__ void k_block_fps(const uint32_t* __restrict__ sig, uint64_t nrows, uint32_t H,
                            uint32_t NB, uint32_t* __restrict__ fps) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nrows * NB) return;
  const uint64_t row = i / NB;
  const uint32_t k = static_cast<uint32_t>(i % NB);
  uint32_t v[BW];
  load_block<BW>(sig + row * H + static_cast<uint64_t>(k) * BW, (H & 3) == 0, v);
  fps[i] = block_fp<BW>(v);
}

// Pairs of one cell already handled at an earlier block (open addressing over
// (d << 12 | e) + 1, d < e < kJoinMax).  A near-duplicate pair shares almost
// every block, so it is rediscovered in almost every block's chains; the set
// answers those rediscoveries from shared memory instead of re-reading two
// blocks of both rows from HBM.  Entries only go from empty to full, and a
// pair is inserted in an earlier phase (barrier-separated) than any lookup
// that must see it.
constexpr int kPsetProbes = 16;  // an entry lies within this many slots of its home
static_assert(kJoinMax <= 4096, "pair keys pack two 12-bit document indices");

__device__ __forceinline__ bool pset_has(const uint32_t* pset, uint32_t smask, uint32_t key) {
  uint32_t h = (key * 0x9E3779B1u) & smask;
  for (int probe = 0; probe < kPsetProbes; ++probe, h = (h + 1) & smask) {
    const uint32_t c = pset[h];
    if (c == key) return true;
    if (c == 0) return false;
  }
  return false;
}

__device__ __forceinline__ void pset_add(uint32_t* pset, uint32_t smask, uint32_t key,
                                         int* full) {
  uint32_t h = (key * 0x9E3779B1u) & smask;
  for (int probe = 0; probe < kPsetProbes; ++probe, h = (h + 1) & smask) {
    const uint32_t old = atomicCAS(&pset[h], 0u, key);
    if (old == 0 || old == key) return;
  }
  *full = 1;  // not recorded: later blocks fall back to the HBM check
}

template <int BW>
__device__ __forceinline__ void join_check_blocks(const SigView sv, uint32_t H,
                                                  uint32_t d, uint32_t e, const uint32_t* rowsm,
                                                  uint32_t k, bool vec, uint32_t* pset,
                                                  uint32_t smask, int* full, bool exact_set,
                                                  uint32_t min_match, int nb,
                                                  uint64_t* __restrict__ out_key,
                                                  uint32_t* __restrict__ out_m,
                                                  unsigned long long* __restrict__ count,
                                                  uint64_t cap, bool looked_up = false) {
  const uint32_t key = ((min(d, e) << 12) | max(d, e)) + 1u;
  // after an overflow the set is dropped (misses would probe long runs)
  if (!looked_up && exact_set && pset_has(pset, smask, key)) return;  // identical at an earlier block
  const uint32_t ra = rowsm[d], rb = rowsm[e];
  const uint32_t* a = sv.row(ra);
  const uint32_t* b = sv.row(rb);
  // with a complete set, absence proves no earlier block is identical (each
  // identical block j < k put the pair into block j's chains and the set);
  // without one (overflow, or ND_JOIN_PSET=0), check the earlier blocks in HBM
  if (!exact_set)
    for (uint32_t j = 0; j < k; ++j)
      if (same_block<BW>(a + j * BW, b + j * BW, vec)) return;
  if (!same_block<BW>(a + k * BW, b + k * BW, vec)) return;  // fingerprint collision
  if (exact_set) pset_add(pset, smask, key, full);
  bool alive;
  const uint32_t m = full_matches(a, b, H, H - min_match, alive);
  if (alive && m >= min_match) emit(ra, rb, m, nb, out_key, out_m, count, cap);
}

// a block defers its candidate checks when the previous block had at least
// this many (ND_JOIN_DEFER sets the queue size; 0 = never defer)
constexpr uint32_t kDeferMin = 64;

// TPB threads per CTA: 256, or 512 for big cells (twice the warps per SM at
// the same 2 CTAs per SM that their shared memory allows)
template <int DPT, int BW, int TPB>
__global__ void __launch_bounds__(TPB, TPB == 512 ? 2 : 8)
    k_join_blocks(const SigView sv, uint32_t H, const uint32_t* __restrict__ rows,
                  const uint64_t* __restrict__ cell_start, const uint32_t* __restrict__ cell_len,
                  uint32_t join_max, uint32_t tbits, uint32_t sbits, uint32_t NB,
                  uint32_t min_match, int nb, uint64_t* __restrict__ out_key,
                  uint32_t* __restrict__ out_m, unsigned long long* __restrict__ count,
                  uint64_t cap, bool two_barriers, uint32_t qcap,
                  bool use_fps, bool exch) {
  // VL values per document and group of BPL = VL / BW blocks: one 32-byte
  // sector (a 16-byte load would still move a whole sector), or 64 bytes
  // for the big-cell variant
  constexpr int VL = (TPB == 512 && BW >= 4) ? 16 : 8;
  constexpr int BPL = VL / BW;
  extern __shared__ uint32_t jsm[];
  __shared__ int pset_full;
  // candidates of a block (after the handled-pair filter) by block % 3: the
  // deferred-check queue's fill, and what decides whether the next block
  // defers (only when the previous block had many, e.g. clusters)
  __shared__ uint32_t qn[3];
  const uint32_t n = cell_len[blockIdx.x];
  if (n > join_max) return;  // big cells go to k_compare
  const uint32_t T = 1u << tbits;
  const uint32_t S = 1u << sbits;
  // keyed table: T keys (tag << 23 | fingerprint, tag 0 = empty); one chain
  // per slot (exch): the documents' fingerprints, double-buffered by parity
  const uint32_t KW = exch ? 2 * join_max : T;
  uint32_t* keys = jsm;                // KW
  uint32_t* head = keys + KW;          // T   (tag << 16 | doc)
  uint32_t* pset = head + T;           // S   handled pairs (pset_has / pset_add)
  uint32_t* rowsm = pset + S;          // join_max
  // chain links, double-buffered by block parity: the walk of block k reads
  // next[k & 1] while faster threads already insert block k + 1 into the
  // other half, so one barrier per block suffices (an insert of block k + 2
  // waits behind block k + 1's barrier, which every walker of k has passed)
  uint16_t* next2 = reinterpret_cast<uint16_t*>(rowsm + join_max);  // 2 x join_max (0xFFFF = end)
  // deferred checks (qcap > 0): the walk only queues the chained pairs the
  // handled-pair set does not answer; after a barrier the whole CTA drains
  // the queue, so the row reads of one block's candidates are spread over
  // every thread (many loads in flight) instead of gating the barrier behind
  // the few walkers that found candidates
  uint2* queue = reinterpret_cast<uint2*>(
      (reinterpret_cast<uintptr_t>(next2 + 2 * join_max) + 7) & ~uintptr_t{7});
  const uint64_t s = cell_start[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < n; i += TPB) rowsm[i] = rows[s + i];
  for (uint32_t i = threadIdx.x; i < KW; i += TPB) keys[i] = 0;
  for (uint32_t i = threadIdx.x; i < T; i += TPB) head[i] = 0;
  for (uint32_t i = threadIdx.x; i < S; i += TPB) pset[i] = 0;
  if (threadIdx.x == 0) {
    pset_full = 0;
    qn[0] = qn[1] = qn[2] = 0;
  }
  uint32_t kblock = 0;  // running block index (k) for the % 3 counters
  __syncthreads();
  const uint32_t mask = T - 1;
  const bool vec = (H & 3) == 0;
  for (uint32_t k0 = 0; k0 < NB; k0 += BPL) {
    // fingerprints of blocks k0 .. k0+BPL-1 of this thread's documents
    uint32_t fp[DPT][BPL];
    if (use_fps) {  // from the precomputed table (k_block_fps): 4 bytes per block
#pragma unroll
      for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x + j * TPB;
        if (d < n) {
          const uint32_t* f = sv.fp(rowsm[d]) + k0;
#pragma unroll
          for (int b = 0; b < BPL; ++b) fp[j][b] = k0 + b < NB ? __ldg(f + b) : 0u;
        }
      }
    }
    const uint32_t p0 = k0 * BW;
    const bool full = vec && p0 + VL <= H;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
      const uint32_t d = threadIdx.x + j * TPB;
      if (!use_fps && d < n) {
        const uint32_t* r = sv.row(rowsm[d]) + p0;
        uint32_t v[VL];
        if (full) {
          load_block<VL>(r, true, v);
        } else {
#pragma unroll
          for (int t = 0; t < VL; ++t) v[t] = p0 + t < H ? __ldg(r + t) : 0u;
        }
#pragma unroll
        for (int b = 0; b < BPL; ++b) {
          uint32_t w[BW];
#pragma unroll
          for (int t = 0; t < BW; ++t) w[t] = v[b * BW + t];
          fp[j][b] = block_fp<BW>(w);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < BPL; ++b) {
      const uint32_t k = k0 + b;
      if (k >= NB) continue;
      const uint32_t tag = k + 1;
      uint16_t* next = next2 + (k & 1) * join_max;
#pragma unroll
      for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x + j * TPB;
        if (d >= n) continue;  // (not break: keeps fp[][] in registers)
        uint32_t h = (fp[j][b] * 0x9E3779B1u) >> (32 - tbits);
        if (exch) {
          // one chain per slot, whatever the fingerprint: the walk skips the
          // chained documents whose fingerprint differs (kept in fpk)
          keys[(k & 1) * join_max + d] = fp[j][b];
        } else {
          const uint32_t key = (tag << 23) | fp[j][b];
          for (;;) {
            const uint32_t cur = keys[h];
            if (cur == key) break;
            if ((cur >> 23) == tag) {  // another fingerprint of this block: probe on
              h = (h + 1) & mask;
              continue;
            }
            const uint32_t old = atomicCAS(&keys[h], cur, key);
            if (old == cur || old == key) break;
          }
        }
        const uint32_t prev = atomicExch(&head[h], (tag << 16) | d);
        next[d] = (prev >> 16) == tag ? static_cast<uint16_t>(prev) : uint16_t{0xFFFF};
      }
      __syncthreads();
      const bool exact_set = S > 1 && *static_cast<volatile int*>(&pset_full) == 0;
      // qn[(k + 1) % 3] was last written in block k - 2's walk and read at
      // block k - 1's decision, both before this barrier: reset it for k + 1
      if (threadIdx.x == 0) qn[(kblock + 1) % 3] = 0;
      uint32_t* q = &qn[kblock % 3];
      const bool defer =
          qcap && kblock > 0 && *static_cast<volatile uint32_t*>(&qn[(kblock + 2) % 3]) >= kDeferMin;
      ++kblock;
      const uint32_t* fpk = keys + (k & 1) * join_max;
      if (defer) {
        for (uint32_t d = threadIdx.x; d < n; d += TPB)
          for (uint32_t e = next[d]; e != 0xFFFFu; e = next[e]) {
            if (exch && fpk[e] != fpk[d]) continue;
            if (exact_set && pset_has(pset, S - 1, ((min(d, e) << 12) | max(d, e)) + 1u)) continue;
            const uint32_t slot = atomicAdd(q, 1u);
            if (slot < qcap)
              queue[slot] = make_uint2(d, e);
            else  // queue full: check inline
              join_check_blocks<BW>(sv, H, d, e, rowsm, k, vec, pset, S - 1, &pset_full,
                                    exact_set, min_match, nb, out_key, out_m, count, cap, true);
          }
        __syncthreads();
        const uint32_t lim = min(*static_cast<volatile uint32_t*>(q), qcap);
        for (uint32_t i = threadIdx.x; i < lim; i += TPB) {
          const uint2 de = queue[i];
          join_check_blocks<BW>(sv, H, de.x, de.y, rowsm, k, vec, pset, S - 1, &pset_full,
                                exact_set, min_match, nb, out_key, out_m, count, cap, true);
        }
      } else {
        for (uint32_t d = threadIdx.x; d < n; d += TPB)
          for (uint32_t e = next[d]; e != 0xFFFFu; e = next[e]) {
            if (exch && fpk[e] != fpk[d]) continue;
            if (exact_set && pset_has(pset, S - 1, ((min(d, e) << 12) | max(d, e)) + 1u)) continue;
            if (qcap) atomicAdd(q, 1u);  // count: does the next block defer?
            join_check_blocks<BW>(sv, H, d, e, rowsm, k, vec, pset, S - 1, &pset_full, exact_set,
                                  min_match, nb, out_key, out_m, count, cap, true);
          }
      }
      if (two_barriers) __syncthreads();
    }
  }
}

using CmpFn = void (*)(SigView, uint32_t, const uint32_t*, const uint64_t*,
                       const uint32_t*, const uint32_t*, const uint64_t*, uint32_t, int,
                       uint64_t*, uint32_t*, unsigned long long*, uint64_t);

}  // namespace

void join_block_shape(uint32_t H, uint32_t min_match, uint32_t* NB, int* BW) {
  *NB = H - min_match + 1;  // A + 1 blocks
  *BW = 1;
  for (int w : {8, 4, 2})
    if (static_cast<uint64_t>(*NB) * w <= H) {
      *BW = w;
      break;
    }
}

void block_fingerprints(const uint32_t* sig, uint64_t nrows, uint32_t H, uint32_t NB, int BW,
                        uint32_t* fps, cudaStream_t s) {
  const uint64_t total = nrows * NB;
  if (!total) return;
  const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
  if (BW == 2) k_block_fps<2><<<blocks, 256, 0, s>>>(sig, nrows, H, NB, fps);
  else if (BW == 4) k_block_fps<4><<<blocks, 256, 0, s>>>(sig, nrows, H, NB, fps);
  else k_block_fps<8><<<blocks, 256, 0, s>>>(sig, nrows, H, NB, fps);
  ND_CHECK_LAUNCH();
}

// Smallest compiled prefilter width >= H - min_matches + 1 that fits in H.
int compare_prefilter_width(uint32_t H, uint32_t min_match) {
  const uint32_t P = H - min_match + 1;
  for (int pf : {16, 28, 32, 52, 64})
    if (static_cast<uint32_t>(pf) >= P && static_cast<uint32_t>(pf) <= H) return pf;
  return 0;
}

void launch_compare(CellSet& cs, const SigView& d_sig, uint32_t H, uint32_t min_match,
                    int nb, uint64_t* out_key, uint32_t* out_m, unsigned long long* count,
                    uint64_t cap, cudaStream_t s, uint64_t nrows) {
  if (cs.ncells == 0 || min_match > H) return;
  // cells of <= kJoinMax documents: hash join (one CTA per cell)
  const uint32_t P = H - min_match + 1;
  // the joins tag table entries with 9-bit block numbers; beyond kJoinMaxP
  // blocks every cell goes to the all-pairs kernel instead (K2 tiled the
  // join's cells with zero all-pairs tiles, so re-tile them first)
  if (P > kJoinMaxP && cs.join_enabled) cells_all_pairs_tiles(cs, s);
  const uint32_t join_max = static_cast<uint32_t>(std::min<uint64_t>(cs.max_len, kJoinMax));
  const char* jb = getenv("ND_JOIN_BLOCKS");  // read per call: tests switch it
  const int join_mode = jb && std::string(jb) == "0" ? 1 : 2;  // 2 = blocks, 1 = per position
  uint32_t NB = 0;
  int BW = 1;
  join_block_shape(H, min_match, &NB, &BW);
  if (cs.join_enabled && join_max >= 2 && P <= kJoinMaxP) {
    // table slots >= n / load; the default load 1/2 (ND_JOIN_LOAD = percent)
    // one chain per table slot, no key CAS loop (ND_JOIN_EXCH=0: the keyed
    // table with probing); -20..-29 % K3 (profiles/r2_k3_defer.txt).  Its
    // table may be fuller (a shared slot only lengthens a chain):
    // ND_JOIN_EXCH_LOAD percent, default 50 (100 / 200 measured 5 / 19 % slower)
    const char* je = getenv("ND_JOIN_EXCH");
    const bool exch = !(je && je[0] == '0');
    const char* jl = getenv("ND_JOIN_LOAD");  // keyed tables (k_join, keyed block join)
    const uint32_t load_pct = jl ? static_cast<uint32_t>(std::max(10, std::min(95, atoi(jl)))) : 50;
    uint32_t tbits = 4;
    while ((1ull << tbits) * load_pct < 100ull * join_max) ++tbits;
    uint32_t tbits_b = tbits;  // block join's table
    if (exch) {
      const char* xl = getenv("ND_JOIN_EXCH_LOAD");
      const uint32_t xpct = xl ? static_cast<uint32_t>(std::max(10, std::min(400, atoi(xl)))) : 50;
      tbits_b = 4;
      while ((1ull << tbits_b) * xpct < 100ull * join_max) ++tbits_b;
    }
    // handled-pair set of the block join: 2^sbits >= join_max / 2 slots
    // (overflow only costs the HBM checks of earlier blocks)
    const char* sd = getenv("ND_JOIN_PSET_DIV");  // tuning: slots >= join_max / div
    const uint32_t sdiv = sd ? std::max(1, atoi(sd)) : 2;
    uint32_t sbits = 8;
    while ((1u << sbits) < join_max / sdiv) ++sbits;
    const char* ps = getenv("ND_JOIN_PSET");  // 0: no set (HBM checks of earlier blocks)
    if (ps && ps[0] == '0') sbits = 0;
    const size_t smem = (2u * (1u << tbits) + 2u * join_max) * sizeof(uint32_t);
    // deferred-check queue (ND_JOIN_DEFER = entries, 0 = check in the walk).
    // Off by default: it halves K3's time on clustered cells (C5: 54.7 ->
    // 36.5 ms at 1024 entries) but its shared memory costs the uniform cells
    // of C2/C3 L1 capacity for the row gathers (C2 cells 5.1 -> 6.9 ms, even
    // at 128 entries; profiles/r2_k3_defer.txt)
    const char* jd = getenv("ND_JOIN_DEFER");
    const uint32_t qcap = jd ? static_cast<uint32_t>(std::max(0, atoi(jd))) : 0u;
    const size_t smem_b = ((exch ? 2u * join_max : (1u << tbits_b)) + (1u << tbits_b) +
                           (sbits ? 1u << sbits : 1u)) * sizeof(uint32_t) +
                          join_max * (sizeof(uint32_t) + 2 * sizeof(uint16_t)) +
                          (qcap ? 8 + qcap * sizeof(uint2) : 0);
    const char* tb = getenv("ND_JOIN_TWO_BARRIERS");  // 1: the barrier after each walk too
    const bool two_barriers = tb && tb[0] == '1';
    if (cs.ncells > 0x7FFFFFFFull) fail(ND_ERR_CONFIG, "too many cells");
    const unsigned grid = static_cast<unsigned>(cs.ncells);
    if (join_mode == 2 && BW > 1) {
      using JoinBFn = void (*)(SigView, uint32_t, const uint32_t*, const uint64_t*,
                               const uint32_t*, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t,
                               int, uint64_t*, uint32_t*, unsigned long long*, uint64_t, bool,
                               uint32_t, bool, bool);
      // block fingerprints of every row, once: computed here for a one-table
      // view; the multi-GPU paths hand in per-rank tables (sv.fp_bases)
      SigView sv = d_sig;
      const char* jf = getenv("ND_JOIN_FPS");  // 0: fingerprints from the rows in the join
      const bool fps_on = !(jf && jf[0] == '0');
      if (fps_on && sv.world <= 1 && nrows > 0 && nrows * NB < (1ull << 40)) {
        uint32_t* f = cs.fps.as<uint32_t>(nrows * NB);
        block_fingerprints(sv.base0, nrows, H, NB, BW, f, s);
        sv.fp0 = f;
        sv.fpNB = NB;
      }
      const bool use_fps = fps_on && sv.fpNB == NB && (sv.world <= 1 ? sv.fp0 != nullptr
                                                                       : sv.fp_bases != nullptr);
      // 512 threads per CTA for cells above 1024 documents: -33 % K3 time on
      // C3-sized cells; smaller cells are faster with 256
      const int tpb = join_max > 1024 ? 512 : 256;
      static_assert(8 * 512 >= kJoinMax, "k_join_blocks<8, *, 512> must cover kJoinMax");
      const int dpt = join_max <= 2u * tpb ? 2 : join_max <= 4u * tpb ? 4 : join_max <= 8u * tpb ? 8 : 16;
      JoinBFn fn = nullptr;
#define ND_JB(D, W, P) \
  if (dpt == D && BW == W && tpb == P) fn = k_join_blocks<D, W, P>;
      ND_JB(2, 2, 256) ND_JB(2, 4, 256) ND_JB(2, 8, 256) ND_JB(4, 2, 256) ND_JB(4, 4, 256)
      ND_JB(4, 8, 256) ND_JB(4, 2, 512) ND_JB(4, 4, 512) ND_JB(4, 8, 512) ND_JB(8, 2, 512)
      ND_JB(8, 4, 512) ND_JB(8, 8, 512)
#undef ND_JB
      if (smem_b > 48 * 1024)
        ND_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem_b)));
      fn<<<grid, tpb, smem_b, s>>>(sv, H, cs.sorted_rows, cs.cell_start, cs.cell_len,
                                   join_max, tbits_b, sbits, NB, min_match, nb, out_key, out_m,
                                   count, cap, two_barriers, qcap, use_fps, exch);
      ND_CHECK_LAUNCH();
    } else {
      using JoinFn = void (*)(SigView, uint32_t, const uint32_t*, const uint64_t*,
                              const uint32_t*, uint32_t, uint32_t, uint32_t, uint32_t, int,
                              uint64_t*, uint32_t*, unsigned long long*, uint64_t);
      JoinFn fn = join_max <= 2 * kJoinThreads   ? k_join<2>
                  : join_max <= 4 * kJoinThreads ? k_join<4>
                  : join_max <= 8 * kJoinThreads ? k_join<8>
                                                 : k_join<16>;
      static_assert(16 * kJoinThreads >= kJoinMax, "k_join<16> must cover kJoinMax");
      if (smem > 48 * 1024)
        ND_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
      fn<<<grid, kJoinThreads, smem, s>>>(d_sig, H, cs.sorted_rows, cs.cell_start, cs.cell_len,
                                          join_max, tbits, P, min_match, nb, out_key, out_m, count,
                                          cap);
      ND_CHECK_LAUNCH();
    }
  }
  if (cs.items == 0) return;  // no cell above kJoinMax
  CmpFn fn = nullptr;
  switch (compare_prefilter_width(H, min_match)) {
    case 16: fn = k_compare<16>; break;
    case 28: fn = k_compare<28>; break;
    case 32: fn = k_compare<32>; break;
    case 52: fn = k_compare<52>; break;
    case 64: fn = k_compare<64>; break;
    default: fn = k_compare<0>; break;
  }
  if (cs.items > 0x7FFFFFFFull) fail(ND_ERR_CONFIG, "too many compare work items");
  fn<<<static_cast<unsigned>(cs.items), kThreads, 0, s>>>(d_sig, H, cs.sorted_rows, cs.cell_start,
                                                       cs.cell_len, cs.item_cell, cs.item_off,
                                                       min_match, nb, out_key, out_m, count, cap);
  ND_CHECK_LAUNCH();
}

}  // namespace ndb
