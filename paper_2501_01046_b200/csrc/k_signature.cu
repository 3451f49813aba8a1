// K1: MinHash signatures + LSH band keys, one warp per work item.
//
// Replaces signature_of_document (minhash.cpp:133-162) and band_bucket_ids
// (lsh.cpp:42-60) as called by the hash stage (pipeline.cpp:214-218).
//
// Arithmetic.  For hash function (p, q) the window value is
//   h_w = sum_{i<L} c_{w+i} q^i mod p          (hash_window_direct, minhash.cpp:111-119)
// Any exact evaluation gives the same bits, and the signature is the min over
// windows, so we walk each work item BACKWARD with the Horner-shift recurrence
//   h_w = c_w + q*h_{w+1} - c_{w+L} q^L  (mod p)
// instead of the reference's forward Eq.5 update (minhash.cpp:121-131).  Per
// (window, function) it costs 8 single-issue integer instructions, split
// 4 fma-pipe / 4 alu-pipe:
//   A  = c_out*QLn + c_in            IMAD        QLn = (p - q^L mod p) mod p
//   u  = q*s + A          (64-bit)   IMAD.WIDE   u < 2^39 + 2^31
//   t  = u >> 8           (32-bit)   SHF
//   k  = hi32(t * M)                 IMAD.HI     M = floor(2^40 / p): k in {Q-1, Q}
//   r  = lo32(u) - k*p               IMAD        r in [0, 2p)
//   r' = min(r, r - p)  (unsigned)   IADD+IMNMX  canonical residue = next state s
//   sig = min(sig, r')               IMNMX
// The window state starts at 0 one position past the item's last character
// and is warmed up over L-1 partial windows (c_out = 0 beyond the item), so no
// separate direct evaluation of the first window is needed.
//
// Layout.  Lane l of the warp owns functions [l*F, l*F+F) of the padded
// family (Hp = 32*F, pad functions are copies of function 0 and never
// stored).  The item's characters are staged per warp in shared memory in
// chunks of kChunk windows and read back as broadcast LDS.U8 (2 per window,
// amortised over F functions).  Long documents are split into items of at
// most kSeg windows; their per-item minima meet through atomicMin and their
// band keys are computed by a follow-up pass.
#include "nd_internal.cuh"

namespace ndb {
namespace {

constexpr int kWarps = 8;           // warps per block
constexpr int kChunk = 512;         // windows staged per chunk
constexpr int kLMax = 64;           // max shingle length
constexpr int kBuf = kChunk + kLMax;
constexpr uint32_t kSeg = 8192;     // max windows per work item

struct FamPtrs {
  const uint32_t* q;
  const uint32_t* qln;
  const uint32_t* m;
  const uint32_t* negp;
};

// ---------------------------------------------------------------------------
// planning: per-document segment counts, short-document detection
__global__ void k_plan(const uint64_t* __restrict__ offsets, uint64_t n, uint32_t L,
                       uint32_t* __restrict__ seg_count, uint32_t* __restrict__ flags) {
  uint64_t d = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (d >= n) return;
  uint64_t len = offsets[d + 1] - offsets[d];
  uint32_t nseg = 1;
  if (len < L) {
    atomicOr(&flags[0], 1u);  // ShortDocumentError
  } else {
    uint64_t nwin = len - L + 1;
    uint64_t s = (nwin + kSeg - 1) / kSeg;
    nseg = static_cast<uint32_t>(s);
    if (s > 1) atomicAdd(&flags[1], 1u);  // multi-segment document count
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

// band keys from finished signature rows (multi-segment documents)
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
// one rolling step for all F functions of this lane
template <int F, bool kMin>
__device__ __forceinline__ void step(uint32_t cin, uint32_t cout, const uint32_t (&q)[F],
                                     const uint32_t (&qln)[F], const uint32_t (&m)[F],
                                     const uint32_t (&negp)[F], uint32_t (&s)[F],
                                     uint32_t (&mn)[F]) {
#pragma unroll
  for (int f = 0; f < F; ++f) {
    uint32_t a = cout * qln[f] + cin;
    uint64_t u = static_cast<uint64_t>(q[f]) * s[f] + a;
    uint32_t lo = static_cast<uint32_t>(u);
    uint32_t t = __funnelshift_r(lo, static_cast<uint32_t>(u >> 32), 8);
    uint32_t k = __umulhi(t, m[f]);
    uint32_t r = lo + k * negp[f];
    uint32_t r2 = r + negp[f];
    uint32_t c = min(r, r2);
    s[f] = c;
    if (kMin) mn[f] = min(mn[f], c);
  }
}

template <int F>
__global__ void __launch_bounds__(kWarps * 32)
    k_signature(const uint8_t* __restrict__ text, const uint64_t* __restrict__ offsets,
                const uint32_t* __restrict__ item_doc, const uint64_t* __restrict__ item_off,
                uint64_t n_items, FamPtrs fam, uint32_t L, uint32_t H, uint32_t bands,
                uint32_t rows, uint32_t K, uint32_t* __restrict__ sig,
                uint32_t* __restrict__ band) {
  __shared__ __align__(16) uint8_t sbuf[kWarps][kBuf];
  __shared__ __align__(16) uint32_t srow[kWarps][32 * F];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t item = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
  if (item >= n_items) return;

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
  const uint64_t we = min(ws + kSeg, nwin);
  const uint64_t e = we + L - 1;  // one past the last character this item reads
  const uint8_t* base = text + off;

  uint32_t q[F], qln[F], m[F], negp[F], s[F], mn[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    int idx = lane * F + f;
    q[f] = fam.q[idx];
    qln[f] = fam.qln[idx];
    m[f] = fam.m[idx];
    negp[f] = fam.negp[idx];
    s[f] = 0;
    mn[f] = 0xFFFFFFFFu;
  }

  uint8_t* buf = sbuf[warp];
  uint64_t p_hi = e;  // positions [p_lo, p_hi) handled per chunk, descending
  bool first = true;
  while (p_hi > ws) {
    const uint64_t p_lo = (p_hi - ws > kChunk) ? p_hi - kChunk : ws;
    const int cnt = static_cast<int>(p_hi - p_lo);
    // stage chars [p_lo, p_hi + L), zero beyond e (virtual characters)
    for (int j = lane; j < cnt + static_cast<int>(L); j += 32) {
      uint64_t pos = p_lo + j;
      buf[j] = pos < e ? base[pos] : 0;
    }
    __syncwarp();
    int j = cnt - 1;
    if (first) {
      // L-1 warm-up positions: partial windows, not part of the minimum
      for (int w = 0; w < static_cast<int>(L) - 1; ++w, --j)
        step<F, false>(buf[j], buf[j + L], q, qln, m, negp, s, mn);
      first = false;
    }
    // main positions, unrolled by 4
    for (; j >= 3; j -= 4) {
      uint32_t c0 = buf[j], o0 = buf[j + L];
      uint32_t c1 = buf[j - 1], o1 = buf[j - 1 + L];
      uint32_t c2 = buf[j - 2], o2 = buf[j - 2 + L];
      uint32_t c3 = buf[j - 3], o3 = buf[j - 3 + L];
      step<F, true>(c0, o0, q, qln, m, negp, s, mn);
      step<F, true>(c1, o1, q, qln, m, negp, s, mn);
      step<F, true>(c2, o2, q, qln, m, negp, s, mn);
      step<F, true>(c3, o3, q, qln, m, negp, s, mn);
    }
    for (; j >= 0; --j) step<F, true>(buf[j], buf[j + L], q, qln, m, negp, s, mn);
    __syncwarp();
    p_hi = p_lo;
  }

  uint32_t* out = sig + doc * H;
  if (multi) {
#pragma unroll
    for (int f = 0; f < F; ++f) {
      int idx = lane * F + f;
      if (idx < static_cast<int>(H)) atomicMin(out + idx, mn[f]);
    }
    return;
  }
  uint32_t* row = srow[warp];
  if ((H % 4) == 0 && (F % 4) == 0 && lane * F + F <= static_cast<int>(H)) {
#pragma unroll
    for (int f = 0; f < F; f += 4)
      *reinterpret_cast<uint4*>(out + lane * F + f) = make_uint4(mn[f], mn[f + 1], mn[f + 2], mn[f + 3]);
  } else {
#pragma unroll
    for (int f = 0; f < F; ++f)
      if (lane * F + f < static_cast<int>(H)) out[lane * F + f] = mn[f];
  }
  if (band == nullptr) return;
#pragma unroll
  for (int f = 0; f < F; ++f) row[lane * F + f] = mn[f];
  __syncwarp();
  for (uint32_t j = lane; j < bands; j += 32) {
    uint64_t sum = 0;
    for (uint32_t r = 0; r < rows; ++r) sum += row[j * rows + r];
    band[doc * bands + j] = K ? static_cast<uint32_t>(sum % K) : static_cast<uint32_t>(sum);
  }
}

template <int F>
void launch_k1(const DevFamily& fam, const uint8_t* d_bytes, const uint64_t* d_offsets,
               const uint32_t* item_doc, const uint64_t* item_off, uint64_t items, uint32_t bands,
               uint32_t rows, uint32_t K, uint32_t* d_sig, uint32_t* d_band, cudaStream_t s) {
  FamPtrs p{fam.q, fam.qln, fam.m, fam.negp};
  uint64_t blocks = (items + kWarps - 1) / kWarps;
  k_signature<F><<<static_cast<unsigned>(blocks), kWarps * 32, 0, s>>>(
      d_bytes, d_offsets, item_doc, item_off, items, p, fam.L, fam.H, bands, rows, K, d_sig,
      d_band);
  ND_CHECK_LAUNCH();
}

}  // namespace

void launch_signatures(const DevFamily& fam, const uint8_t* d_bytes, const uint64_t* d_offsets,
                       uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                       uint32_t* d_band, SigScratch& sc, cudaStream_t s, bool check_short,
                       const uint64_t* h_offsets) {
  if (n == 0) return;
  if (fam.L == 0 || fam.L > static_cast<uint32_t>(kLMax))
    fail(ND_ERR_CONFIG, "shingle length must be in [1, 64] on the GPU path");
  if (n > 0xFFFFFFFFull) fail(ND_ERR_CONFIG, "batch exceeds 2^32 documents");
  unsigned tb = 256;
  uint32_t hflags[4] = {0, 0, 0, 0};
  if (h_offsets) {  // host planning: only multi-item batches need the device plan
    for (uint64_t d = 0; d < n; ++d) {
      uint64_t len = h_offsets[d + 1] - h_offsets[d];
      if (len < fam.L) hflags[0] = 1;
      else if (len - fam.L + 1 > kSeg) ++hflags[1];
    }
    if (check_short && hflags[0]) fail(ND_ERR_SHORT, "a document has fewer units than the shingle length");
  }
  uint32_t* seg_count = nullptr;
  uint32_t* flags = nullptr;
  if (!h_offsets || hflags[1]) {
    seg_count = sc.seg_count.as<uint32_t>(n);
    flags = sc.flags.as<uint32_t>(4);
    ND_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(uint32_t), s));
    k_plan<<<static_cast<unsigned>((n + tb - 1) / tb), tb, 0, s>>>(d_offsets, n, fam.L, seg_count,
                                                                    flags);
    ND_CHECK_LAUNCH();
    ND_CUDA(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
    if (check_short && hflags[0]) fail(ND_ERR_SHORT, "a document has fewer units than the shingle length");
  }

  const uint32_t* item_doc = nullptr;
  const uint64_t* item_off = nullptr;
  uint64_t items = n;
  uint32_t nmulti = hflags[1];
  uint32_t* multi_docs = nullptr;
  if (nmulti) {
    uint64_t* off = sc.item_off.as<uint64_t>(n + 1);
    scan_u32_to_u64(seg_count, off, n, sc.scan_tmp, s);
    ND_CUDA(cudaMemcpyAsync(&items, off + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
    uint32_t* idoc = sc.item_doc.as<uint32_t>(items);
    multi_docs = sc.multi_docs.as<uint32_t>(nmulti + 1);
    uint32_t* counter = flags + 2;
    ND_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    k_item_scatter<<<static_cast<unsigned>((n + tb - 1) / tb), tb, 0, s>>>(off, n, idoc, multi_docs,
                                                                           counter);
    ND_CHECK_LAUNCH();
    k_fill_multi<<<1024, 256, 0, s>>>(multi_docs, nmulti, fam.H, d_sig);
    ND_CHECK_LAUNCH();
    item_doc = idoc;
    item_off = off;
  }
  switch (fam.Hp / 32) {
    case 1: launch_k1<1>(fam, d_bytes, d_offsets, item_doc, item_off, items, bands, rows, K, d_sig, d_band, s); break;
    case 2: launch_k1<2>(fam, d_bytes, d_offsets, item_doc, item_off, items, bands, rows, K, d_sig, d_band, s); break;
    case 4: launch_k1<4>(fam, d_bytes, d_offsets, item_doc, item_off, items, bands, rows, K, d_sig, d_band, s); break;
    case 8: launch_k1<8>(fam, d_bytes, d_offsets, item_doc, item_off, items, bands, rows, K, d_sig, d_band, s); break;
    case 16: launch_k1<16>(fam, d_bytes, d_offsets, item_doc, item_off, items, bands, rows, K, d_sig, d_band, s); break;
    default: fail(ND_ERR_CONFIG, "hash count must be at most 512 on the GPU path");
  }
  if (nmulti && d_band) {
    uint64_t total = static_cast<uint64_t>(nmulti) * bands;
    k_bands_from_rows<<<static_cast<unsigned>((total + tb - 1) / tb), tb, 0, s>>>(
        multi_docs, nmulti, d_sig, fam.H, bands, rows, K, d_band);
    ND_CHECK_LAUNCH();
  }
}

}  // namespace ndb
