// In-memory dedup driver (K1 -> K2 -> K3 -> K4) and the C-ABI of the compare,
// union and dedup stages.
//
// run_dedup (pipeline.cpp:510-532) chains three file-backed stages: hash
// (.feds files), gather-compare (.pairs files) and union.  Here the same
// stages run back to back on one device with every intermediate resident in
// HBM: signatures + band keys (K1), stable cell grouping (K2), in-cell
// comparison (K3), distinct pairs + components (K4).  Only the report leaves
// the device.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "nd_capi_impl.cuh"

namespace ndb {
namespace {

struct EventTimer {
  cudaEvent_t e[8];
  int n = 0;
  cudaStream_t s;
  explicit EventTimer(cudaStream_t st) : s(st) {
    for (auto& x : e) cudaEventCreate(&x);
  }
  ~EventTimer() {
    for (auto& x : e) cudaEventDestroy(x);
  }
  void mark() { cudaEventRecord(e[n++], s); }
  double seconds(int a, int b) {
    float ms = 0;
    cudaEventSynchronize(e[b]);
    cudaEventElapsedTime(&ms, e[a], e[b]);
    return ms / 1e3;
  }
};

}  // namespace

void validate(const nd_params& p) {
  // RunConfig::validate (pipeline.cpp:20-33), artifact-shaping fields
  if (p.bands == 0 || p.rows == 0) fail(ND_ERR_CONFIG, "bands and rows must be positive");
  if (static_cast<uint64_t>(p.bands) * p.rows != p.hash_count)
    fail(ND_ERR_CONFIG, "hash count " + std::to_string(p.hash_count) + " must equal bands*rows = " +
                            std::to_string(p.bands) + "*" + std::to_string(p.rows));
  if (p.shingle_len == 0) fail(ND_ERR_CONFIG, "shingle length must be positive");
  if (p.threshold_den == 0) fail(ND_ERR_CONFIG, "ratio denominator must be positive");
  if (p.threshold_num > p.threshold_den) fail(ND_ERR_CONFIG, "threshold must be at most 1");
  if (p.bucket_count == 0 && (p.scale_num == 0 || p.scale_den == 0))
    fail(ND_ERR_CONFIG, "bucket scale must be positive");
}

void ensure_family(nd_ctx* ctx, const nd_params& p) {
  const auto& fam = ctx->fam;
  if (fam.q && fam.H == p.hash_count && fam.L == p.shingle_len && fam.unit == p.unit &&
      ctx->family_seed == p.seed && ctx->family_derived)
    return;
  std::vector<nd_hash_fn> f = derive_family(p.seed, p.hash_count, p.shingle_len, p.unit);
  int rc = nd_family_upload(ctx, f.data(), p.hash_count, p.shingle_len, p.unit);
  if (rc != ND_OK) fail(rc, ctx->err);
  ctx->family_seed = p.seed;
  ctx->family_derived = true;
}

// compare + distinct pairs over a prepared CellSet (grows the pair buffer and
// re-runs once if the first pass overflowed it)
void compare_and_unique(DedupState& st, const uint32_t* d_sig, uint32_t H, uint32_t mm,
                        uint64_t nrows, cudaStream_t s) {
  compare_and_unique(st, SigView(d_sig, H), H, mm, nrows, s);
}

void compare_and_unique(DedupState& st, const SigView& d_sig, uint32_t H, uint32_t mm,
                        uint64_t nrows, cudaStream_t s) {
  compare_pairs(st, d_sig, H, mm, nrows, s);
  unique_pairs(st.pairs, s);
}

// K3 only: accepted pairs (with repeats across bands) into st.pairs
void compare_pairs(DedupState& st, const SigView& d_sig, uint32_t H, uint32_t mm, uint64_t nrows,
                   cudaStream_t s) {
  PairSet& ps = st.pairs;
  ps.nb = std::max(1, bits_for(nrows ? nrows - 1 : 0));
  if (2 * ps.nb > 64) fail(ND_ERR_CONFIG, "too many rows for packed pair keys");
  ps.counter = ps.dcount.as<unsigned long long>(1);
  if (ps.cap == 0) ps.cap = std::max<uint64_t>(1 << 20, 2 * nrows);
  for (int attempt = 0; attempt < 2; ++attempt) {
    ps.keys = ps.dkeys.as<uint64_t>(ps.cap);
    ps.vals = ps.dvals.as<uint32_t>(ps.cap);
    ND_CUDA(cudaMemsetAsync(ps.counter, 0, sizeof(unsigned long long), s));
    launch_compare(st.cells, d_sig, H, mm, ps.nb, ps.keys, ps.vals, ps.counter, ps.cap, s, nrows);
    unsigned long long got = 0;
    ND_CUDA(cudaMemcpyAsync(&got, ps.counter, sizeof got, cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
    ps.count = got;
    if (got <= ps.cap) break;
    ps.cap = got + got / 4;
  }
}

namespace {

template <class T>
std::vector<T> d2h(const T* d, uint64_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) ND_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  return h;
}

uint64_t id_of(const DedupState& st, uint32_t row) {
  return st.doc_ids.empty() ? row : st.doc_ids[row];
}

}  // namespace

// Host text -> device signatures/band keys: chunks (h2d_chunk_bytes) are copied
// on the h2d stream into a ring of chunk buffers and signed on the ctx stream
// as each lands (PCIe overlaps K1; the paper's double buffering).
namespace {
bool k1j_one_stream() {  // read per call (A/B runs in one process)
  const char* v = getenv("ND_K1J_STREAMS");
  return v && v[0] == '1';
}
}  // namespace

void h2d_signatures(nd_ctx* ctx, DedupState& st, const uint8_t* bytes, const uint64_t* offsets,
                    uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                    uint32_t* d_band) {
  if (n == 0) return;
  cudaStream_t s = ctx->stream;
  ctx->ensure_streams();
  const uint32_t H = ctx->fam.H;
  const uint32_t L = ctx->fam.L;
  if (offsets[n] < offsets[0])
    fail(ND_ERR_SHORT, "document offsets decrease: a document has fewer units than the shingle length");
  uint64_t* d_off = st.offs.as<uint64_t>(n + 1);
  uint64_t* h_off = static_cast<uint64_t*>(ctx->pinned_off.get((n + 1) * sizeof(uint64_t)));
  // chunks of <= h2d_chunk_bytes of text (a longer document is a chunk of its
  // own), bounds by binary search; each chunk's relative offsets are filled,
  // its documents checked and its offsets copied just before its text, so the
  // first copy waits for one chunk's host work, not the batch's
  std::vector<std::pair<uint64_t, uint64_t>> chunks;
  uint64_t max_bytes = 0;
  // gated K1j chunks (K1Gate, as in signatures_host) also ramp down at the end
  // (off by default here: C3 from host 3.452 s gated vs 3.451 s ungated, C2
  // 74.4 vs 73.2 ms; ND_K1J_RING_GATE=1 turns it on)
  const char* rg = getenv("ND_K1J_RING_GATE");
  const bool gated = ctx->gate_on() && !k1j_one_stream() && rg && rg[0] == '1';
  const uint64_t first_cap = h2d_chunk_bytes(ctx->fam, 0);
  for (uint64_t d0 = 0; d0 < n;) {
    uint64_t cap = h2d_chunk_bytes(ctx->fam, chunks.size());
    if (gated) cap = std::min(cap, std::max(first_cap, (offsets[n] - offsets[d0]) / 2));
    const uint64_t* it = std::upper_bound(offsets + d0 + 1, offsets + n + 1, offsets[d0] + cap);
    const uint64_t d1 = std::max<uint64_t>(d0 + 1, static_cast<uint64_t>(it - offsets) - 1);
    if (offsets[d1] < offsets[d0])
      fail(ND_ERR_SHORT, "document offsets decrease: a document has fewer units than the shingle length");
    chunks.push_back({d0, d1});
    max_bytes = std::max(max_bytes, offsets[d1] - offsets[d0]);
    d0 = d1;
  }
  // the text streams through a ring of kRing chunk buffers: only signatures
  // and band keys stay in HBM, so the batch is bounded by 4H+4b bytes per
  // document, not by its text.  Each slot has its own compute stream and K1
  // scratch, so consecutive chunks' K1 launches overlap and one launch's tail
  // (the longest documents of a lognormal chunk) does not idle the GPU.
  constexpr int kRing = 3;
  uint8_t* ring[kRing];
  for (int r = 0; r < kRing; ++r) ring[r] = ctx->ring[r].as<uint8_t>(max_bytes + 16);
  ctx->ensure_ring_streams();
  cudaEvent_t start, k1_done[kRing];
  ND_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  for (auto& e : k1_done) ND_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  ND_CUDA(cudaEventRecord(start, s));
  ND_CUDA(cudaStreamWaitEvent(ctx->h2d, start, 0));
  std::vector<cudaEvent_t> evs;
  auto drain_and_fail = [&](int code, const std::string& msg) {
    cudaStreamSynchronize(ctx->h2d);
    for (auto rs : ctx->ring_stream) cudaStreamSynchronize(rs);
    for (auto ev : evs) cudaEventDestroy(ev);
    for (auto e : k1_done) cudaEventDestroy(e);
    cudaEventDestroy(start);
    fail(code, msg);
  };
  for (size_t c = 0; c < chunks.size(); ++c) {
    const auto [d0, d1] = chunks[c];
    const int r = static_cast<int>(c % kRing);
    for (uint64_t i = d0; i < d1; ++i) {
      // (every document is checked before its chunk is signed; as before, a
      // decreasing offset reads as a short document)
      if (offsets[i + 1] < offsets[i] || offsets[i + 1] - offsets[i] < L)
        drain_and_fail(ND_ERR_SHORT, "document " + std::to_string(i) +
                                         " has fewer units than the shingle length");
    }
    for (uint64_t i = (c == 0 ? d0 : d0 + 1); i <= d1; ++i) h_off[i] = offsets[i] - offsets[0];
    ND_CUDA(cudaMemcpyAsync(d_off + d0, h_off + d0, (d1 - d0 + 1) * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, ctx->h2d));
    // (ND_K1J_STREAMS=1: K1j chunks on one stream; the ring's three streams
    // measured faster: C3 from host 3.45 vs 3.64 s, C2 73 vs 75 ms)
    const bool one = k1j_one_stream();
    cudaStream_t cs = (ctx->fam.jit && one) ? ctx->ring_stream[0] : ctx->ring_stream[r];
    if (c >= kRing) ND_CUDA(cudaStreamWaitEvent(ctx->h2d, k1_done[r], 0));  // slot free again
    ND_CUDA(cudaMemcpyAsync(ring[r], bytes + offsets[0] + h_off[d0], h_off[d1] - h_off[d0],
                            cudaMemcpyHostToDevice, ctx->h2d));
    cudaEvent_t ev;
    ND_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ND_CUDA(cudaEventRecord(ev, ctx->h2d));
    ND_CUDA(cudaStreamWaitEvent(cs, ev, 0));
    evs.push_back(ev);
    K1Gate gate_buf;
    K1Gate* gate = gated ? ctx->next_gate(gate_buf) : nullptr;
    if (gate && c > 0) k1_gate_wait(gate->flag, gate->epoch - 1, cs);
    // offsets stay batch-absolute: the kernel reads text + offset, so the
    // text pointer is the slot shifted back by the chunk's first offset
    launch_signatures(ctx->fam, ring[r] - h_off[d0], d_off + d0, d1 - d0, bands, rows, K,
                      d_sig + d0 * H, d_band ? d_band + d0 * bands : nullptr,
                      ctx->ring_scratch[r], cs, false, h_off + d0, gate);
    ND_CUDA(cudaEventRecord(k1_done[r], cs));
  }
  for (int r = 0; r < kRing; ++r) ND_CUDA(cudaStreamWaitEvent(s, k1_done[r], 0));
  // events may be destroyed once enqueued work referencing them is recorded
  for (auto ev : evs) cudaEventDestroy(ev);
  for (auto e : k1_done) cudaEventDestroy(e);
  cudaEventDestroy(start);
}

namespace {

// The shared tail of nd_dedup / nd_dedup_device: K2..K4 on the signatures and
// band keys already in st.sig / st.band.
void dedup_tail(nd_ctx* ctx, DedupState& st, const nd_params& p, uint64_t n, nd_dedup_stats* stats,
                EventTimer& t) {
  cudaStream_t s = ctx->stream;
  const uint32_t H = p.hash_count;
  const uint32_t mm = min_matches(H, p.threshold_num, p.threshold_den);
  const uint32_t* sig = st.sig.as<uint32_t>(n * H);
  const uint32_t* band = st.band.as<uint32_t>(n * p.bands);
  uint64_t emitted = 0;
  if (global_join_eligible(n, H, p.bands, st.K, mm)) {
    // K3g: the cells only for the reference's counters, every block joined
    // once over all rows (k_gjoin.cu)
    gj_cell_counts(st.gj, band, n, p.bands, st.K, s);
    t.mark();  // 2
    PairSet& ps = st.pairs;
    ps.nb = std::max(1, bits_for(n ? n - 1 : 0));
    ps.counter = ps.dcount.as<unsigned long long>(1);
    if (ps.cap == 0) ps.cap = std::max<uint64_t>(1 << 20, 2 * n);
    for (int attempt = 0; attempt < 2; ++attempt) {
      ps.keys = ps.dkeys.as<uint64_t>(ps.cap);
      ps.vals = ps.dvals.as<uint32_t>(ps.cap);
      ND_CUDA(cudaMemsetAsync(ps.counter, 0, sizeof(unsigned long long), s));
      gj_pairs(st.gj, sig, band, n, H, p.bands, mm, ps.nb, ps.keys, ps.vals, ps.counter, ps.cap, s);
      unsigned long long got = 0;
      ND_CUDA(cudaMemcpyAsync(&got, ps.counter, sizeof got, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
      ps.count = got;
      if (got <= ps.cap) break;
      ps.cap = got + got / 4;
    }
    t.mark();  // 3
    const GJoinCounts c = gj_read(st.gj, s);
    st.cells.ncells = c.ncells;
    st.cells.candidate_pairs = c.candidate_pairs;
    st.cells.cell_records = c.cell_records;
    emitted = c.emitted;
    st.compare_kind = "global";
  } else {
    build_cells_from_bands(st.cells, band, n, p.bands, st.K, kCmpRows, s);
    t.mark();  // 2
    compare_pairs(st, SigView(sig, H), H, mm, n, s);
    t.mark();  // 3
    emitted = st.pairs.count;
    st.compare_kind = "cells";
  }
  unique_pairs(st.pairs, s);
  t.mark();  // 4
  components(st.groups, st.pairs.lo, st.pairs.hi, st.pairs.distinct, n, s);
  t.mark();  // 5
  ND_CUDA(cudaStreamSynchronize(s));
  st.documents = n;
  st.bands = p.bands;
  st.H = H;
  st.valid = true;
  if (stats) {
    stats->documents = n;
    stats->bucket_count = st.K;
    stats->nonsingleton_cells = st.cells.ncells;
    stats->candidate_pairs = st.cells.candidate_pairs;
    stats->emitted_pairs = emitted;
    stats->distinct_pairs = st.pairs.distinct;
    stats->duplicate_groups = st.groups.groups;
    stats->near_duplicates = st.groups.members;
    stats->removals = st.groups.removals;
    stats->seconds[0] = t.seconds(0, 1);
    stats->seconds[1] = t.seconds(1, 2);
    stats->seconds[2] = t.seconds(2, 3);
    stats->seconds[3] = t.seconds(3, 4);
    stats->seconds[4] = t.seconds(4, 5);
    stats->seconds[5] = 0;
    stats->cell_records = st.cells.cell_records;
    stats->intervals = 1;
  }
}

// need: the bytes the caller is about to compare against the budget (the
// free-memory query is skipped when need is far below it)
uint64_t hbm_budget_of(nd_ctx* ctx, uint64_t need) {
  if (ctx->hbm_budget) return ctx->hbm_budget;
  return device_free_bytes(need, 7, 10) / 10 * 7;
}

// Device bytes of the in-memory dedup per document: signature + band ids +
// doc map, and per (document, band) record: key + row, their sort
// alternates and the cell CSR (the same estimate as the staged compare's
// interval plan, nd_stages.cu).
constexpr uint64_t kRecBytes = 8 * 4;
// (+ 4H: K3's block-fingerprint table, at most one u32 per signature value)
uint64_t row_bytes_of(const nd_params& p) { return 8ull * p.hash_count + 4ull * p.bands + 8; }

// Out-of-core in-memory dedup (plan_gather's idea, sigstore.cpp:288-329,
// applied to HBM instead of host RAM): when the signatures and cell records of
// the batch would not fit the HBM budget, K1 streams them back to host memory
// (nd_signatures' pipeline), the buckets are cut into intervals [k0, k1) whose
// documents + records fit, and each interval runs K2 + K3 on just the
// documents with a band bucket inside it and their in-range records.  Cells
// are (band, bucket), so every cell lies in exactly one interval: the
// candidate count is the sum over intervals, and the union of the intervals'
// accepted pairs, sorted + uniqued once more, is the single-pass pair set
// (a pair can be accepted in two intervals through two bands).
void dedup_out_of_core(nd_ctx* ctx, DedupState& st, const nd_params& p, const uint8_t* bytes,
                       const uint64_t* offsets, uint64_t n, uint64_t budget, nd_dedup_stats* stats) {
  using clk = std::chrono::steady_clock;
  auto sec = [](clk::time_point a) { return std::chrono::duration<double>(clk::now() - a).count(); };
  cudaStream_t s = ctx->stream;
  const uint32_t H = p.hash_count, B = p.bands, K = st.K;
  auto t0 = clk::now();
  st.host_sig.resize(n * H);
  st.host_band.resize(n * B);
  signatures_host(ctx, bytes, offsets, n, B, p.rows, K, st.host_sig.data(), st.host_band.data());
  const double t_sig = sec(t0);
  auto t1 = clk::now();
  const uint32_t* hband = st.host_band.data();
  std::vector<uint64_t> per_bucket(K, 0);
  for (uint64_t i = 0; i < n * B; ++i) ++per_bucket[hband[i]];
  const uint64_t row_bytes = row_bytes_of(p);
  std::vector<std::pair<uint32_t, uint32_t>> intervals;
  {
    uint32_t k0 = 0;
    uint64_t acc = 0;
    for (uint32_t k = 0; k < K; ++k) {
      const uint64_t bytes_k = per_bucket[k] * (row_bytes + kRecBytes);  // a record may bring its row
      if (k > k0 && acc + bytes_k > budget) {
        intervals.push_back({k0, k});
        k0 = k;
        acc = 0;
      }
      acc += bytes_k;
    }
    intervals.push_back({k0, K});
  }
  const uint32_t mm = min_matches(H, p.threshold_num, p.threshold_den);
  uint64_t candidates = 0, emitted = 0, cell_records = 0, ncells = 0;
  std::vector<uint32_t> all_lo, all_hi, all_m, sel, rkeys, rvals, gs, hl, hh, hm;
  double t_cells = 0, t_cmp = 0;
  for (auto [k0, k1] : intervals) {
    auto ta = clk::now();
    sel.clear();
    rkeys.clear();
    rvals.clear();
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t* bi = hband + i * B;
      bool any = false;
      for (uint32_t j = 0; j < B && !any; ++j) any = bi[j] >= k0 && bi[j] < k1;
      if (!any) continue;
      const uint32_t local = static_cast<uint32_t>(sel.size());
      sel.push_back(static_cast<uint32_t>(i));
      for (uint32_t j = 0; j < B; ++j)
        if (bi[j] >= k0 && bi[j] < k1) {
          rkeys.push_back(j * K + bi[j]);
          rvals.push_back(local);
        }
    }
    const uint64_t m = sel.size();
    if (m == 0) continue;
    gs.resize(m * H);
    for (uint64_t r = 0; r < m; ++r)
      std::memcpy(gs.data() + r * H, st.host_sig.data() + uint64_t(sel[r]) * H, 4ull * H);
    uint32_t* d_sig = st.sig.as<uint32_t>(m * H + 1);
    ND_CUDA(cudaMemcpyAsync(d_sig, gs.data(), m * H * 4, cudaMemcpyHostToDevice, s));
    const uint64_t nr = rkeys.size();
    uint32_t* dk = st.cells.rec_keys.as<uint32_t>(nr + 1);
    uint32_t* dv = st.cells.rec_vals.as<uint32_t>(nr + 1);
    ND_CUDA(cudaMemcpyAsync(dk, rkeys.data(), nr * 4, cudaMemcpyHostToDevice, s));
    ND_CUDA(cudaMemcpyAsync(dv, rvals.data(), nr * 4, cudaMemcpyHostToDevice, s));
    build_cells_from_records(st.cells, dk, dv, nr, uint64_t(B) * K, kCmpRows, s);
    ND_CUDA(cudaStreamSynchronize(s));
    auto tb = clk::now();
    t_cells += std::chrono::duration<double>(tb - ta).count();
    candidates += st.cells.candidate_pairs;
    cell_records += st.cells.cell_records;
    ncells += st.cells.ncells;
    compare_and_unique(st, SigView(d_sig, H), H, mm, m, s);
    emitted += st.pairs.count;
    const uint64_t d = st.pairs.distinct;
    hl.resize(d);
    hh.resize(d);
    hm.resize(d);
    if (d) {
      ND_CUDA(cudaMemcpyAsync(hl.data(), st.pairs.lo, d * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaMemcpyAsync(hh.data(), st.pairs.hi, d * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaMemcpyAsync(hm.data(), st.pairs.mc, d * 4, cudaMemcpyDeviceToHost, s));
    }
    ND_CUDA(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < d; ++i) {  // interval-local rows -> batch rows
      all_lo.push_back(sel[hl[i]]);
      all_hi.push_back(sel[hh[i]]);
      all_m.push_back(hm[i]);
    }
    t_cmp += sec(tb);
  }
  // the intervals' pairs -> one distinct set -> components over all rows
  auto t2 = clk::now();
  const uint64_t np = all_lo.size();
  uint32_t* d_lo = st.cells.rec_keys.as<uint32_t>(np + 1);
  uint32_t* d_hi = st.cells.rec_vals.as<uint32_t>(np + 1);
  uint32_t* d_m = st.cells.run_idx.as<uint32_t>(np + 1);
  if (np) {
    ND_CUDA(cudaMemcpyAsync(d_lo, all_lo.data(), np * 4, cudaMemcpyHostToDevice, s));
    ND_CUDA(cudaMemcpyAsync(d_hi, all_hi.data(), np * 4, cudaMemcpyHostToDevice, s));
    ND_CUDA(cudaMemcpyAsync(d_m, all_m.data(), np * 4, cudaMemcpyHostToDevice, s));
  }
  st.pairs.nb = std::max(1, bits_for(n - 1));
  pack_pairs(st.pairs, d_lo, d_hi, d_m, np, s);
  unique_pairs(st.pairs, s);
  ND_CUDA(cudaStreamSynchronize(s));
  const double t_uni = sec(t2);
  auto t3 = clk::now();
  components(st.groups, st.pairs.lo, st.pairs.hi, st.pairs.distinct, n, s);
  ND_CUDA(cudaStreamSynchronize(s));
  st.sig.release();  // the rows live in host memory
  st.sig_on_host = true;
  st.documents = n;
  st.bands = B;
  st.H = H;
  st.intervals = static_cast<uint32_t>(intervals.size());
  st.compare_kind = "cells";
  st.valid = true;
  if (stats) {
    *stats = nd_dedup_stats{};
    stats->documents = n;
    stats->bucket_count = K;
    stats->nonsingleton_cells = ncells;
    stats->candidate_pairs = candidates;
    stats->emitted_pairs = emitted;
    stats->distinct_pairs = st.pairs.distinct;
    stats->duplicate_groups = st.groups.groups;
    stats->near_duplicates = st.groups.members;
    stats->removals = st.groups.removals;
    stats->seconds[0] = t_sig;
    stats->seconds[1] = t_cells;
    stats->seconds[2] = t_cmp;
    stats->seconds[3] = t_uni;
    stats->seconds[4] = sec(t3);
    stats->cell_records = cell_records;
    stats->intervals = st.intervals;
  }
}

uint32_t bucket_count_for(const nd_params& p, uint64_t n) {
  return p.bucket_count ? p.bucket_count : choose_bucket_count(n, p.scale_num, p.scale_den);
}

void set_doc_ids(DedupState& st, const uint64_t* doc_ids, uint64_t n) {
  st.doc_ids.clear();
  if (!doc_ids) return;
  for (uint64_t i = 1; i < n; ++i)
    if (doc_ids[i] <= doc_ids[i - 1]) fail(ND_ERR_CONFIG, "doc_ids must be strictly ascending");
  st.doc_ids.assign(doc_ids, doc_ids + n);
}

}  // namespace
}  // namespace ndb

using namespace ndb;

extern "C" {

int nd_dedup(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, const uint64_t* doc_ids,
             uint64_t n, const nd_params* params, nd_dedup_stats* stats) {
  return guarded_impl(ctx, [&] {
    // ND_DEDUP_TRACE=1: host milliseconds of the call's phases on stderr
    const char* tr = getenv("ND_DEDUP_TRACE");
    const bool trace = tr && tr[0] == '1';
    const auto h0 = std::chrono::steady_clock::now();
    auto ms = [&] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
    };
    const nd_params p = *params;
    validate(p);
    if (is_group(ctx)) {  // sharded over the group's devices (nd_multi.cu)
      multi_dedup(ctx, bytes, offsets, doc_ids, n, p, stats);
      return;
    }
    ensure_family(ctx, p);
    const double f_ms = ms();
    DedupState& st = ctx->dedup;
    st.valid = false;
    set_doc_ids(st, doc_ids, n);
    if (n == 0) fail(ND_ERR_CONFIG, "no documents survive preprocessing; nothing to deduplicate");
    st.K = bucket_count_for(p, n);
    st.sig_on_host = false;
    st.host_sig.clear();
    st.host_band.clear();
    st.intervals = 1;
    const uint64_t need = n * row_bytes_of(p) + n * p.bands * kRecBytes;
    const uint64_t budget = hbm_budget_of(ctx, need);
    const double b_ms = ms();
    if (need > budget) {
      for (uint64_t i = 0; i < n; ++i)
        if (offsets[i + 1] < offsets[i] || offsets[i + 1] - offsets[i] < p.shingle_len)
          fail(ND_ERR_SHORT, "document " + std::to_string(i) + " has fewer units than the shingle length");
      dedup_out_of_core(ctx, st, p, bytes, offsets, n, budget, stats);
      return;
    }
    cudaStream_t s = ctx->stream;
    EventTimer t(s);
    t.mark();  // 0
    const double a = ms();
    h2d_signatures(ctx, st, bytes, offsets, n, p.bands, p.rows, st.K,
                   st.sig.as<uint32_t>(n * p.hash_count), st.band.as<uint32_t>(n * p.bands));
    const double b = ms();
    t.mark();  // 1
    dedup_tail(ctx, st, p, n, stats, t);
    if (trace)
      std::fprintf(stderr, "nd_dedup host ms: family %.2f, budget %.2f, timers %.2f, enqueue K1 %.2f, "
                   "tail (waits for K1) %.2f\n", f_ms, b_ms - f_ms, a - b_ms, b - a, ms() - b);
  });
}

int nd_signatures_h2d(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                      uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig, uint32_t* d_band) {
  return guarded_impl(ctx, [&] {
    ctx->require_family();
    if (d_band && (bands == 0 || rows == 0 || static_cast<uint64_t>(bands) * rows != ctx->fam.H))
      fail(ND_ERR_CONFIG, "banding shape does not match the hash count");
    h2d_signatures(ctx, ctx->h2d_state, bytes, offsets, n, bands, rows, K, d_sig, d_band);
    ND_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int nd_dedup_device(nd_ctx* ctx, const uint8_t* d_bytes, const uint64_t* d_offsets,
                    const uint64_t* doc_ids, uint64_t n, const nd_params* params,
                    nd_dedup_stats* stats) {
  return guarded_impl(ctx, [&] {
    if (is_group(ctx))
      fail(ND_ERR_CONFIG, "nd_dedup_device takes one device's buffers; use nd_dedup with host "
                          "buffers on a multi-device context");
    const nd_params p = *params;
    validate(p);
    ensure_family(ctx, p);
    DedupState& st = ctx->dedup;
    st.valid = false;
    set_doc_ids(st, doc_ids, n);
    if (n == 0) fail(ND_ERR_CONFIG, "no documents survive preprocessing; nothing to deduplicate");
    st.K = bucket_count_for(p, n);
    st.sig_on_host = false;
    st.host_sig.clear();
    st.host_band.clear();
    st.intervals = 1;
    cudaStream_t s = ctx->stream;
    EventTimer t(s);
    t.mark();
    launch_signatures(ctx->fam, d_bytes, d_offsets, n, p.bands, p.rows, st.K,
                      st.sig.as<uint32_t>(n * p.hash_count), st.band.as<uint32_t>(n * p.bands),
                      st.sig_scratch, s, true, nullptr);
    t.mark();
    dedup_tail(ctx, st, p, n, stats, t);
  });
}

int nd_dedup_signatures(nd_ctx* ctx, const uint32_t* sig, const uint32_t* band,
                        const uint64_t* doc_ids, uint64_t n, const nd_params* params,
                        nd_dedup_stats* stats) {
  return guarded_impl(ctx, [&] {
    if (is_group(ctx)) fail(ND_ERR_CONFIG, "nd_dedup_signatures runs on one device");
    const nd_params p = *params;
    validate(p);
    DedupState& st = ctx->dedup;
    st.valid = false;
    set_doc_ids(st, doc_ids, n);
    if (n == 0) fail(ND_ERR_CONFIG, "no documents survive preprocessing; nothing to deduplicate");
    st.K = bucket_count_for(p, n);
    for (uint64_t i = 0; i < n * p.bands; ++i)
      if (band[i] >= st.K)
        fail(ND_ERR_CONFIG, "band id " + std::to_string(band[i]) + " of row " +
                                std::to_string(i / p.bands) + " is not below the bucket count " +
                                std::to_string(st.K));
    st.sig_on_host = false;
    st.host_sig.clear();
    st.host_band.clear();
    st.intervals = 1;
    cudaStream_t s = ctx->stream;
    uint32_t* d_sig = st.sig.as<uint32_t>(n * p.hash_count);
    uint32_t* d_band = st.band.as<uint32_t>(n * p.bands);
    ND_CUDA(cudaMemcpyAsync(d_sig, sig, n * p.hash_count * 4, cudaMemcpyHostToDevice, s));
    ND_CUDA(cudaMemcpyAsync(d_band, band, n * p.bands * 4, cudaMemcpyHostToDevice, s));
    EventTimer t(s);
    t.mark();
    t.mark();  // (no K1)
    dedup_tail(ctx, st, p, n, stats, t);
  });
}

int nd_dedup_fetch_signatures(nd_ctx* ctx, uint32_t* sig, uint32_t* band) {
  return guarded_impl(ctx, [&] {
    if (is_group(ctx)) {
      multi_fetch_signatures(ctx, sig, band);
      return;
    }
    DedupState& st = ctx->dedup;
    if (!st.valid || !ctx->fam.q) fail(ND_ERR_PREREQ, "no dedup result; run nd_dedup first");
    cudaStream_t s = ctx->stream;
    const uint64_t n = st.documents, H = st.H;
    if (st.sig_on_host) {  // out-of-core run: rows in host memory
      if (sig && n) std::memcpy(sig, st.host_sig.data(), n * H * 4);
      if (band && n) std::memcpy(band, st.host_band.data(), n * st.bands * 4);
      return;
    }
    if (sig && n)
      ND_CUDA(cudaMemcpyAsync(sig, st.sig.ptr, n * H * 4, cudaMemcpyDeviceToHost, s));
    if (band && n)
      ND_CUDA(cudaMemcpyAsync(band, st.band.ptr, n * st.bands * 4, cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
  });
}

int nd_dedup_fetch_pairs(nd_ctx* ctx, uint64_t* lo, uint64_t* hi, uint32_t* match_count) {
  if (is_group(ctx)) {  // the group's result lives in shard 0's state
    const int rc = nd_dedup_fetch_pairs(ctx->shards[0], lo, hi, match_count);
    if (rc != ND_OK) ctx->err = ctx->shards[0]->err;
    return rc;
  }
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->dedup;
    if (!st.valid) fail(ND_ERR_PREREQ, "no dedup result; run nd_dedup first");
    cudaStream_t s = ctx->stream;
    const uint64_t d = st.pairs.distinct;
    auto l = d2h(st.pairs.lo, d, s);
    auto h = d2h(st.pairs.hi, d, s);
    auto m = d2h(st.pairs.mc, d, s);
    ND_CUDA(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < d; ++i) {
      if (lo) lo[i] = id_of(st, l[i]);
      if (hi) hi[i] = id_of(st, h[i]);
      if (match_count) match_count[i] = m[i];
    }
  });
}

int nd_dedup_fetch_groups(nd_ctx* ctx, uint64_t* members, uint64_t* group_start) {
  if (is_group(ctx)) {  // the group's result lives in shard 0's state
    const int rc = nd_dedup_fetch_groups(ctx->shards[0], members, group_start);
    if (rc != ND_OK) ctx->err = ctx->shards[0]->err;
    return rc;
  }
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->dedup;
    if (!st.valid) fail(ND_ERR_PREREQ, "no dedup result; run nd_dedup first");
    cudaStream_t s = ctx->stream;
    const GroupSet& g = st.groups;
    auto mem = d2h(g.member_rows, g.members, s);
    auto gs = d2h(g.group_start, g.groups ? g.groups + 1 : 0, s);
    ND_CUDA(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < g.members; ++i) members[i] = id_of(st, mem[i]);
    if (g.groups)
      std::memcpy(group_start, gs.data(), (g.groups + 1) * sizeof(uint64_t));
    else
      group_start[0] = 0;
  });
}

int nd_dedup_write_report(nd_ctx* ctx, const char* dir, uint64_t total_records) {
  return nd_dedup_write_report_ex(ctx, dir, total_records, 0);
}

int nd_dedup_write_report_ex(nd_ctx* ctx, const char* dir, uint64_t total_records,
                             int fsync_files) {
  if (is_group(ctx)) {
    const int rc = nd_dedup_write_report_ex(ctx->shards[0], dir, total_records, fsync_files);
    if (rc != ND_OK) ctx->err = ctx->shards[0]->err;
    return rc;
  }
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->dedup;
    if (!st.valid) fail(ND_ERR_PREREQ, "no dedup result; run nd_dedup first");
    cudaStream_t s = ctx->stream;
    const GroupSet& g = st.groups;
    auto mem = d2h(g.member_rows, g.members, s);
    auto gs = d2h(g.group_start, g.groups ? g.groups + 1 : 0, s);
    auto near = d2h(g.near, g.members, s);
    auto rem = d2h(g.removal, g.removals, s);
    ND_CUDA(cudaStreamSynchronize(s));
    std::vector<uint64_t> members(mem.size()), nearv(near.size()), remv(rem.size());
    for (size_t i = 0; i < mem.size(); ++i) members[i] = id_of(st, mem[i]);
    for (size_t i = 0; i < near.size(); ++i) nearv[i] = id_of(st, near[i]);
    for (size_t i = 0; i < rem.size(); ++i) remv[i] = id_of(st, rem[i]);
    write_report(dir, members, gs, nearv, remv, st.documents,
                 total_records ? total_records : st.documents, st.pairs.distinct,
                 fsync_files != 0);
  });
}

// ---- multi-GPU stage entry points (device pointers) -----------------------

int nd_stage_cell_records(nd_ctx* ctx, const uint32_t* d_band, uint64_t n, uint32_t bands,
                          uint32_t K, uint32_t doc_base, uint32_t* d_keys, uint32_t* d_vals) {
  return guarded_impl(ctx, [&] {
    if (bands == 0 || K == 0) fail(ND_ERR_CONFIG, "bands and bucket count must be positive");
    cudaStream_t s = ctx->stream;
    const uint64_t m = n * bands;
    make_records(d_band, n, bands, K, doc_base, d_keys, d_vals, s);
    radix_sort_u32(d_keys, d_vals, m, bits_for(static_cast<uint64_t>(bands) * K - 1),
                   ctx->stage_sort, s);
  });
}

int nd_stage_compare(nd_ctx* ctx, const uint32_t* d_sig, uint64_t nrows, uint32_t H,
                     const uint32_t* d_keys, const uint32_t* d_vals, uint64_t m, uint64_t key_limit,
                     uint64_t num, uint64_t den, uint64_t* npairs_out, uint64_t* cand_out) {
  return guarded_impl(ctx, [&] {
    if (H == 0) fail(ND_ERR_CONFIG, "hash count must be positive");
    if (den == 0) fail(ND_ERR_CONFIG, "ratio denominator must be positive");
    DedupState& st = ctx->api;
    cudaStream_t s = ctx->stream;
    st.valid = false;
    uint32_t* k = st.cells.rec_keys.as<uint32_t>(m + 1);
    uint32_t* v = st.cells.rec_vals.as<uint32_t>(m + 1);
    if (m) {
      ND_CUDA(cudaMemcpyAsync(k, d_keys, m * 4, cudaMemcpyDeviceToDevice, s));
      ND_CUDA(cudaMemcpyAsync(v, d_vals, m * 4, cudaMemcpyDeviceToDevice, s));
    }
    build_cells_from_records(st.cells, k, v, m, key_limit, kCmpRows, s);
    compare_and_unique(st, d_sig, H, min_matches(H, num, den), nrows, s);
    ND_CUDA(cudaStreamSynchronize(s));
    st.valid = true;
    *npairs_out = st.pairs.distinct;
    if (cand_out) *cand_out = st.cells.candidate_pairs;
  });
}

int nd_stage_pairs_copy(nd_ctx* ctx, uint32_t* d_lo, uint32_t* d_hi, uint32_t* d_match) {
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->api;
    if (!st.valid) fail(ND_ERR_PREREQ, "no compare result; run nd_stage_compare first");
    cudaStream_t s = ctx->stream;
    const uint64_t d = st.pairs.distinct;
    if (d) {
      ND_CUDA(cudaMemcpyAsync(d_lo, st.pairs.lo, d * 4, cudaMemcpyDeviceToDevice, s));
      ND_CUDA(cudaMemcpyAsync(d_hi, st.pairs.hi, d * 4, cudaMemcpyDeviceToDevice, s));
      ND_CUDA(cudaMemcpyAsync(d_match, st.pairs.mc, d * 4, cudaMemcpyDeviceToDevice, s));
    }
  });
}

int nd_stage_union(nd_ctx* ctx, const uint32_t* d_lo, const uint32_t* d_hi, const uint32_t* d_match,
                   uint64_t npairs, uint64_t nnodes, nd_dedup_stats* stats) {
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->dedup;
    cudaStream_t s = ctx->stream;
    st.valid = false;
    st.doc_ids.clear();
    st.pairs.nb = std::max(1, bits_for(nnodes ? nnodes - 1 : 0));
    if (2 * st.pairs.nb > 64) fail(ND_ERR_CONFIG, "too many rows for packed pair keys");
    pack_pairs(st.pairs, d_lo, d_hi, d_match, npairs, s);
    unique_pairs(st.pairs, s);
    components(st.groups, st.pairs.lo, st.pairs.hi, st.pairs.distinct, nnodes, s);
    ND_CUDA(cudaStreamSynchronize(s));
    st.documents = nnodes;
    st.valid = true;
    if (stats) {
      *stats = nd_dedup_stats{};
      stats->documents = nnodes;
      stats->emitted_pairs = npairs;
      stats->distinct_pairs = st.pairs.distinct;
      stats->duplicate_groups = st.groups.groups;
      stats->near_duplicates = st.groups.members;
      stats->removals = st.groups.removals;
    }
  });
}

// ---- stage entry points over caller-provided signatures / cells / pairs -----

int nd_band_keys(nd_ctx* ctx, const uint32_t* sigs, uint64_t n, uint32_t H, uint32_t bands,
                 uint32_t rows, uint32_t K, uint32_t* band_out) {
  return guarded_impl(ctx, [&] {
    // band_bucket_ids' shape checks (lsh.cpp:45-51)
    if (bands == 0 || rows == 0) fail(ND_ERR_CONFIG, "bands and rows must be positive");
    if (static_cast<uint64_t>(bands) * rows != H)
      fail(ND_ERR_CONFIG, "signature has " + std::to_string(H) + " values, banding needs " +
                              std::to_string(bands) + "*" + std::to_string(rows));
    if (n == 0) return;
    DedupState& st = ctx->api;
    cudaStream_t s = ctx->stream;
    uint32_t* d_sig = st.sig.as<uint32_t>(n * H);
    uint32_t* d_band = st.band.as<uint32_t>(n * bands);
    uint32_t* d_docs = st.cells.rec_vals.as<uint32_t>(n);
    ND_CUDA(cudaMemcpyAsync(d_sig, sigs, n * H * 4, cudaMemcpyHostToDevice, s));
    launch_band_keys(d_sig, n, H, bands, rows, K, d_band, d_docs, s);
    ND_CUDA(cudaMemcpyAsync(band_out, d_band, n * bands * 4, cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
  });
}

int nd_compare_cells(nd_ctx* ctx, const uint32_t* sigs, uint64_t nrows, uint32_t H,
                     const uint64_t* cell_offsets, const uint32_t* cell_rows, uint64_t ncells,
                     uint64_t num, uint64_t den, uint64_t* npairs_out) {
  return guarded_impl(ctx, [&] {
    if (H == 0) fail(ND_ERR_CONFIG, "hash count must be positive");
    if (den == 0) fail(ND_ERR_CONFIG, "ratio denominator must be positive");
    DedupState& st = ctx->api;
    cudaStream_t s = ctx->stream;
    st.valid = false;
    const uint64_t total = ncells ? cell_offsets[ncells] : 0;
    for (uint64_t c = 0; c < ncells; ++c) {
      if (cell_offsets[c + 1] < cell_offsets[c]) fail(ND_ERR_CONFIG, "cell offsets must ascend");
      for (uint64_t k = cell_offsets[c]; k < cell_offsets[c + 1]; ++k) {
        if (cell_rows[k] >= nrows) fail(ND_ERR_CONFIG, "cell row out of range");
        if (k > cell_offsets[c] && cell_rows[k] <= cell_rows[k - 1])
          fail(ND_ERR_CONFIG, "rows inside a cell must ascend");
      }
    }
    uint32_t* d_sig = st.sig.as<uint32_t>(nrows * H + 1);
    if (nrows) ND_CUDA(cudaMemcpyAsync(d_sig, sigs, nrows * H * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    // cells as records: key = cell index, value = row; stable grouping keeps the order
    std::vector<uint32_t> keys(total), vals(cell_rows, cell_rows + total);
    for (uint64_t c = 0; c < ncells; ++c)
      for (uint64_t k = cell_offsets[c]; k < cell_offsets[c + 1]; ++k) keys[k] = static_cast<uint32_t>(c);
    uint32_t* dk = st.cells.rec_keys.as<uint32_t>(total + 1);
    uint32_t* dv = st.cells.rec_vals.as<uint32_t>(total + 1);
    if (total) {
      ND_CUDA(cudaMemcpyAsync(dk, keys.data(), total * 4, cudaMemcpyHostToDevice, s));
      ND_CUDA(cudaMemcpyAsync(dv, vals.data(), total * 4, cudaMemcpyHostToDevice, s));
    }
    build_cells_from_records(st.cells, dk, dv, total, ncells ? ncells : 1, kCmpRows, s);
    compare_and_unique(st, d_sig, H, min_matches(H, num, den), nrows, s);
    ND_CUDA(cudaStreamSynchronize(s));
    st.doc_ids.clear();
    st.documents = nrows;
    st.valid = true;
    *npairs_out = st.pairs.distinct;
  });
}

int nd_pairs_fetch(nd_ctx* ctx, uint32_t* lo, uint32_t* hi, uint32_t* match_count) {
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->api;
    if (!st.valid) fail(ND_ERR_PREREQ, "no compare result; run nd_compare_cells first");
    cudaStream_t s = ctx->stream;
    const uint64_t d = st.pairs.distinct;
    if (d) {
      if (lo) ND_CUDA(cudaMemcpyAsync(lo, st.pairs.lo, d * 4, cudaMemcpyDeviceToHost, s));
      if (hi) ND_CUDA(cudaMemcpyAsync(hi, st.pairs.hi, d * 4, cudaMemcpyDeviceToHost, s));
      if (match_count) ND_CUDA(cudaMemcpyAsync(match_count, st.pairs.mc, d * 4, cudaMemcpyDeviceToHost, s));
    }
    ND_CUDA(cudaStreamSynchronize(s));
  });
}

int nd_union(nd_ctx* ctx, const uint32_t* lo, const uint32_t* hi, uint64_t npairs, uint32_t nnodes,
             uint64_t* nmembers_out, uint64_t* ngroups_out) {
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->api2;
    cudaStream_t s = ctx->stream;
    st.valid = false;
    for (uint64_t i = 0; i < npairs; ++i)
      if (lo[i] >= nnodes || hi[i] >= nnodes) fail(ND_ERR_CONFIG, "pair endpoint out of range");
    uint32_t* dlo = st.pairs.dlo.as<uint32_t>(npairs + 1);
    uint32_t* dhi = st.pairs.dhi.as<uint32_t>(npairs + 1);
    if (npairs) {
      ND_CUDA(cudaMemcpyAsync(dlo, lo, npairs * 4, cudaMemcpyHostToDevice, s));
      ND_CUDA(cudaMemcpyAsync(dhi, hi, npairs * 4, cudaMemcpyHostToDevice, s));
    }
    components(st.groups, dlo, dhi, npairs, nnodes, s);
    ND_CUDA(cudaStreamSynchronize(s));
    st.valid = true;
    *nmembers_out = st.groups.members;
    *ngroups_out = st.groups.groups;
  });
}

int nd_groups_fetch(nd_ctx* ctx, uint32_t* members, uint64_t* group_start) {
  return guarded_impl(ctx, [&] {
    DedupState& st = ctx->api2;
    if (!st.valid) fail(ND_ERR_PREREQ, "no union result; run nd_union first");
    cudaStream_t s = ctx->stream;
    const GroupSet& g = st.groups;
    if (g.members) ND_CUDA(cudaMemcpyAsync(members, g.member_rows, g.members * 4, cudaMemcpyDeviceToHost, s));
    if (g.groups)
      ND_CUDA(cudaMemcpyAsync(group_start, g.group_start, (g.groups + 1) * 8, cudaMemcpyDeviceToHost, s));
    else
      group_start[0] = 0;
    ND_CUDA(cudaStreamSynchronize(s));
  });
}

}  // extern "C"
