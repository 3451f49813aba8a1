// Multi-GPU behind the C-ABI: one nd_ctx over several devices, one host
// thread per shard (the reference's in-process parallel compare,
// pipeline.cpp:387-420, and band_partition, lsh.cpp:62-72, generalised to
// cell ranges over GPUs).
//
// nd_dedup on a group context:
//   A. every shard signs a contiguous, byte-balanced range of the batch (its
//      own H2D ring + K1, K from the GLOBAL document count, pipeline.cpp:300)
//      and stably partitions its (document, band) records by owner -- one
//      radix digit; the cell owner is floor(cell * G / (bands * K)), the
//      inverse of nd_cell_partition;
//   B. the all-to-all is fused into that partition's scatter: each record is
//      formed from its band id and stored straight into its owner's receive
//      buffer (peer stores over NVLink/NVSwitch), at the owner's offset for
//      the source -- source order s = 0..G-1, then document order, so each
//      cell's rows stay ascending as scan_gather requires
//      (sigstore.cpp:259-262).  Each owner then builds its cells (K2, the
//      only full sort of the records) and compares them (K3) reading every
//      signature row in place from the GPU that computed it, through a
//      SigView over the G shards' row arrays;
//   C. the shards' distinct pairs are gathered on shard 0 over peer copies,
//      sorted + uniqued once more and clustered (K4).
// Outputs are identical for any shard count (the union of pairs is
// order-free and every cell lies on exactly one owner).  Several shards may
// share a device (the loopback used to test the exchange on one GPU).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "nd_capi_impl.cuh"

namespace ndb {
namespace {

__global__ void k_owner_splits(const uint32_t* __restrict__ keys, uint64_t m,
                               const uint64_t* __restrict__ first_cell, uint32_t G,
                               uint64_t* __restrict__ split) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > G) return;
  // lower_bound(keys, first_cell[g]) over the cell-sorted records
  const uint64_t target = first_cell[g];
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1; else hi = mid;
  }
  split[g] = lo;
}

// owner of each (document, band) record, and its index: the key/value pair of
// the one-digit stable partition by owner.  owner(cell) = floor(cell * G /
// cells) is the inverse of nd_cell_partition's first_cell = ceil(cells * o / G)
__global__ void k_owner_keys(const uint32_t* __restrict__ band, uint64_t m, uint32_t bands,
                             uint32_t K, uint64_t cells, uint32_t G, uint32_t* __restrict__ keys,
                             uint32_t* __restrict__ vals) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t cell = static_cast<uint64_t>(i % bands) * K + band[i];
    keys[i] = static_cast<uint32_t>(cell * G / cells);
    vals[i] = static_cast<uint32_t>(i);
  }
}

// The exchange itself, fused into the partition's scatter: record p of the
// owner-sorted order goes straight into its owner's receive buffer (a peer
// store over NVLink when the owner is another GPU), at the owner's offset
// for this source plus the record's rank among this source's records for
// that owner -- source order, then document order, as scan_gather's rows.
struct OwnerDst {
  uint32_t* keys[64];
  uint32_t* vals[64];
  uint64_t base[64];   // this source's first slot in each owner's buffer
  uint64_t start[65];  // where each owner's run starts in the sorted order
};
__global__ void k_scatter_owners(const uint32_t* __restrict__ okeys,
                                 const uint32_t* __restrict__ oidx, uint64_t m,
                                 const uint32_t* __restrict__ band, uint32_t bands, uint32_t K,
                                 uint32_t doc_base, const OwnerDst* __restrict__ dst) {
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < m;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t o = okeys[p], i = oidx[p];
    const uint64_t q = dst->base[o] + (p - dst->start[o]);
    dst->keys[o][q] = (i % bands) * K + band[i];
    dst->vals[o][q] = doc_base + i / bands;
  }
}

// runs fn(shard index) on one host thread per shard; rethrows the first error
void run_shards(nd_ctx* g, const std::function<void(uint32_t)>& fn) {
  const uint32_t G = static_cast<uint32_t>(g->shards.size());
  std::vector<std::thread> th;
  std::mutex mu;
  int code = ND_OK;
  std::string msg;
  for (uint32_t s = 0; s < G; ++s)
    th.emplace_back([&, s] {
      try {
        ND_CUDA(cudaSetDevice(g->shards[s]->device));
        fn(s);
      } catch (const NdError& e) {
        std::lock_guard<std::mutex> l(mu);
        if (code == ND_OK) { code = e.code; msg = e.what(); }
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> l(mu);
        if (code == ND_OK) { code = ND_ERR_INTERNAL; msg = e.what(); }
      }
    });
  for (auto& t : th) t.join();
  if (code != ND_OK) fail(code, msg);
}

// contiguous document ranges balanced by text bytes
std::vector<uint64_t> shard_ranges(const uint64_t* offsets, uint64_t n, uint32_t G) {
  std::vector<uint64_t> r(G + 1, n);
  r[0] = 0;
  const uint64_t total = offsets[n] - offsets[0];
  for (uint32_t s = 1; s < G; ++s) {
    const uint64_t want = offsets[0] + total / G * s;
    r[s] = static_cast<uint64_t>(std::lower_bound(offsets, offsets + n, want) - offsets);
    r[s] = std::max(r[s], r[s - 1]);
  }
  return r;
}

double since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count();
}

}  // namespace

bool is_group(const nd_ctx* ctx) { return ctx && !ctx->shards.empty(); }

void multi_family_upload(nd_ctx* g, const nd_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit) {
  run_shards(g, [&](uint32_t s) {
    const int rc = nd_family_upload(g->shards[s], fns, H, L, unit);
    if (rc != ND_OK) fail(rc, g->shards[s]->err);
  });
}

void multi_signatures(nd_ctx* g, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                      uint32_t bands, uint32_t rows, uint32_t K, uint32_t* sig_out,
                      uint32_t* band_out) {
  const uint32_t G = static_cast<uint32_t>(g->shards.size());
  const uint32_t H = g->shards[0]->fam.H;
  const auto r = shard_ranges(offsets, n, G);
  run_shards(g, [&](uint32_t s) {
    const uint64_t d0 = r[s], m = r[s + 1] - r[s];
    if (m == 0) return;
    signatures_host(g->shards[s], bytes, offsets + d0, m, bands, rows, K, sig_out + d0 * H,
                    band_out ? band_out + d0 * bands : nullptr);
  });
}

// C (both compares): the owners' distinct pairs gathered on shard 0 over peer
// copies, sorted + uniqued once more, components (K4); stats
void multi_finish(nd_ctx* g, const std::vector<uint64_t>& r, const uint64_t* doc_ids, uint64_t n,
                  uint32_t B, uint32_t K, nd_dedup_stats* stats, const std::vector<double>& t_k1,
                  double sec_a, double sec_b, uint64_t ncells, uint64_t cand, uint64_t crec,
                  uint64_t emitted, const char* kind) {
  // ---- C: the pairs of every owner -> shard 0, distinct + components ----------
  const uint32_t G = static_cast<uint32_t>(g->shards.size());
  auto tc = std::chrono::steady_clock::now();
  nd_ctx* c0 = g->shards[0];
  ND_CUDA(cudaSetDevice(c0->device));
  DedupState& st0 = c0->dedup;
  cudaStream_t s0 = c0->stream;
  uint64_t np = 0;
  for (uint32_t s = 0; s < G; ++s) np += g->shards[s]->dedup.pairs.distinct;
  uint32_t* glo = c0->multi.pair_lo.as<uint32_t>(np + 1);
  uint32_t* ghi = c0->multi.pair_hi.as<uint32_t>(np + 1);
  uint32_t* gm = c0->multi.pair_m.as<uint32_t>(np + 1);
  for (uint32_t s = 0, at = 0; s < G; ++s) {
    const PairSet& ps = g->shards[s]->dedup.pairs;
    if (!ps.distinct) continue;
    const int dev = g->shards[s]->device;
    ND_CUDA(cudaMemcpyPeerAsync(glo + at, c0->device, ps.lo, dev, ps.distinct * 4, s0));
    ND_CUDA(cudaMemcpyPeerAsync(ghi + at, c0->device, ps.hi, dev, ps.distinct * 4, s0));
    ND_CUDA(cudaMemcpyPeerAsync(gm + at, c0->device, ps.mc, dev, ps.distinct * 4, s0));
    at += static_cast<uint32_t>(ps.distinct);
  }
  PairSet& fin = c0->multi.final_pairs;
  fin.nb = std::max(1, bits_for(n - 1));
  pack_pairs(fin, glo, ghi, gm, np, s0);
  unique_pairs(fin, s0);
  components(st0.groups, fin.lo, fin.hi, fin.distinct, n, s0);
  ND_CUDA(cudaStreamSynchronize(s0));
  // the result lives in shard 0's state (pairs, groups) -- the fetch calls of
  // the group context read it there
  std::swap(st0.pairs, fin);
  st0.doc_ids.clear();
  if (doc_ids) st0.doc_ids.assign(doc_ids, doc_ids + n);
  st0.documents = n;
  st0.bands = B;
  st0.K = K;
  st0.intervals = 1;
  st0.valid = true;
  g->multi.ranges = r;
  g->multi.last_valid = true;
  const double sec_c = since(tc);
  st0.compare_kind = kind;
  if (stats) {
    *stats = nd_dedup_stats{};
    stats->documents = n;
    stats->bucket_count = K;
    stats->nonsingleton_cells = ncells;
    stats->candidate_pairs = cand;
    stats->emitted_pairs = emitted;
    stats->cell_records = crec;
    stats->distinct_pairs = st0.pairs.distinct;
    stats->duplicate_groups = st0.groups.groups;
    stats->near_duplicates = st0.groups.members;
    stats->removals = st0.groups.removals;
    // wall clock per phase (max over shards): signatures, records + exchange
    // setup, exchange + K2 + K3, gather + K4
    stats->seconds[0] = *std::max_element(t_k1.begin(), t_k1.end());
    stats->seconds[1] = sec_a - stats->seconds[0];
    stats->seconds[2] = sec_b;
    stats->seconds[3] = 0;
    stats->seconds[4] = sec_c;
    stats->intervals = 1;
  }
}

void multi_dedup(nd_ctx* g, const uint8_t* bytes, const uint64_t* offsets,
                 const uint64_t* doc_ids, uint64_t n, const nd_params& p, nd_dedup_stats* stats) {
  const uint32_t G = static_cast<uint32_t>(g->shards.size());
  const uint32_t H = p.hash_count, B = p.bands;
  if (n == 0) fail(ND_ERR_CONFIG, "no documents survive preprocessing; nothing to deduplicate");
  if (n > 0xFFFFFFFFull) fail(ND_ERR_CONFIG, "batch exceeds 2^32 documents");
  for (uint64_t i = 0; i < n; ++i)
    if (offsets[i + 1] < offsets[i] || offsets[i + 1] - offsets[i] < p.shingle_len)
      fail(ND_ERR_SHORT, "document " + std::to_string(i) + " has fewer units than the shingle length");
  if (doc_ids)
    for (uint64_t i = 1; i < n; ++i)
      if (doc_ids[i] <= doc_ids[i - 1]) fail(ND_ERR_CONFIG, "doc_ids must be strictly ascending");
  const uint32_t K = p.bucket_count ? p.bucket_count : choose_bucket_count(n, p.scale_num, p.scale_den);
  const uint64_t cells_total = static_cast<uint64_t>(B) * K;
  if (cells_total > 0xFFFFFFFFull) fail(ND_ERR_CONFIG, "bands * bucket_count exceeds 2^32 cells");
  const uint32_t mm = min_matches(H, p.threshold_num, p.threshold_den);
  const auto r = shard_ranges(offsets, n, G);
  // K3's block fingerprints are computed by each shard for its own rows (A)
  // and read by every owner through peer memory (B), like the rows
  uint32_t fpNB = 0;
  int fpBW = 1;
  join_block_shape(H, mm, &fpNB, &fpBW);
  const char* jf = getenv("ND_JOIN_FPS");
  const bool fps_on = fpBW > 1 && !(jf && jf[0] == '0');
  std::vector<const uint32_t*> fp_bases(G, nullptr);
  // the global block join (K3g) when the single-device dedup would use it:
  // every shard fingerprints its rows (block-major) and counts its cells; the
  // owner of block k (k mod G) joins that block over ALL rows, reading the
  // fingerprints, rows and band ids in place on the shards that computed them
  const bool global = [&] {
    ND_CUDA(cudaSetDevice(g->shards[0]->device));
    return global_join_eligible(n, H, B, K, mm);
  }();
  std::vector<const uint32_t*> gfp_bases(G, nullptr), cnt_bases(G, nullptr);
  std::vector<uint64_t> first_cell(G + 1);
  for (uint32_t s = 0; s <= G; ++s)
    first_cell[s] = static_cast<uint64_t>(
        (static_cast<unsigned __int128>(cells_total) * s + G - 1) / G);
  std::vector<std::vector<uint64_t>> split(G, std::vector<uint64_t>(G + 1, 0));
  std::vector<double> t_a(G, 0), t_b(G, 0), t_k1(G, 0);
  std::vector<uint64_t> cand(G, 0), emitted(G, 0), ncells(G, 0), crec(G, 0);

  // ---- A: signatures + cell records per shard --------------------------------
  auto ta = std::chrono::steady_clock::now();
  run_shards(g, [&](uint32_t s) {
    nd_ctx* c = g->shards[s];
    auto t0 = std::chrono::steady_clock::now();
    ensure_family(c, p);
    DedupState& st = c->dedup;
    st.valid = false;
    st.doc_ids.clear();
    st.sig_on_host = false;
    const uint64_t d0 = r[s], m = r[s + 1] - r[s];
    cudaStream_t cs = c->stream;
    uint32_t* sig = st.sig.as<uint32_t>(m * H + 1);
    uint32_t* band = st.band.as<uint32_t>(m * B + 1);
    if (m) h2d_signatures(c, st, bytes, offsets + d0, m, B, p.rows, K, sig, band);
    if (global) {
      uint32_t* f = st.gj.fps_buf.as<uint32_t>(m * fpNB + 1);
      gj_fps(sig, m, H, mm, f, cs);
      gj_cell_hist(st.gj, band, m, B, K, cs);
      gfp_bases[s] = f;
      cnt_bases[s] = static_cast<const uint32_t*>(st.gj.cnt.ptr);
      ND_CUDA(cudaStreamSynchronize(cs));
      t_k1[s] = t_a[s] = since(t0);
      return;
    }
    if (fps_on) {
      uint32_t* f = c->multi.fps.as<uint32_t>(m * fpNB + 1);
      block_fingerprints(sig, m, H, fpNB, fpBW, f, cs);
      fp_bases[s] = f;
    }
    ND_CUDA(cudaStreamSynchronize(cs));
    t_k1[s] = since(t0);
    // one-digit stable partition of the records by owner (their cell order
    // is the owner's business): keys = owner, values = record index
    const uint64_t recs = m * B;
    uint32_t* keys = c->multi.send_keys.as<uint32_t>(recs + 1);
    uint32_t* vals = c->multi.send_vals.as<uint32_t>(recs + 1);
    if (recs) {
      k_owner_keys<<<4 * sm_count(), 256, 0, cs>>>(band, recs, B, K, cells_total, G, keys, vals);
      ND_CHECK_LAUNCH();
      radix_sort_u32(keys, vals, recs, std::max(1, bits_for(G - 1)), c->multi.sort, cs);
    }
    std::vector<uint64_t> owner_ids(G + 1);
    for (uint32_t o = 0; o <= G; ++o) owner_ids[o] = o;
    uint64_t* d_fc = c->multi.first_cell.as<uint64_t>(G + 1);
    uint64_t* d_split = c->multi.split.as<uint64_t>(G + 1);
    ND_CUDA(cudaMemcpyAsync(d_fc, owner_ids.data(), (G + 1) * 8, cudaMemcpyHostToDevice, cs));
    k_owner_splits<<<1, 64 * ((G + 64) / 64), 0, cs>>>(keys, recs, d_fc, G, d_split);
    ND_CHECK_LAUNCH();
    ND_CUDA(cudaMemcpyAsync(split[s].data(), d_split, (G + 1) * 8, cudaMemcpyDeviceToHost, cs));
    ND_CUDA(cudaStreamSynchronize(cs));
    split[s][G] = recs;
    t_a[s] = since(t0);
  });
  const double sec_a = since(ta);

  // ---- B: receive buffers, the fused exchange, K2 + K3 per owner -------------
  std::vector<const uint32_t*> bases(G);
  std::vector<uint64_t> row_base(G + 1);
  for (uint32_t s = 0; s < G; ++s) {
    bases[s] = static_cast<const uint32_t*>(g->shards[s]->dedup.sig.ptr);
    row_base[s] = r[s];
  }
  row_base[G] = n;
  // owner o receives source s's run at recv_base[s][o] (source order)
  std::vector<std::vector<uint64_t>> recv_base(G, std::vector<uint64_t>(G, 0));
  std::vector<uint64_t> recv_total(G, 0);
  for (uint32_t o = 0; o < G; ++o)
    for (uint32_t s = 0; s < G; ++s) {
      recv_base[s][o] = recv_total[o];
      recv_total[o] += split[s][o + 1] - split[s][o];
    }
  std::vector<uint32_t*> rkeys(G), rvals(G);
  if (global) {  // ---- B': the blocks, each joined by its owner over all rows
    std::vector<const uint32_t*> band_bases(G);
    for (uint32_t s = 0; s < G; ++s)
      band_bases[s] = static_cast<const uint32_t*>(g->shards[s]->dedup.band.ptr);
    std::vector<GJoinCounts> counts(G);
    auto tb = std::chrono::steady_clock::now();
    run_shards(g, [&](uint32_t d) {
      nd_ctx* c = g->shards[d];
      auto t0 = std::chrono::steady_clock::now();
      DedupState& st = c->dedup;
      cudaStream_t cs = c->stream;
      auto** d_sb = c->multi.row_bases.as<const uint32_t*>(G);
      auto** d_bb = c->multi.bases.as<const uint32_t*>(G);
      auto** d_fb = c->multi.fp_bases.as<const uint32_t*>(G);
      auto** d_cb = c->multi.first_cell.as<const uint32_t*>(G);
      uint64_t* d_rb = c->multi.row_base.as<uint64_t>(G + 1);
      ND_CUDA(cudaMemcpyAsync(d_sb, bases.data(), G * sizeof(void*), cudaMemcpyHostToDevice, cs));
      ND_CUDA(cudaMemcpyAsync(d_bb, band_bases.data(), G * sizeof(void*), cudaMemcpyHostToDevice, cs));
      ND_CUDA(cudaMemcpyAsync(d_fb, gfp_bases.data(), G * sizeof(void*), cudaMemcpyHostToDevice, cs));
      ND_CUDA(cudaMemcpyAsync(d_cb, cnt_bases.data(), G * sizeof(void*), cudaMemcpyHostToDevice, cs));
      ND_CUDA(cudaMemcpyAsync(d_rb, row_base.data(), (G + 1) * 8, cudaMemcpyHostToDevice, cs));
      SigView sv(bases[0], H), bv(band_bases[0], B);
      sv.bases = d_sb;
      bv.bases = d_bb;
      sv.row_base = bv.row_base = d_rb;
      sv.world = bv.world = G;
      FpCols fc;
      fc.bases = d_fb;
      fc.row_base = d_rb;
      fc.world = G;
      if (G == 1) fc.base0 = gfp_bases[0];  // one table: [NB][n]
      std::vector<uint32_t> mine;
      for (uint32_t k = d; k < fpNB && mm <= H; k += G) mine.push_back(k);
      gj_reset(st.gj, cs);
      if (d == 0) gj_cell_stats(st.gj, d_cb, G, cells_total, cs);
      PairSet& ps = st.pairs;
      ps.nb = std::max(1, bits_for(n - 1));
      ps.counter = ps.dcount.as<unsigned long long>(1);
      if (ps.cap == 0) ps.cap = std::max<uint64_t>(1 << 20, 2 * n / G);
      for (int attempt = 0; attempt < 2; ++attempt) {
        ps.keys = ps.dkeys.as<uint64_t>(ps.cap);
        ps.vals = ps.dvals.as<uint32_t>(ps.cap);
        ND_CUDA(cudaMemsetAsync(ps.counter, 0, sizeof(unsigned long long), cs));
        gj_join(st.gj, fc, sv, bv, n, mm, mine, ps.nb, ps.keys, ps.vals, ps.counter, ps.cap, cs);
        unsigned long long got = 0;
        ND_CUDA(cudaMemcpyAsync(&got, ps.counter, sizeof got, cudaMemcpyDeviceToHost, cs));
        ND_CUDA(cudaStreamSynchronize(cs));
        ps.count = got;
        if (got <= ps.cap) break;
        ps.cap = got + got / 4;
      }
      unique_pairs(ps, cs);
      counts[d] = gj_read(st.gj, cs);
      st.compare_kind = "global";
      t_b[d] = since(t0);
    });
    const double sec_b = since(tb);
    multi_finish(g, r, doc_ids, n, B, K, stats, t_k1, sec_a, sec_b, counts[0].ncells,
                 counts[0].candidate_pairs, counts[0].cell_records,
                 [&] {
                   uint64_t e = 0;
                   for (auto& c : counts) e += c.emitted;
                   return e;
                 }(), "global");
    return;
  }
  run_shards(g, [&](uint32_t d) {  // allocate on the owner's device
    CellSet& cs = g->shards[d]->dedup.cells;
    rkeys[d] = cs.rec_keys.as<uint32_t>(recv_total[d] + 1);
    rvals[d] = cs.rec_vals.as<uint32_t>(recv_total[d] + 1);
  });
  auto tb = std::chrono::steady_clock::now();
  run_shards(g, [&](uint32_t s) {  // every source scatters into every owner
    nd_ctx* c = g->shards[s];
    cudaStream_t cs = c->stream;
    const uint64_t recs = (r[s + 1] - r[s]) * B;
    if (!recs) return;
    OwnerDst h{};
    for (uint32_t o = 0; o < G; ++o) {
      h.keys[o] = rkeys[o];
      h.vals[o] = rvals[o];
      h.base[o] = recv_base[s][o];
    }
    for (uint32_t o = 0; o <= G; ++o) h.start[o] = split[s][o];
    OwnerDst* d_h = reinterpret_cast<OwnerDst*>(c->multi.bases.as<uint8_t>(sizeof(OwnerDst)));
    ND_CUDA(cudaMemcpyAsync(d_h, &h, sizeof h, cudaMemcpyHostToDevice, cs));
    k_scatter_owners<<<4 * sm_count(), 256, 0, cs>>>(
        static_cast<const uint32_t*>(c->multi.send_keys.ptr),
        static_cast<const uint32_t*>(c->multi.send_vals.ptr), recs,
        static_cast<const uint32_t*>(c->dedup.band.ptr), B, K, static_cast<uint32_t>(r[s]), d_h);
    ND_CHECK_LAUNCH();
    ND_CUDA(cudaStreamSynchronize(cs));  // the peer stores have landed
  });
  run_shards(g, [&](uint32_t d) {
    nd_ctx* c = g->shards[d];
    auto t0 = std::chrono::steady_clock::now();
    DedupState& st = c->dedup;
    cudaStream_t cs = c->stream;
    const uint64_t m = recv_total[d];
    uint32_t* rk = rkeys[d];
    uint32_t* rv = rvals[d];
    // every shard's signature rows, read in place (peer memory over NVLink)
    auto** d_bases = c->multi.row_bases.as<const uint32_t*>(G);
    uint64_t* d_rb = c->multi.row_base.as<uint64_t>(G + 1);
    ND_CUDA(cudaMemcpyAsync(d_bases, bases.data(), G * sizeof(void*), cudaMemcpyHostToDevice, cs));
    ND_CUDA(cudaMemcpyAsync(d_rb, row_base.data(), (G + 1) * 8, cudaMemcpyHostToDevice, cs));
    SigView view(bases[0], H);
    view.bases = d_bases;
    view.row_base = d_rb;
    view.world = G;
    if (fps_on) {
      auto** d_fpb = c->multi.fp_bases.as<const uint32_t*>(G);
      ND_CUDA(cudaMemcpyAsync(d_fpb, fp_bases.data(), G * sizeof(void*), cudaMemcpyHostToDevice, cs));
      view.fp_bases = d_fpb;
      view.fpNB = fpNB;
    }
    build_cells_from_records(st.cells, rk, rv, m, cells_total, kCmpRows, cs);
    compare_and_unique(st, view, H, mm, n, cs);
    ND_CUDA(cudaStreamSynchronize(cs));
    cand[d] = st.cells.candidate_pairs;
    emitted[d] = st.pairs.count;
    ncells[d] = st.cells.ncells;
    crec[d] = st.cells.cell_records;
    t_b[d] = since(t0);
  });
  const double sec_b = since(tb);

  uint64_t sc = 0, sn = 0, sr = 0, se = 0;
  for (uint32_t s = 0; s < G; ++s) {
    sn += ncells[s];
    sc += cand[s];
    se += emitted[s];
    sr += crec[s];
  }
  multi_finish(g, r, doc_ids, n, B, K, stats, t_k1, sec_a, sec_b, sn, sc, sr, se, "cells");
}

void multi_fetch_signatures(nd_ctx* g, uint32_t* sig, uint32_t* band) {
  if (!g->multi.last_valid) fail(ND_ERR_PREREQ, "no dedup result; run nd_dedup first");
  const uint32_t G = static_cast<uint32_t>(g->shards.size());
  const auto& r = g->multi.ranges;
  const uint32_t H = g->shards[0]->fam.H, B = g->shards[0]->dedup.bands;
  run_shards(g, [&](uint32_t s) {
    nd_ctx* c = g->shards[s];
    const uint64_t d0 = r[s], m = r[s + 1] - r[s];
    if (!m) return;
    if (sig)
      ND_CUDA(cudaMemcpyAsync(sig + d0 * H, c->dedup.sig.ptr, m * H * 4, cudaMemcpyDeviceToHost,
                              c->stream));
    if (band)
      ND_CUDA(cudaMemcpyAsync(band + d0 * B, c->dedup.band.ptr, m * B * 4, cudaMemcpyDeviceToHost,
                              c->stream));
    ND_CUDA(cudaStreamSynchronize(c->stream));
  });
  (void)G;
}

}  // namespace ndb

using namespace ndb;

extern "C" {

int nd_ctx_create_multi(const int* devices, int ndev, nd_ctx** out) {
  return guarded_impl(nullptr, [&] {
    if (!devices || ndev < 1) fail(ND_ERR_CONFIG, "device list must not be empty");
    if (ndev > 64) fail(ND_ERR_CONFIG, "at most 64 shards");
    std::vector<nd_ctx*> subs;
    try {
      for (int i = 0; i < ndev; ++i) {
        nd_ctx* c = nullptr;
        const int rc = nd_ctx_create(devices[i], &c);
        if (rc != ND_OK) fail(rc, nd_last_error_global());
        subs.push_back(c);
      }
      // peer access between distinct devices (NVLink / NVSwitch); the
      // exchange and the in-place row reads need it
      for (int i = 0; i < ndev; ++i)
        for (int j = 0; j < ndev; ++j) {
          if (devices[i] == devices[j]) continue;
          int can = 0;
          ND_CUDA(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]));
          if (!can)
            fail(ND_ERR_DEVICE, "device " + std::to_string(devices[i]) + " cannot access device " +
                                    std::to_string(devices[j]) + " (peer access is required)");
          ND_CUDA(cudaSetDevice(devices[i]));
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else ND_CUDA(e);
        }
      nd_ctx* gctx = nullptr;
      const int rc = nd_ctx_create(devices[0], &gctx);
      if (rc != ND_OK) fail(rc, nd_last_error_global());
      gctx->shards = subs;
      *out = gctx;
    } catch (...) {
      for (nd_ctx* c : subs) nd_ctx_destroy(c);
      throw;
    }
  });
}

int nd_ctx_shard_count(const nd_ctx* ctx) {
  return ctx ? (ctx->shards.empty() ? 1 : static_cast<int>(ctx->shards.size())) : 0;
}

}  // extern "C"
