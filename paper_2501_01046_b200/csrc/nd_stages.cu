// The staged, file-backed workflow on the GPU (pipeline.hpp:62-96):
//   nd_hash_file      hash_one_file (pipeline.cpp:171-240): K1 -> .feds
//   nd_compare_stage  run_compare_stage (pipeline.cpp:347-432): .feds -> HBM ->
//                     K2/K3 over every cell at once -> per-pass .pairs files
//   nd_union_stage    run_union_stage (pipeline.cpp:434-508): .pairs -> K4 -> report
//
// The reference's compare stage re-scans every .feds file once per gather pass
// (scan_gather, sigstore.cpp:228-286) so that each pass's cells fit a host-RAM
// budget.  Here the records are read once into host memory and the cells go to
// the GPU in as few bucket intervals as the HBM budget allows (one, holding
// every cell, for every configuration measured here; more when the signatures
// exceed the budget -- out-of-core passes, each a union of whole gather passes);
// each interval's cells are compared in one K3 launch, and the pass structure
// only decides which file each accepted pair is written to.
// A pass is (worker w = owner of band j, bucket interval [p*C, (p+1)*C)), and
// acceptance depends on the two signatures only, so a distinct accepted pair
// (lo, hi) belongs to exactly the passes {pass(j, bucket_j(lo)) : bucket_j(lo)
// == bucket_j(hi)}; compare_pass's per-pass sort + unique (compare.cpp:77-84)
// is a stable sort of those (pass, pair) tags by pass and a first-of-run skip.
#include <algorithm>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "nd_capi_impl.cuh"

namespace ndb {
namespace {

unsigned blocks_for(uint64_t n, unsigned tb) {
  return static_cast<unsigned>(std::min<uint64_t>((n + tb - 1) / tb, 1u << 30));
}

// number of bands in which the two rows of distinct pair i share a bucket
// inside the current bucket interval [k0, k1)
__global__ void k_pair_pass_count(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi,
                                  uint64_t np, const uint32_t* __restrict__ band, uint32_t bands,
                                  uint32_t k0, uint32_t k1, uint32_t* __restrict__ cnt) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= np) return;
  const uint32_t* a = band + static_cast<uint64_t>(lo[i]) * bands;
  const uint32_t* b = band + static_cast<uint64_t>(hi[i]) * bands;
  uint32_t c = 0;
  for (uint32_t j = 0; j < bands; ++j) c += a[j] == b[j] && a[j] >= k0 && a[j] < k1;
  cnt[i] = c;
}

// (pass, pair) tags; pass(j, k) = band_base[j] + k / C
__global__ void k_pair_pass_emit(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi,
                                 uint64_t np, const uint32_t* __restrict__ band, uint32_t bands,
                                 uint32_t k0, uint32_t k1, const uint32_t* __restrict__ band_base,
                                 uint32_t C, const uint64_t* __restrict__ off,
                                 uint32_t* __restrict__ pass, uint32_t* __restrict__ pair) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= np) return;
  const uint32_t* a = band + static_cast<uint64_t>(lo[i]) * bands;
  const uint32_t* b = band + static_cast<uint64_t>(hi[i]) * bands;
  uint64_t o = off[i];
  for (uint32_t j = 0; j < bands; ++j) {
    if (a[j] != b[j] || a[j] < k0 || a[j] >= k1) continue;
    pass[o] = band_base[j] + a[j] / C;
    pair[o] = static_cast<uint32_t>(i);
    ++o;
  }
}

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

nd_params params_of(const nd_feds_header& h, uint64_t num, uint64_t den) {
  nd_params p{};
  p.hash_count = h.hash_count;
  p.bands = h.bands;
  p.rows = h.rows;
  p.shingle_len = h.shingle_len;
  p.unit = h.unit;
  p.bucket_count = h.bucket_count;
  p.threshold_num = num;
  p.threshold_den = den;
  p.scale_num = h.scale_num;
  p.scale_den = h.scale_den;
  p.seed = h.family_seed;
  return p;
}

}  // namespace
}  // namespace ndb

using namespace ndb;

extern "C" {

int nd_feds_write(const char* path, const nd_feds_header* h, const uint64_t* doc_ids,
                  const uint32_t* sig, const uint32_t* band, uint64_t n, int fsync_file) {
  return guarded_impl(nullptr, [&] {
    if (!path || !h) fail(ND_ERR_CONFIG, "null argument");
    feds_write(path, *h, doc_ids, sig, band, n, fsync_file != 0);
  });
}

int nd_feds_read_header(const char* path, nd_feds_header* out) {
  return guarded_impl(nullptr, [&] { *out = feds_read_header(path, nullptr); });
}

int nd_feds_read(const char* path, uint64_t* doc_ids, uint32_t* sig, uint32_t* band) {
  return guarded_impl(nullptr, [&] {
    nd_feds_header h = feds_read_header(path, nullptr);
    std::vector<uint32_t> tmp;
    if (!band) {
      tmp.resize(h.record_count * h.bands);
      band = tmp.data();
    }
    feds_read_records(path, h, doc_ids, sig, band);
  });
}

int nd_pairs_write(const char* path, const uint64_t* lo, const uint64_t* hi, const uint32_t* m,
                   uint64_t n, int fsync_file) {
  return guarded_impl(nullptr, [&] { pairs_write(path, lo, hi, m, n, fsync_file != 0); });
}

int nd_pairs_read(const char* path, uint64_t* lo, uint64_t* hi, uint32_t* m, uint64_t* n) {
  return guarded_impl(nullptr, [&] {
    std::vector<uint64_t> l, h;
    std::vector<uint32_t> mm;
    pairs_read(path, l, h, mm);
    if (lo || hi || m) {
      if (*n < l.size()) fail(ND_ERR_CONFIG, "pair buffers too small");
      if (lo) std::copy(l.begin(), l.end(), lo);
      if (hi) std::copy(h.begin(), h.end(), hi);
      if (m) std::copy(mm.begin(), mm.end(), m);
    }
    *n = l.size();
  });
}

int nd_plan_gather(uint64_t total_bytes, uint32_t K, uint32_t bands, uint32_t workers,
                   uint64_t budget, uint32_t override_c, uint32_t* c_out, uint32_t* passes_out) {
  return guarded_impl(nullptr, [&] {
    if (workers == 0) fail(ND_ERR_CONFIG, "worker count must be positive");
    std::vector<uint32_t> wb(workers);
    for (uint32_t w = 0; w < workers; ++w) wb[w] = bands / workers + (w < bands % workers ? 1 : 0);
    std::vector<uint32_t> passes;
    *c_out = plan_gather(total_bytes, K, wb, budget, override_c, passes);
    if (passes_out) std::copy(passes.begin(), passes.end(), passes_out);
  });
}

int nd_hash_file(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets,
                 const uint64_t* doc_ids, uint64_t n, const nd_feds_header* header,
                 const char* path, int fsync_file) {
  return guarded_impl(ctx, [&] {
    const nd_feds_header h = *header;
    const nd_params p = params_of(h, 0, 1);
    validate(p);
    ensure_family(ctx, p);
    for (uint64_t i = 1; i < n; ++i)
      if (doc_ids[i] <= doc_ids[i - 1]) fail(ND_ERR_CONFIG, "doc_ids must be strictly ascending");
    std::vector<uint32_t> sig(n * h.hash_count), band(n * h.bands);
    if (n) {
      const int rc = nd_signatures(ctx, bytes, offsets, n, h.bands, h.rows, h.bucket_count,
                                   sig.data(), band.data());
      if (rc != ND_OK) fail(rc, ctx->err);
    }
    feds_write(path, h, doc_ids, sig.data(), band.data(), n, fsync_file != 0);
  });
}

int nd_compare_stage(nd_ctx* ctx, const char* const* feds_paths, uint32_t nfiles,
                     const nd_feds_header* expected, uint64_t total_signature_bytes,
                     uint32_t workers, uint64_t memory_budget, uint32_t buckets_per_pass,
                     uint64_t thr_num, uint64_t thr_den, const char* pairs_dir, int fsync_files,
                     nd_compare_stage_stats* stats) {
  return guarded_impl(ctx, [&] {
    auto t0 = std::chrono::steady_clock::now();
    const nd_feds_header ex = *expected;
    const nd_params p = params_of(ex, thr_num, thr_den);
    validate(p);
    if (workers == 0) fail(ND_ERR_CONFIG, "worker count must be positive");
    const uint32_t H = ex.hash_count, B = ex.bands, K = ex.bucket_count;
    // band_partition (lsh.cpp:62-72) + plan_gather (sigstore.cpp:288-329)
    std::vector<uint32_t> wbands(workers), passes;
    for (uint32_t w = 0; w < workers; ++w) wbands[w] = B / workers + (w < B % workers ? 1 : 0);
    const uint32_t C = plan_gather(total_signature_bytes, K, wbands, memory_budget,
                                   buckets_per_pass, passes);
    std::vector<uint32_t> pass_base(workers + 1, 0), band_base(B);
    for (uint32_t w = 0; w < workers; ++w) pass_base[w + 1] = pass_base[w] + passes[w];
    const uint32_t total_passes = pass_base[workers];
    for (uint32_t w = 0, j = 0; w < workers; ++w)
      for (uint32_t k = 0; k < wbands[w]; ++k) band_base[j++] = pass_base[w];

    // ---- every record into host SoA buffers
    std::vector<nd_feds_header> hs(nfiles);
    uint64_t n = 0;
    for (uint32_t f = 0; f < nfiles; ++f) {
      hs[f] = feds_read_header(feds_paths[f], nullptr);
      if (!feds_run_compatible(hs[f], ex))
        fail(ND_ERR_CONFIG, std::string("'") + feds_paths[f] +
                                "' was written with different parameters than this run");
      n += hs[f].record_count;
    }
    if (n > 0xFFFFFFFFull) fail(ND_ERR_CONFIG, "more than 2^32 signature records");
    DedupState& st = ctx->dedup;
    st.valid = false;
    std::vector<uint64_t> ids(n);
    std::vector<uint32_t> hsig(n * H), hband(n * B);
    for (uint32_t f = 0, r = 0; f < nfiles; r += static_cast<uint32_t>(hs[f].record_count), ++f)
      feds_read_records(feds_paths[f], hs[f], ids.data() + r, hsig.data() + uint64_t(r) * H,
                        hband.data() + uint64_t(r) * B);
    for (uint64_t i = 1; i < n; ++i)
      if (ids[i] <= ids[i - 1])
        fail(ND_ERR_CONFIG, "signature files are not in ascending doc_id order; "
                            "pass them in manifest order");
    const double t_load = since(t0);
    auto t1 = std::chrono::steady_clock::now();

    // ---- records per bucket -> bucket intervals [k0, k1) that fit the HBM
    // budget, aligned to the gather passes (multiples of C) so that every
    // pass lies inside exactly one interval.  One interval = everything in
    // HBM at once; more = out-of-core passes over the host-resident records.
    std::vector<uint64_t> per_bucket(K, 0);
    for (uint64_t i = 0; i < n * B; ++i) ++per_bucket[hband[i]];
    const uint64_t row_bytes = 4ull * H + 4ull * B + 8;   // signature + band ids + doc map
    const uint64_t rec_bytes = 8 * 4;                      // record + sort scratch + cell CSR
    uint64_t budget = ctx->hbm_budget;
    if (budget == 0) {
      size_t fr = 0, tot = 0;
      ND_CUDA(cudaMemGetInfo(&fr, &tot));
      budget = static_cast<uint64_t>(fr) / 10 * 7;
    }
    std::vector<std::pair<uint32_t, uint32_t>> intervals;
    {
      const uint64_t whole = n * row_bytes + n * B * rec_bytes;
      if (whole <= budget) {
        intervals.push_back({0, K});
      } else {
        uint32_t k0 = 0;
        uint64_t acc = 0;
        for (uint32_t k = 0; k < K; k += C) {
          const uint32_t k1 = std::min<uint64_t>(K, uint64_t(k) + C);
          uint64_t recs = 0;
          for (uint32_t b = k; b < k1; ++b) recs += per_bucket[b];
          const uint64_t bytes = recs * (row_bytes + rec_bytes);  // a record may bring its row
          if (k > k0 && acc + bytes > budget) {
            intervals.push_back({k0, k});
            k0 = k;
            acc = 0;
          }
          acc += bytes;
        }
        intervals.push_back({k0, K});
      }
    }

    cudaStream_t s = ctx->stream;
    const uint32_t mm = min_matches(H, thr_num, thr_den);
    uint64_t candidates = 0, distinct_total = 0;
    // accepted (pass, lo doc, hi doc, match) in per-pass (lo, hi) order
    std::vector<uint32_t> out_pass, out_m;
    std::vector<uint64_t> out_lo, out_hi;
    std::vector<uint32_t> sel;                  // rows of this interval
    std::vector<uint32_t> rkeys, rvals;         // (cell, local row) records
    for (auto [k0, k1] : intervals) {
      // documents with a band bucket in [k0, k1), and their in-range records
      const bool all = k0 == 0 && k1 == K;
      sel.clear();
      rkeys.clear();
      rvals.clear();
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t* bi = hband.data() + i * B;
        bool any = all;
        for (uint32_t j = 0; j < B && !any; ++j) any = bi[j] >= k0 && bi[j] < k1;
        if (!any) continue;
        const uint32_t local = static_cast<uint32_t>(sel.size());
        sel.push_back(static_cast<uint32_t>(i));
        if (!all)
          for (uint32_t j = 0; j < B; ++j)
            if (bi[j] >= k0 && bi[j] < k1) {
              rkeys.push_back(j * K + bi[j]);
              rvals.push_back(local);
            }
      }
      const uint64_t m = sel.size();
      if (m == 0) continue;
      uint32_t* d_sig = st.sig.as<uint32_t>(m * H + 1);
      uint32_t* d_band = st.band.as<uint32_t>(m * B + 1);
      if (all) {
        ND_CUDA(cudaMemcpyAsync(d_sig, hsig.data(), m * H * 4, cudaMemcpyHostToDevice, s));
        ND_CUDA(cudaMemcpyAsync(d_band, hband.data(), m * B * 4, cudaMemcpyHostToDevice, s));
        build_cells_from_bands(st.cells, d_band, m, B, K, kCmpRows, s);
      } else {
        std::vector<uint32_t> gs(m * H), gb(m * B);
        for (uint64_t r = 0; r < m; ++r) {
          std::memcpy(gs.data() + r * H, hsig.data() + uint64_t(sel[r]) * H, 4ull * H);
          std::memcpy(gb.data() + r * B, hband.data() + uint64_t(sel[r]) * B, 4ull * B);
        }
        ND_CUDA(cudaMemcpyAsync(d_sig, gs.data(), m * H * 4, cudaMemcpyHostToDevice, s));
        ND_CUDA(cudaMemcpyAsync(d_band, gb.data(), m * B * 4, cudaMemcpyHostToDevice, s));
        const uint64_t nr = rkeys.size();
        uint32_t* dk = st.cells.rec_keys.as<uint32_t>(nr + 1);
        uint32_t* dv = st.cells.rec_vals.as<uint32_t>(nr + 1);
        ND_CUDA(cudaMemcpyAsync(dk, rkeys.data(), nr * 4, cudaMemcpyHostToDevice, s));
        ND_CUDA(cudaMemcpyAsync(dv, rvals.data(), nr * 4, cudaMemcpyHostToDevice, s));
        build_cells_from_records(st.cells, dk, dv, nr, uint64_t(B) * K, kCmpRows, s);
        ND_CUDA(cudaStreamSynchronize(s));  // gs / gb / rkeys / rvals leave scope
      }
      compare_and_unique(st, d_sig, H, mm, m, s);
      candidates += st.cells.candidate_pairs;
      const uint64_t distinct = st.pairs.distinct;
      distinct_total += distinct;
      if (distinct == 0) continue;
      PairSet& ps = st.pairs;
      uint32_t* d_bb = st.cells.maxbuf.as<uint32_t>(B);
      ND_CUDA(cudaMemcpyAsync(d_bb, band_base.data(), B * 4, cudaMemcpyHostToDevice, s));
      uint32_t* cnt = ps.flag.as<uint32_t>(distinct);
      uint64_t* off = ps.idx.as<uint64_t>(distinct + 1);
      k_pair_pass_count<<<blocks_for(distinct, 256), 256, 0, s>>>(ps.lo, ps.hi, distinct, d_band, B,
                                                                 k0, k1, cnt);
      ND_CHECK_LAUNCH();
      scan_u32_to_u64(cnt, off, distinct, ps.scan, s);
      uint64_t tagged = 0;
      ND_CUDA(cudaMemcpyAsync(&tagged, off + distinct, 8, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
      uint32_t* d_pass = st.cells.rec_keys.as<uint32_t>(tagged + 1);
      uint32_t* d_pair = st.cells.rec_vals.as<uint32_t>(tagged + 1);
      k_pair_pass_emit<<<blocks_for(distinct, 256), 256, 0, s>>>(ps.lo, ps.hi, distinct, d_band, B,
                                                                k0, k1, d_bb, C, off, d_pass,
                                                                d_pair);
      ND_CHECK_LAUNCH();
      // stable by pass: pairs stay in (lo, hi) order inside each pass
      radix_sort_u32(d_pass, d_pair, tagged, bits_for(total_passes ? total_passes - 1 : 0),
                     st.cells.sort, s);
      std::vector<uint32_t> hpass(tagged), hpair(tagged), plo(distinct), phi(distinct), pm(distinct);
      ND_CUDA(cudaMemcpyAsync(hpass.data(), d_pass, tagged * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaMemcpyAsync(hpair.data(), d_pair, tagged * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaMemcpyAsync(plo.data(), ps.lo, distinct * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaMemcpyAsync(phi.data(), ps.hi, distinct * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaMemcpyAsync(pm.data(), ps.mc, distinct * 4, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
      for (uint64_t t = 0; t < tagged; ++t) {
        const uint32_t i = hpair[t];
        // the pair shares this pass through two bands: compare_pass's unique
        if (t > 0 && hpass[t] == hpass[t - 1] && hpair[t - 1] == i) continue;
        out_pass.push_back(hpass[t]);
        out_lo.push_back(ids[sel[plo[i]]]);
        out_hi.push_back(ids[sel[phi[i]]]);
        out_m.push_back(pm[i]);
      }
    }
    // passes in increasing order across intervals (intervals ascend in bucket,
    // passes of one worker ascend in bucket, workers interleave): group by pass
    std::vector<uint64_t> order(out_pass.size());
    for (uint64_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](uint64_t x, uint64_t y) { return out_pass[x] < out_pass[y]; });
    const double t_gpu = since(t1);
    auto t2 = std::chrono::steady_clock::now();

    // ---- one pair file per (worker, pass)
    uint64_t emitted = 0, cursor = 0;
    const uint64_t tagged = order.size();
    std::vector<uint64_t> lo, hi;
    std::vector<uint32_t> m;
    const std::string dir(pairs_dir);
    for (uint32_t w = 0; w < workers; ++w) {
      for (uint32_t pp = 0; pp < passes[w]; ++pp) {
        const uint32_t gp = pass_base[w] + pp;
        lo.clear();
        hi.clear();
        m.clear();
        for (; cursor < tagged && out_pass[order[cursor]] == gp; ++cursor) {
          const uint64_t x = order[cursor];
          lo.push_back(out_lo[x]);
          hi.push_back(out_hi[x]);
          m.push_back(out_m[x]);
        }
        emitted += lo.size();
        pairs_write(dir + "/w" + std::to_string(w) + "_p" + std::to_string(pp) + ".pairs",
                    lo.data(), hi.data(), m.data(), lo.size(), fsync_files != 0);
      }
    }
    if (cursor != tagged) fail(ND_ERR_INTERNAL, "pass tags out of range");
    // scan_gather's gauge: every record of a pass is resident at the end of
    // its scan; workers run their p-th passes side by side
    const uint64_t entry = 8 + 4ull * H;
    std::vector<uint64_t> hist(std::max<uint32_t>(total_passes, 1), 0);
    for (uint64_t i = 0; i < n; ++i)
      for (uint32_t j = 0; j < B; ++j) ++hist[band_base[j] + hband[i * B + j] / C];
    uint64_t peak = 0;
    const uint32_t maxp = passes.empty() ? 0 : *std::max_element(passes.begin(), passes.end());
    for (uint32_t pp = 0; pp < maxp; ++pp) {
      uint64_t sum = 0;
      for (uint32_t w = 0; w < workers; ++w)
        if (pp < passes[w]) sum += hist[pass_base[w] + pp] * entry;
      peak = std::max(peak, sum);
    }
    if (stats) {
      *stats = nd_compare_stage_stats{};
      stats->buckets_per_pass = C;
      stats->pass_count = total_passes;
      stats->candidate_pairs = candidates;
      stats->emitted_pairs = emitted;
      stats->gather_peak_bytes = peak;
      stats->records = n;
      stats->distinct_pairs = distinct_total;
      stats->intervals = static_cast<uint32_t>(intervals.size());
      stats->seconds[0] = t_load;
      stats->seconds[1] = t_gpu;
      stats->seconds[2] = since(t2);
    }
  });
}

int nd_set_hbm_budget(nd_ctx* ctx, uint64_t bytes) {
  return guarded_impl(ctx, [&] { ctx->hbm_budget = bytes; });
}

int nd_union_stage(nd_ctx* ctx, const char* const* pair_paths, uint32_t nfiles,
                   uint64_t total_surviving, uint64_t total_records, const char* workspace,
                   int fsync_files, nd_dedup_stats* stats) {
  return guarded_impl(ctx, [&] {
    std::vector<uint64_t> lo, hi;
    std::vector<uint32_t> m;
    for (uint32_t f = 0; f < nfiles; ++f) pairs_read(pair_paths[f], lo, hi, m);
    const uint64_t np = lo.size();
    // node ids: doc ids themselves when they are dense enough (the union
    // arrays are sized by the largest id), else a dense renumbering of the
    // ids that occur in pairs (union_pairs renumbers densely, dedup_graph.cpp:48-54)
    uint64_t maxid = 0;
    for (uint64_t i = 0; i < np; ++i) maxid = std::max(maxid, std::max(lo[i], hi[i]));
    const bool direct = maxid < 0x7FFFFFFFull && maxid < 16 * np + (1ull << 20);
    DedupState& st = ctx->dedup;
    st.valid = false;
    st.doc_ids.clear();
    std::vector<uint32_t> l32(np), h32(np);
    uint64_t nnodes = np ? maxid + 1 : 1;
    if (direct) {
      for (uint64_t i = 0; i < np; ++i) {
        l32[i] = static_cast<uint32_t>(lo[i]);
        h32[i] = static_cast<uint32_t>(hi[i]);
      }
    } else {
      std::vector<uint64_t> idv(lo);
      idv.insert(idv.end(), hi.begin(), hi.end());
      std::sort(idv.begin(), idv.end());
      idv.erase(std::unique(idv.begin(), idv.end()), idv.end());
      auto rank = [&](uint64_t d) {
        return static_cast<uint32_t>(std::lower_bound(idv.begin(), idv.end(), d) - idv.begin());
      };
      for (uint64_t i = 0; i < np; ++i) {
        l32[i] = rank(lo[i]);
        h32[i] = rank(hi[i]);
      }
      nnodes = idv.size();
      st.doc_ids = std::move(idv);
    }
    cudaStream_t s = ctx->stream;
    uint32_t* d_lo = st.cells.rec_keys.as<uint32_t>(np + 1);
    uint32_t* d_hi = st.cells.rec_vals.as<uint32_t>(np + 1);
    uint32_t* d_m = st.cells.run_idx.as<uint32_t>(np + 1);
    if (np) {
      ND_CUDA(cudaMemcpyAsync(d_lo, l32.data(), np * 4, cudaMemcpyHostToDevice, s));
      ND_CUDA(cudaMemcpyAsync(d_hi, h32.data(), np * 4, cudaMemcpyHostToDevice, s));
      ND_CUDA(cudaMemcpyAsync(d_m, m.data(), np * 4, cudaMemcpyHostToDevice, s));
    }
    st.pairs.nb = std::max(1, bits_for(nnodes - 1));
    if (2 * st.pairs.nb > 64) fail(ND_ERR_CONFIG, "too many nodes for packed pair keys");
    // sort + distinct (pipeline.cpp:466-473), union + components (:475-476)
    pack_pairs(st.pairs, d_lo, d_hi, d_m, np, s);
    unique_pairs(st.pairs, s);
    components(st.groups, st.pairs.lo, st.pairs.hi, st.pairs.distinct, nnodes, s);
    ND_CUDA(cudaStreamSynchronize(s));
    st.documents = total_surviving;
    st.valid = true;
    if (stats) {
      *stats = nd_dedup_stats{};
      stats->documents = total_surviving;
      stats->emitted_pairs = np;
      stats->distinct_pairs = st.pairs.distinct;
      stats->duplicate_groups = st.groups.groups;
      stats->near_duplicates = st.groups.members;
      stats->removals = st.groups.removals;
    }
    const int rc = nd_dedup_write_report_ex(ctx, workspace, total_records, fsync_files);
    if (rc != ND_OK) fail(rc, ctx->err);
  });
}

}  // extern "C"
