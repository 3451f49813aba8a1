// Multi-GPU compare over peer memory: instead of all-gathering
// every rank's signature rows (N * 4H bytes to every GPU), each rank exports
// its rows once through a CUDA IPC handle, maps the other ranks' rows
// (NVLink / NVSwitch peer memory; the same device when ranks share a GPU),
// and the K3 kernels read exactly the rows their cells need straight from the
// owning GPU's HBM (SigView in nd_internal.cuh).  The record exchange stays an
// NCCL all-to-all; only the signature all-gather is replaced.
#include <cstring>
#include <string>
#include <vector>

#include "nd_capi_impl.cuh"

using namespace ndb;

namespace {
__global__ void k_pack_records(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                               uint64_t m, uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = (static_cast<uint64_t>(keys[i]) << 32) | vals[i];
}
__global__ void k_unpack_records(const uint64_t* __restrict__ in, uint64_t m,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = in[i];
    keys[i] = static_cast<uint32_t>(r >> 32);
    vals[i] = static_cast<uint32_t>(r);
  }
}
// owner run starts in the cell-sorted keys: lower_bound of each owner's first cell
__global__ void k_splits(const uint32_t* __restrict__ keys, uint64_t m,
                         const uint64_t* __restrict__ first_cell, uint32_t G,
                         uint64_t* __restrict__ split) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g > G) return;
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < first_cell[g]) lo = mid + 1; else hi = mid;
  }
  split[g] = lo;
}
}  // namespace

extern "C" {

int nd_stage_records_packed(nd_ctx* ctx, const uint32_t* d_band, uint64_t n, uint32_t bands,
                            uint32_t K, uint32_t doc_base, uint32_t world, uint64_t* d_rec,
                            uint64_t* owner_split) {
  return guarded_impl(ctx, [&] {
    if (bands == 0 || K == 0) fail(ND_ERR_CONFIG, "bands and bucket count must be positive");
    if (world == 0) fail(ND_ERR_CONFIG, "world size must be positive");
    cudaStream_t s = ctx->stream;
    const uint64_t m = n * bands;
    const uint64_t cells = static_cast<uint64_t>(bands) * K;
    uint32_t* keys = ctx->multi.send_keys.as<uint32_t>(m + 1);
    uint32_t* vals = ctx->multi.send_vals.as<uint32_t>(m + 1);
    make_records(d_band, n, bands, K, doc_base, keys, vals, s);
    radix_sort_u32(keys, vals, m, bits_for(cells - 1), ctx->stage_sort, s);
    if (m) {
      k_pack_records<<<4 * sm_count(), 256, 0, s>>>(keys, vals, m, d_rec);
      ND_CHECK_LAUNCH();
    }
    std::vector<uint64_t> first(world + 1);
    for (uint32_t g = 0; g <= world; ++g)
      first[g] = static_cast<uint64_t>((static_cast<unsigned __int128>(cells) * g + world - 1) / world);
    uint64_t* d_first = ctx->multi.first_cell.as<uint64_t>(world + 1);
    uint64_t* d_split = ctx->multi.split.as<uint64_t>(world + 1);
    ND_CUDA(cudaMemcpyAsync(d_first, first.data(), (world + 1) * 8, cudaMemcpyHostToDevice, s));
    k_splits<<<1, 64 * ((world + 64) / 64), 0, s>>>(keys, m, d_first, world, d_split);
    ND_CHECK_LAUNCH();
    ND_CUDA(cudaMemcpyAsync(owner_split, d_split, (world + 1) * 8, cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
    owner_split[world] = m;
  });
}

int nd_stage_compare_peer_packed(nd_ctx* ctx, const uint64_t* d_rec, uint64_t m,
                                 uint64_t key_limit, uint64_t num, uint64_t den,
                                 uint64_t* npairs_out, uint64_t* cand_out) {
  return guarded_impl(ctx, [&] {
    cudaStream_t s = ctx->stream;
    uint32_t* k = ctx->multi.send_keys.as<uint32_t>(m + 1);
    uint32_t* v = ctx->multi.send_vals.as<uint32_t>(m + 1);
    if (m) {
      k_unpack_records<<<4 * sm_count(), 256, 0, s>>>(d_rec, m, k, v);
      ND_CHECK_LAUNCH();
    }
    const int rc = nd_stage_compare_peer(ctx, k, v, m, key_limit, num, den, npairs_out, cand_out);
    if (rc != ND_OK) fail(rc, ctx->err);
  });
}


int nd_peer_export(nd_ctx* ctx, const uint32_t* d_sig, uint64_t rows, uint32_t H,
                   uint8_t* handle_out) {
  return guarded_impl(ctx, [&] {
    if (H == 0) fail(ND_ERR_CONFIG, "hash count must be positive");
    // an allocation of our own: IPC handles name whole allocations, and the
    // rows must stay put until every peer has finished reading them
    ctx->peer.own.release();
    uint32_t* own = ctx->peer.own.as<uint32_t>(rows * H + 32);
    if (rows)
      ND_CUDA(cudaMemcpyAsync(own, d_sig, rows * H * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    ND_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaIpcMemHandle_t h;
    ND_CUDA(cudaIpcGetMemHandle(&h, own));
    static_assert(sizeof(h) == ND_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof h);
    ctx->peer.H = H;
    ctx->peer.B = 0;  // rows only (the cell compare)
  });
}

namespace {
uint64_t align256(uint64_t b) { return (b + 255) & ~uint64_t{255}; }
}  // namespace

int nd_peer_export_gjoin(nd_ctx* ctx, const uint32_t* d_sig, const uint32_t* d_band, uint64_t rows,
                         uint32_t H, uint32_t bands, uint64_t num, uint64_t den,
                         uint8_t* handle_out) {
  return guarded_impl(ctx, [&] {
    if (H == 0 || bands == 0) fail(ND_ERR_CONFIG, "hash count and bands must be positive");
    if (den == 0) fail(ND_ERR_CONFIG, "ratio denominator must be positive");
    const uint32_t mm = min_matches(H, num, den);
    uint32_t NB = 0;
    int BW = 1;
    if (mm <= H) join_block_shape(H, mm, &NB, &BW);
    if (NB > kGJoinMaxBlocks) fail(ND_ERR_CONFIG, "threshold needs more than 64 blocks: use the cell compare");
    // one allocation: [rows x H signatures][rows x bands band ids][NB x rows fingerprints]
    const uint64_t sb = align256(rows * H * 4), bb = align256(rows * bands * 4);
    ctx->peer.own.release();
    uint8_t* own = ctx->peer.own.as<uint8_t>(sb + bb + rows * NB * 4 + 256);
    cudaStream_t s = ctx->stream;
    if (rows) {
      ND_CUDA(cudaMemcpyAsync(own, d_sig, rows * H * 4, cudaMemcpyDeviceToDevice, s));
      ND_CUDA(cudaMemcpyAsync(own + sb, d_band, rows * bands * 4, cudaMemcpyDeviceToDevice, s));
      gj_fps(d_sig, rows, H, mm, reinterpret_cast<uint32_t*>(own + sb + bb), s);
    }
    ND_CUDA(cudaStreamSynchronize(s));
    cudaIpcMemHandle_t h;
    ND_CUDA(cudaIpcGetMemHandle(&h, own));
    std::memcpy(handle_out, &h, sizeof h);
    ctx->peer.H = H;
    ctx->peer.B = bands;
    ctx->peer.mm = mm;
    ctx->peer.NB = NB;
  });
}

int nd_peer_open(nd_ctx* ctx, const uint8_t* handles, const uint64_t* row_base, uint32_t world,
                 uint32_t self) {
  return guarded_impl(ctx, [&] {
    if (world == 0 || self >= world) fail(ND_ERR_CONFIG, "bad peer rank");
    if (!ctx->peer.own.ptr) fail(ND_ERR_PREREQ, "export the local rows first (nd_peer_export)");
    auto& P = ctx->peer;
    for (void* p : P.opened) cudaIpcCloseMemHandle(p);
    P.opened.clear();
    std::vector<const uint32_t*> bases(world);
    for (uint32_t r = 0; r < world; ++r) {
      if (r == self) {
        bases[r] = static_cast<const uint32_t*>(P.own.ptr);
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + static_cast<size_t>(r) * ND_IPC_HANDLE_BYTES, sizeof h);
      void* p = nullptr;
      ND_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      P.opened.push_back(p);
      bases[r] = static_cast<const uint32_t*>(p);
    }
    auto** d_bases = P.bases.as<const uint32_t*>(world);
    uint64_t* d_rb = P.row_base.as<uint64_t>(world + 1);
    ND_CUDA(cudaMemcpyAsync(d_bases, bases.data(), world * sizeof(void*), cudaMemcpyHostToDevice,
                            ctx->stream));
    ND_CUDA(cudaMemcpyAsync(d_rb, row_base, (world + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                            ctx->stream));
    ND_CUDA(cudaStreamSynchronize(ctx->stream));
    P.world = world;
    P.rows = row_base[world];
    P.view = SigView(bases[0], P.H);
    P.view.bases = d_bases;
    P.view.row_base = d_rb;
    P.view.world = world;
    if (P.B) {  // nd_peer_export_gjoin's layout: band ids and fingerprints follow
      std::vector<const uint32_t*> bb(world), fb(world);
      for (uint32_t r = 0; r < world; ++r) {
        const uint64_t rows = row_base[r + 1] - row_base[r];
        const uint8_t* b = reinterpret_cast<const uint8_t*>(bases[r]);
        const uint64_t sb = align256(rows * P.H * 4), bsz = align256(rows * P.B * 4);
        bb[r] = reinterpret_cast<const uint32_t*>(b + sb);
        fb[r] = reinterpret_cast<const uint32_t*>(b + sb + bsz);
      }
      auto** d_bb = P.band_bases.as<const uint32_t*>(world);
      auto** d_fb = P.fp_bases.as<const uint32_t*>(world);
      ND_CUDA(cudaMemcpyAsync(d_bb, bb.data(), world * sizeof(void*), cudaMemcpyHostToDevice,
                              ctx->stream));
      ND_CUDA(cudaMemcpyAsync(d_fb, fb.data(), world * sizeof(void*), cudaMemcpyHostToDevice,
                              ctx->stream));
      ND_CUDA(cudaStreamSynchronize(ctx->stream));
      P.band_view = SigView(bb[0], P.B);
      P.band_view.bases = d_bb;
      P.band_view.row_base = d_rb;
      P.band_view.world = world;
      P.fps = FpCols{};
      P.fps.bases = d_fb;
      P.fps.row_base = d_rb;
      P.fps.world = world;
      if (world == 1) P.fps.base0 = fb[0];
    }
  });
}

int nd_stage_gjoin_peer(nd_ctx* ctx, uint32_t self, uint64_t* npairs_out, uint64_t* emitted_out) {
  return guarded_impl(ctx, [&] {
    auto& P = ctx->peer;
    if (P.world == 0 || P.B == 0)
      fail(ND_ERR_PREREQ, "no peer rows mapped with nd_peer_export_gjoin + nd_peer_open");
    if (self >= P.world) fail(ND_ERR_CONFIG, "bad peer rank");
    DedupState& st = ctx->api;
    cudaStream_t s = ctx->stream;
    st.valid = false;
    std::vector<uint32_t> mine;  // the blocks this rank joins: k = self (mod world)
    for (uint32_t k = self; k < P.NB; k += P.world) mine.push_back(k);
    const uint64_t n = P.rows;
    gj_reset(st.gj, s);
    PairSet& ps = st.pairs;
    ps.nb = std::max(1, bits_for(n ? n - 1 : 0));
    ps.counter = ps.dcount.as<unsigned long long>(1);
    if (ps.cap == 0) ps.cap = std::max<uint64_t>(1 << 20, 2 * n / P.world);
    for (int attempt = 0; attempt < 2; ++attempt) {
      ps.keys = ps.dkeys.as<uint64_t>(ps.cap);
      ps.vals = ps.dvals.as<uint32_t>(ps.cap);
      ND_CUDA(cudaMemsetAsync(ps.counter, 0, sizeof(unsigned long long), s));
      gj_join(st.gj, P.fps, P.view, P.band_view, n, P.mm, mine, ps.nb, ps.keys, ps.vals,
              ps.counter, ps.cap, s);
      unsigned long long got = 0;
      ND_CUDA(cudaMemcpyAsync(&got, ps.counter, sizeof got, cudaMemcpyDeviceToHost, s));
      ND_CUDA(cudaStreamSynchronize(s));
      ps.count = got;
      if (got <= ps.cap) break;
      ps.cap = got + got / 4;
    }
    unique_pairs(ps, s);
    const GJoinCounts c = gj_read(st.gj, s);
    st.valid = true;
    *npairs_out = ps.distinct;
    if (emitted_out) *emitted_out = c.emitted;
  });
}

int nd_stage_cell_hist(nd_ctx* ctx, const uint32_t* d_band, uint64_t n, uint32_t bands, uint32_t K,
                       uint32_t* d_cnt) {
  return guarded_impl(ctx, [&] {
    if (bands == 0 || K == 0) fail(ND_ERR_CONFIG, "bands and bucket count must be positive");
    GJoin& g = ctx->api.gj;
    unsigned int* bad = reinterpret_cast<unsigned int*>(g.acc.as<uint64_t>(4));
    ND_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned int), ctx->stream));
    gj_cell_hist(g, d_band, n, bands, K, ctx->stream, bad);
    ND_CUDA(cudaMemcpyAsync(d_cnt, g.cnt.ptr, static_cast<uint64_t>(bands) * K * 4,
                            cudaMemcpyDeviceToDevice, ctx->stream));
    unsigned int h_bad = 0;
    ND_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof h_bad, cudaMemcpyDeviceToHost, ctx->stream));
    ND_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h_bad) fail(ND_ERR_CONFIG, std::to_string(h_bad) + " band ids are not below the bucket count");
  });
}

int nd_stage_compare_peer(nd_ctx* ctx, const uint32_t* d_keys, const uint32_t* d_vals,
                          uint64_t m, uint64_t key_limit, uint64_t num, uint64_t den,
                          uint64_t* npairs_out, uint64_t* cand_out) {
  return guarded_impl(ctx, [&] {
    if (ctx->peer.world == 0) fail(ND_ERR_PREREQ, "no peer rows mapped (nd_peer_open)");
    if (den == 0) fail(ND_ERR_CONFIG, "ratio denominator must be positive");
    const uint32_t H = ctx->peer.H;
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
    compare_and_unique(st, ctx->peer.view, H, min_matches(H, num, den), ctx->peer.rows, s);
    ND_CUDA(cudaStreamSynchronize(s));
    st.valid = true;
    *npairs_out = st.pairs.distinct;
    if (cand_out) *cand_out = st.cells.candidate_pairs;
  });
}

int nd_peer_close(nd_ctx* ctx) {
  return guarded_impl(ctx, [&] {
    auto& P = ctx->peer;
    for (void* p : P.opened) cudaIpcCloseMemHandle(p);
    P.opened.clear();
    P.world = 0;
    P.B = 0;
    P.own.release();
  });
}

}  // extern "C"
