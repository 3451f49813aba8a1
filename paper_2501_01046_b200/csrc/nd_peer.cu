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

extern "C" {

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
    P.own.release();
  });
}

}  // extern "C"
