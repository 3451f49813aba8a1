// C-ABI of neardup_b200 (include/neardup_b200.h): context, family upload,
// signature entry points (host-pipelined and device-resident), and the
// exception -> status mapping (reference taxonomy util.hpp:13-26).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nd_capi_impl.cuh"

namespace {
thread_local std::string g_error;
}

namespace ndb {

std::atomic<uint64_t> g_launches{0};

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

int guarded_impl(nd_ctx* ctx, const std::function<void()>& fn) {
  try {
    if (ctx) ND_CUDA(cudaSetDevice(ctx->device));
    fn();
    return ND_OK;
  } catch (const NdError& e) {
    (ctx ? ctx->err : g_error) = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    (ctx ? ctx->err : g_error) = std::string("host allocation failed: ") + e.what();
    return ND_ERR_INTERNAL;
  } catch (const std::exception& e) {
    (ctx ? ctx->err : g_error) = e.what();
    return ND_ERR_INTERNAL;
  }
}

}  // namespace ndb

using ndb::fail;

nd_ctx::~nd_ctx() {
  for (auto* b : {&fam_buf, &sig_in_text, &sig_in_off, &gate_flag}) b->release();
  for (int i = 0; i < kSlots; ++i) {
    slot[i].text.release();
    slot[i].off.release();
    slot[i].sig.release();
    slot[i].band.release();
    slot[i].scratch.release();
    if (slot[i].h2d_done) cudaEventDestroy(slot[i].h2d_done);
    if (slot[i].comp_done) cudaEventDestroy(slot[i].comp_done);
    if (slot[i].d2h_done) cudaEventDestroy(slot[i].d2h_done);
    if (slot[i].comp) cudaStreamDestroy(slot[i].comp);
  }
  pinned_off.release();
  multi.release();
  for (void* p : peer.opened) cudaIpcCloseMemHandle(p);
  for (auto* b : {&peer.own, &peer.bases, &peer.row_base}) b->release();
  for (auto& r : ring) r.release();
  for (auto& r : ring_scratch) r.release();
  for (auto& r : ring_stream)
    if (r) cudaStreamDestroy(r);
  synth_buf.release();
  sig_scratch.release();
  dedup.release();
  api.release();
  api2.release();
  h2d_state.release();
  stage_sort.release();
  if (h2d) cudaStreamDestroy(h2d);
  if (d2h) cudaStreamDestroy(d2h);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

bool nd_ctx::gate_on() const {
  const char* v = getenv("ND_K1J_GATE");  // read per call (A/B runs in one process)
  const bool on = !(v && v[0] == '0');
  return on && fam.jit && fam.unit == 0;
}

ndb::K1Gate* nd_ctx::next_gate(ndb::K1Gate& g) {
  if (!gate_on()) return nullptr;
  if (!gate_flag.ptr) {
    ND_CUDA(cudaMemset(gate_flag.as<unsigned int>(1), 0, sizeof(unsigned int)));
    gate_epoch = 0;
  }
  g.flag = static_cast<unsigned int*>(gate_flag.ptr);
  g.epoch = ++gate_epoch;
  return &g;
}

void nd_ctx::ensure_streams() {
  if (h2d) return;
  ND_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
  ND_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
  for (int i = 0; i < kSlots; ++i) {
    ND_CUDA(cudaStreamCreateWithFlags(&slot[i].comp, cudaStreamNonBlocking));
    ND_CUDA(cudaEventCreateWithFlags(&slot[i].h2d_done, cudaEventDisableTiming));
    ND_CUDA(cudaEventCreateWithFlags(&slot[i].comp_done, cudaEventDisableTiming));
    ND_CUDA(cudaEventCreateWithFlags(&slot[i].d2h_done, cudaEventDisableTiming));
  }
}

void nd_ctx::ensure_ring_streams() {
  for (auto& r : ring_stream)
    if (!r) ND_CUDA(cudaStreamCreateWithFlags(&r, cudaStreamNonBlocking));
}

void nd_ctx::require_family() const {
  if (!fam.q) fail(ND_ERR_PREREQ, "no hash family uploaded (call nd_family_upload first)");
}

namespace ndb {

// Text per chunk of the host pipelines (nd_signatures, nd_dedup).  64 MB
// keeps the pipeline fill and drain short for the register-constant K1.
// K1j runs pass-major over the chunk's items and needs ~1e5 items per launch
// to occupy the GPU, so its chunks ramp up 64, 128, 256, 512 MB: the first
// copy still lands quickly, later launches are large.
uint64_t h2d_chunk_bytes(const DevFamily& fam, size_t chunk_index) {
  static const uint64_t first_mb = [] {
    const char* v = getenv("ND_H2D_FIRST_MB");  // tuning
    return v ? std::max(1, atoi(v)) : 48;  // 32 -> 48: C2 host e2e 70.6 -> 69.0 ms (mean)
  }();
  static const uint64_t max_mb = [] {
    const char* v = getenv("ND_H2D_MAX_MB");  // tuning
    return v ? std::max(1, atoi(v)) : 512;
  }();
  // growth per chunk in percent (ND_H2D_GROWTH, tuning): a chunk's copy must
  // land before the kernels of the chunks before it finish
  static const uint64_t growth = [] {
    const char* v = getenv("ND_H2D_GROWTH");
    return static_cast<uint64_t>(v ? std::max(110, std::min(400, atoi(v))) : 200);
  }();
  constexpr uint64_t kSmall = 64ull << 20;
  if (!fam.jit) return kSmall;
  uint64_t b = first_mb << 20;
  for (size_t c = 0; c < chunk_index && b < (max_mb << 20); ++c) b = b * growth / 100;
  return std::min<uint64_t>(max_mb << 20, b);
}

// Host-pipelined signatures: chunks of documents are copied in (h2d stream),
// signed on alternating compute streams, and copied out (d2h stream), so the
// PCIe transfers of chunk c+1 / c-1 overlap the kernel of chunk c (the
// paper's double buffering; reference slab queue
// pipeline.cpp:121-169).
void signatures_host(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                     uint32_t bands, uint32_t rows, uint32_t K, uint32_t* sig_out,
                     uint32_t* band_out) {
  ctx->require_family();
  const uint32_t H = ctx->fam.H;
  const uint32_t L = ctx->fam.L;
  if (n == 0) return;
  if (band_out && (bands == 0 || rows == 0 || static_cast<uint64_t>(bands) * rows != H))
    fail(ND_ERR_CONFIG, "signature has " + std::to_string(H) + " values, banding needs " +
                            std::to_string(bands) + "*" + std::to_string(rows));
  // a bad document stops the run after the chunks already issued have
  // drained (no copy into the caller's buffers after the error returns)
  auto drain_and_fail = [&](int code, const std::string& msg) {
    if (ctx->h2d) {
      cudaStreamSynchronize(ctx->h2d);
      for (auto& sl : ctx->slot) cudaStreamSynchronize(sl.comp);
      cudaStreamSynchronize(ctx->d2h);
    }
    fail(code, msg);
  };
  auto check_docs = [&](uint64_t a, uint64_t b) {
    for (uint64_t i = a; i < b; ++i) {
      if (offsets[i + 1] < offsets[i]) drain_and_fail(ND_ERR_CONFIG, "offsets must be non-decreasing");
      if (offsets[i + 1] - offsets[i] < L)
        drain_and_fail(ND_ERR_SHORT, "document " + std::to_string(i) + " has " +
                                         std::to_string(offsets[i + 1] - offsets[i]) +
                                         " units, needs " + std::to_string(L));
    }
  };
  // the offsets are checked chunk by chunk as the chunks are issued (the
  // first copy starts after one chunk's worth of host work, not n's); the
  // chunk boundaries need them ascending, checked once, cheaply, up front
  if (offsets[n] < offsets[0]) fail(ND_ERR_CONFIG, "offsets must be non-decreasing");
  ctx->ensure_streams();
  cudaEvent_t start;
  ND_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  ND_CUDA(cudaEventRecord(start, ctx->stream));
  ND_CUDA(cudaStreamWaitEvent(ctx->h2d, start, 0));

  // chunking: <= chunk_bytes(c) of text and <= kChunkDocs documents per chunk
  // (binary search over the offsets; a longer document is a chunk of its own)
  constexpr uint64_t kChunkDocs = 1ull << 20;
  // ramp down at the end (ND_H2D_TAIL_DIV=d, default 2: a chunk takes at
  // most 1/d of the text left, down to the first chunk's size) so the last
  // copy out is short; with the chunk gate the extra launches' tails overlap
  // (C2 shard: 74.7 -> 72.1 ms; without the gate no faster)
  const uint64_t tail_div = [] {
    const char* v = getenv("ND_H2D_TAIL_DIV");
    return static_cast<uint64_t>(v ? std::max(0, atoi(v)) : 2);
  }();
  const uint64_t first_cap = h2d_chunk_bytes(ctx->fam, 0);
  const bool gated = ctx->gate_on();
  auto chunk_end = [&](uint64_t d0, size_t index) {
    uint64_t cap = h2d_chunk_bytes(ctx->fam, index);
    if (tail_div && ctx->fam.jit && gated)
      cap = std::min(cap, std::max(first_cap, (offsets[n] - offsets[d0]) / tail_div));
    const uint64_t lim = std::min(n, d0 + kChunkDocs);
    // largest d1 in (d0, lim] with offsets[d1] - offsets[d0] <= cap
    const uint64_t* it = std::upper_bound(offsets + d0 + 1, offsets + lim + 1, offsets[d0] + cap);
    return std::max<uint64_t>(d0 + 1, static_cast<uint64_t>(it - offsets) - 1);
  };
  // slot buffers sized for the largest chunk the ramp can produce
  uint64_t max_docs = 0, max_bytes = 0;
  {
    uint64_t d0 = 0;
    for (size_t c = 0; d0 < n; ++c) {
      const uint64_t d1 = chunk_end(d0, c);
      if (offsets[d1] < offsets[d0]) fail(ND_ERR_CONFIG, "offsets must be non-decreasing");
      max_docs = std::max(max_docs, d1 - d0);
      max_bytes = std::max(max_bytes, offsets[d1] - offsets[d0]);
      d0 = d1;
    }
  }
  // slots in flight: with three, chunk c+3's copy in waits only for chunk
  // c's results to leave, so the copies run ahead of the kernels through the
  // ramp (ND_H2D_SLOTS=2: double buffering)
  static const int nslots = [] {
    const char* v = getenv("ND_H2D_SLOTS");
    return v ? std::max(2, std::min(nd_ctx::kSlots, atoi(v))) : nd_ctx::kSlots;
  }();
  uint64_t* hoff = static_cast<uint64_t*>(
      ctx->pinned_off.get(nslots * (max_docs + 1) * sizeof(uint64_t)));
  bool first_use[nd_ctx::kSlots] = {true, true, true};
  // ND_PIPE_TRACE=1: per chunk, device times (ms from the call's start) of
  // copy in / kernel / copy out, on stderr
  const bool trace = [] {
    const char* v = getenv("ND_PIPE_TRACE");
    return v && v[0] == '1';
  }();
  struct Tr { cudaEvent_t e[6]; uint64_t bytes; };
  std::vector<Tr> tr;
  cudaEvent_t t0ev = nullptr;
  if (trace) {
    ND_CUDA(cudaEventCreate(&t0ev));
    ND_CUDA(cudaEventRecord(t0ev, ctx->stream));
  }
  auto mark = [&](size_t c, int k, cudaStream_t st) {
    if (!trace) return;
    if (tr.size() <= c) {
      tr.resize(c + 1);
      for (auto& e : tr[c].e) cudaEventCreate(&e);
    }
    cudaEventRecord(tr[c].e[k], st);
  };
  uint64_t next_d0 = 0;
  for (size_t c = 0; next_d0 < n; ++c) {
    const int si = static_cast<int>(c % nslots);
    auto& sl = ctx->slot[si];
    const uint64_t d0 = next_d0, d1 = chunk_end(d0, c), m = d1 - d0;
    next_d0 = d1;
    check_docs(d0, d1);
    const uint64_t tb = offsets[d1] - offsets[d0];
    uint8_t* dtext = sl.text.as<uint8_t>(max_bytes + 16);
    uint64_t* doff = sl.off.as<uint64_t>(max_docs + 1);
    uint32_t* dsig = sl.sig.as<uint32_t>(max_docs * H);
    uint32_t* dband = band_out ? sl.band.as<uint32_t>(max_docs * bands) : nullptr;
    uint64_t* ho = hoff + si * (max_docs + 1);
    // the slot is free once its previous chunk's results left the device
    if (!first_use[si]) {
      ND_CUDA(cudaEventSynchronize(sl.d2h_done));  // host offsets buffer reuse
      ND_CUDA(cudaStreamWaitEvent(ctx->h2d, sl.d2h_done, 0));
    }
    first_use[si] = false;
    for (uint64_t i = 0; i <= m; ++i) ho[i] = offsets[d0 + i] - offsets[d0];
    mark(c, 0, ctx->h2d);
    ND_CUDA(cudaMemcpyAsync(dtext, bytes + offsets[d0], tb, cudaMemcpyHostToDevice, ctx->h2d));
    ND_CUDA(cudaMemcpyAsync(doff, ho, (m + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->h2d));
    ND_CUDA(cudaEventRecord(sl.h2d_done, ctx->h2d));
    mark(c, 1, ctx->h2d);
    if (trace) tr[c].bytes = tb;
    // K1j chunks: two pass-major launches side by side would interleave
    // their passes' code, so chunk c+1 is gated (K1Gate) until chunk c's
    // first warp enters its last pass, on the other of two streams; the next
    // launch then fills the SMs the last pass frees (ND_K1J_GATE=0: one
    // stream, launches back to back; ND_K1J_SIG_STREAMS=3: ungated streams)
    static const bool per_slot = [] {
      const char* v = getenv("ND_K1J_SIG_STREAMS");
      return v && v[0] == '3';
    }();
    K1Gate gate_buf;
    K1Gate* gate = ctx->fam.jit && !per_slot ? ctx->next_gate(gate_buf) : nullptr;
    cudaStream_t comp = !ctx->fam.jit || per_slot ? sl.comp
                        : gate                   ? ctx->slot[c & 1].comp
                                                 : ctx->slot[0].comp;
    ND_CUDA(cudaStreamWaitEvent(comp, sl.h2d_done, 0));
    if (gate && c > 0) k1_gate_wait(gate->flag, gate->epoch - 1, comp);
    mark(c, 2, comp);
    launch_signatures(ctx->fam, dtext, doff, m, bands, rows, K, dsig, dband, sl.scratch,
                      comp, /*check_short=*/false, ho, gate);
    ND_CUDA(cudaEventRecord(sl.comp_done, comp));
    mark(c, 3, comp);
    ND_CUDA(cudaStreamWaitEvent(ctx->d2h, sl.comp_done, 0));
    mark(c, 4, ctx->d2h);
    ND_CUDA(cudaMemcpyAsync(sig_out + d0 * H, dsig, m * H * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, ctx->d2h));
    if (band_out)
      ND_CUDA(cudaMemcpyAsync(band_out + d0 * bands, dband, m * bands * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, ctx->d2h));
    ND_CUDA(cudaEventRecord(sl.d2h_done, ctx->d2h));
    mark(c, 5, ctx->d2h);
  }
  if (trace) {
    ND_CUDA(cudaStreamSynchronize(ctx->d2h));
    for (size_t c = 0; c < tr.size(); ++c) {
      float t[6];
      for (int k = 0; k < 6; ++k) cudaEventElapsedTime(&t[k], t0ev, tr[c].e[k]);
      fprintf(stderr, "chunk %zu %6.1f MB  in %7.2f-%7.2f  k1 %7.2f-%7.2f  out %7.2f-%7.2f ms\n", c,
              tr[c].bytes / 1048576.0, t[0], t[1], t[2], t[3], t[4], t[5]);
      for (auto& e : tr[c].e) cudaEventDestroy(e);
    }
    cudaEventDestroy(t0ev);
  }
  cudaEvent_t end;
  ND_CUDA(cudaEventCreateWithFlags(&end, cudaEventDisableTiming));
  ND_CUDA(cudaEventRecord(end, ctx->d2h));
  ND_CUDA(cudaStreamWaitEvent(ctx->stream, end, 0));
  ND_CUDA(cudaStreamSynchronize(ctx->d2h));
  cudaEventDestroy(start);
  cudaEventDestroy(end);
}

}  // namespace ndb

using namespace ndb;

extern "C" {

const char* nd_version(void) { return "neardup_b200 0.1 (sm_100a)"; }
uint64_t nd_launch_count(void) { return g_launches.load(); }
const char* nd_last_error_global(void) { return g_error.c_str(); }

int nd_derive_family(uint64_t seed, uint32_t H, uint32_t L, uint32_t unit, nd_hash_fn* out) {
  return guarded_impl(nullptr, [&] {
    if (!out) fail(ND_ERR_CONFIG, "null output");
    std::vector<nd_hash_fn> fam = derive_family(seed, H, L, unit);
    std::memcpy(out, fam.data(), fam.size() * sizeof(nd_hash_fn));
  });
}

int nd_mod_pow(uint64_t base, uint64_t exp, uint64_t mod, uint64_t* out) {
  return guarded_impl(nullptr, [&] { *out = mod_pow_checked(base, exp, mod); });
}

int nd_is_prime_u32(uint32_t n) { return is_prime(n) ? 1 : 0; }

int nd_hash_window_direct(const uint32_t* window, uint32_t len, const nd_hash_fn* f,
                          uint32_t* out) {
  return guarded_impl(nullptr, [&] { *out = hash_window_direct(window, len, *f); });
}

uint32_t nd_roll_next(uint32_t state, uint32_t outgoing, uint32_t incoming, const nd_hash_fn* f) {
  return roll_next(state, outgoing, incoming, *f);
}

int nd_choose_bucket_count(uint64_t n, uint64_t num, uint64_t den, uint32_t* out) {
  return guarded_impl(nullptr, [&] { *out = choose_bucket_count(n, num, den); });
}

uint32_t nd_min_matches(uint32_t H, uint64_t num, uint64_t den) { return min_matches(H, num, den); }

int nd_band_partition(uint32_t bands, uint32_t workers, uint32_t* ranges) {
  return guarded_impl(nullptr, [&] {
    if (workers == 0) fail(ND_ERR_CONFIG, "worker count must be positive");
    uint32_t cursor = 0;
    for (uint32_t w = 0; w < workers; ++w) {
      uint32_t len = bands / workers + (w < bands % workers ? 1 : 0);
      ranges[2 * w] = cursor;
      ranges[2 * w + 1] = cursor + len;
      cursor += len;
    }
  });
}

int nd_cell_partition(uint32_t bands, uint32_t K, uint32_t shards, uint64_t* first_cell) {
  return guarded_impl(nullptr, [&] {
    if (shards == 0) fail(ND_ERR_CONFIG, "shard count must be positive");
    uint64_t cells = static_cast<uint64_t>(bands) * K;
    for (uint32_t g = 0; g <= shards; ++g)
      first_cell[g] = static_cast<uint64_t>((static_cast<unsigned __int128>(cells) * g + shards - 1) / shards);
  });
}

int nd_synth_generate(const nd_synth_spec* spec, uint8_t* bytes, uint64_t* offsets,
                      uint64_t* nbytes_out) {
  return guarded_impl(nullptr, [&] { synth_generate(*spec, bytes, offsets, nbytes_out); });
}

int nd_synth_text_device(nd_ctx* ctx, const nd_synth_spec* spec, const uint64_t* d_offsets,
                         uint8_t* d_bytes) {
  return guarded_impl(ctx, [&] { synth_text_device(*spec, d_offsets, d_bytes, ctx->synth_buf, ctx->stream); });
}

int nd_ctx_create(int device, nd_ctx** out) {
  return guarded_impl(nullptr, [&] {
    int count = 0;
    ND_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(ND_ERR_DEVICE, "no such CUDA device");
    ND_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    ND_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(ND_ERR_DEVICE, "neardup_b200 requires an sm_100 (Blackwell) device");
    auto* ctx = new nd_ctx();
    ctx->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete ctx;
      fail(ND_ERR_DEVICE, cudaGetErrorString(e));
    }
    ctx->own_stream = true;
    *out = ctx;
  });
}

void nd_ctx_destroy(nd_ctx* ctx) {
  if (!ctx) return;
  for (nd_ctx* c : ctx->shards) nd_ctx_destroy(c);
  ctx->shards.clear();
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  delete ctx;
}

const char* nd_last_error(const nd_ctx* ctx) { return ctx ? ctx->err.c_str() : g_error.c_str(); }

int nd_ctx_set_stream(nd_ctx* ctx, void* stream) {
  return guarded_impl(ctx, [&] {
    if (ctx->own_stream && ctx->stream) {
      ND_CUDA(cudaStreamSynchronize(ctx->stream));
      ND_CUDA(cudaStreamDestroy(ctx->stream));
    }
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
      ctx->own_stream = false;
    } else {
      ND_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
  });
}

int nd_family_upload(nd_ctx* ctx, const nd_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit) {
  return guarded_impl(ctx, [&] {
    family_upload_one(ctx, fns, H, L, unit);
    if (is_group(ctx)) multi_family_upload(ctx, fns, H, L, unit);
  });
}

}  // extern "C"

namespace ndb {
void family_upload_one(nd_ctx* ctx, const nd_hash_fn* fns, uint32_t H, uint32_t L, uint32_t unit) {
  {
    if (H == 0 || L == 0) fail(ND_ERR_CONFIG, "hash count and shingle length must be positive");
    if (unit > 1) fail(ND_ERR_CONFIG, "unknown shingle unit");
    if (L > 64) fail(ND_ERR_CONFIG, "shingle length above 64 is not supported on the GPU path");
    uint32_t Hp = 32;
    while (Hp < H) Hp *= 2;
    if (Hp > 512) fail(ND_ERR_CONFIG, "hash count above 512 is not supported on the GPU path");
    // Validate every function against the reference's own preconditions.
    // roll_next (minhash.cpp:121-131) is the exact window hash only when the
    // units are residues (minhash.cpp:107-109: "units < 2^21 <= modulus") and
    // base_inverse / base_power / reduce_factor are the constants derive_family
    // computes (minhash.cpp:99-101); a hand-built HashFunctionParams (a public
    // struct) that breaks them makes the reference compute something other
    // than the window hash, which no exact GPU evaluation can reproduce.
    bool fast = true;
    bool narrow = unit == 1;  // codepoint family inside the byte fq domain
    for (uint32_t i = 0; i < H; ++i) {
      const nd_hash_fn& f = fns[i];
      const uint64_t p = f.modulus;
      const uint64_t max_unit = unit == 1 ? 0x10FFFF : 0xFF;
      if (p <= max_unit)
        fail(ND_ERR_CONFIG, std::string("hash function ") + std::to_string(i) + ": modulus " +
                                std::to_string(p) + " does not exceed the largest " +
                                (unit == 1 ? "code point" : "byte") +
                                " unit (units must be residues, minhash.cpp:107-109)");
      if (p >= (1ull << 31))
        fail(ND_ERR_CONFIG, "hash function " + std::to_string(i) +
                                ": modulus must be below 2^31 on the GPU path");
      const uint64_t q = f.base % p;
      if (q * (f.base_inverse % p) % p != 1)
        fail(ND_ERR_CONFIG, "hash function " + std::to_string(i) +
                                ": base_inverse is not the inverse of base mod modulus");
      uint64_t qpow = 1;
      for (uint32_t e = 1; e < L; ++e) qpow = qpow * q % p;
      if (f.base_power != qpow)
        fail(ND_ERR_CONFIG, "hash function " + std::to_string(i) +
                                ": base_power is not base^(L-1) mod modulus");
      if (f.reduce_factor !=
          static_cast<uint64_t>((static_cast<unsigned __int128>(1) << 64) / p))
        fail(ND_ERR_CONFIG, "hash function " + std::to_string(i) +
                                ": reduce_factor is not floor(2^64 / modulus)");
      const uint64_t p_lo = unit == 1 ? 0x110000ull : (1ull << 21);
      if (p < p_lo || p >= (1ull << 23) || f.base == 0 || f.base >= (1u << 16)) fast = false;
      if (p < (1ull << 21) || p >= (1ull << 23) || f.base == 0 || f.base >= (1u << 16))
        narrow = false;
    }
    const char* fe = getenv("ND_K1_EXACT");  // 1: exact arithmetic for every family (tests)
    if (fe && fe[0] == '1') fast = false;
    // 9 arrays of Hp entries: q, QLn, M, -p, c3 (u32), q/p, QLn/p, c1e (f32), M45 (u32),
    // then p (u32) and reduce_factor (u64, 8-byte aligned: Hp is even)
    std::vector<uint32_t> host(12 * Hp);
    for (uint32_t i = 0; i < Hp; ++i) {
      const nd_hash_fn& f = fns[i < H ? i : 0];  // pad with copies of fn 0 (never stored)
      uint64_t p = f.modulus;
      host[9 * Hp + i] = static_cast<uint32_t>(p);
      std::memcpy(&host[10 * Hp + 2 * i], &f.reduce_factor, 8);
      if (!fast) {  // exact variant: q (reduced) and QLn only
        const uint64_t q = f.base % p;
        host[i] = static_cast<uint32_t>(q);
        host[Hp + i] = static_cast<uint32_t>((p - static_cast<uint64_t>(f.base_power) * q % p) % p);
        continue;
      }
      uint64_t qL = static_cast<uint64_t>(f.base_power) * f.base % p;  // q^L = q^(L-1) * q
      uint32_t qln = static_cast<uint32_t>((p - qL) % p);
      float qp = static_cast<float>(static_cast<double>(f.base) / static_cast<double>(p));
      float qlnp = static_cast<float>(static_cast<double>(qln) / static_cast<double>(p));
      float c1e = -std::ldexp(qp, 23) + 0.03125f;  // exact: ulp(2^23 qp) <= 2^-6
      host[i] = f.base;
      host[Hp + i] = qln;
      host[2 * Hp + i] = static_cast<uint32_t>((1ull << 40) / p);
      host[3 * Hp + i] = static_cast<uint32_t>(0u - static_cast<uint32_t>(p));
      host[4 * Hp + i] = static_cast<uint32_t>(0x4B000000ull * p);
      std::memcpy(&host[5 * Hp + i], &qp, 4);
      std::memcpy(&host[6 * Hp + i], &qlnp, 4);
      std::memcpy(&host[7 * Hp + i], &c1e, 4);
      host[8 * Hp + i] = static_cast<uint32_t>((1ull << 45) / p);
    }
    uint32_t* d = ctx->fam_buf.as<uint32_t>(12 * Hp);
    ND_CUDA(cudaMemcpy(d, host.data(), host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    ctx->fam.q = d;
    ctx->fam.qln = d + Hp;
    ctx->fam.m = d + 2 * Hp;
    ctx->fam.negp = d + 3 * Hp;
    ctx->fam.c3 = d + 4 * Hp;
    ctx->fam.qp = reinterpret_cast<float*>(d + 5 * Hp);
    ctx->fam.qlnp = reinterpret_cast<float*>(d + 6 * Hp);
    ctx->fam.c1e = reinterpret_cast<float*>(d + 7 * Hp);
    ctx->fam.m45 = d + 8 * Hp;
    ctx->fam.p = d + 9 * Hp;
    ctx->fam.rf = reinterpret_cast<unsigned long long*>(d + 10 * Hp);
    ctx->fam.exact = !fast;
    ctx->fam.narrow_ok = narrow && fast;
    ctx->fam.unit = unit;
    ctx->fam.H = H;
    ctx->fam.L = L;
    // K1j: compile (or find) the kernel specialised for this family; when
    // NVRTC is unavailable the register-constant K1 runs (same bits)
    ctx->fam.jit = nullptr;
    ctx->fam.jit16 = nullptr;
    ctx->k1_note.clear();
    if (k1_jit_eligible(ctx->fam)) {
      try {
        ctx->fam.jit = k1_jit_prepare(fns, H, L);
        // codepoint families: K1j over 16-bit units for documents whose code
        // points are all < 2^16 (ND_K1J_U16=0: those run K1w)
        const char* u16 = getenv("ND_K1J_U16");
        if (unit == 1 && !(u16 && u16[0] == '0')) ctx->fam.jit16 = k1_jit_prepare(fns, H, L, 2);
      } catch (const NdError& e) {
        ctx->k1_note = e.what();
      }
    }
    ctx->fam.H = H;
    ctx->fam.Hp = Hp;
    ctx->fam.L = L;
    ctx->family_host.assign(fns, fns + H);
    ctx->family_derived = false;
  }
}
}  // namespace ndb

extern "C" {

const char* nd_k1_kernel(nd_ctx* ctx) {
  static thread_local std::string out;
  if (is_group(ctx)) ctx = ctx->shards[0];
  if (!ctx || !ctx->fam.q) return "";
  if (ctx->fam.exact) out = "k1x";
  else if (ctx->fam.unit == 1)
    out = ctx->fam.jit16 ? "k1j+k1j16+k1w" : ctx->fam.jit ? "k1j+k1w" : ctx->fam.narrow_ok ? "k1+k1w" : "k1w";
  else out = ctx->fam.jit ? "k1j" : "k1";
  if (!ctx->k1_note.empty()) out += ": " + ctx->k1_note;
  return out.c_str();
}

const char* nd_dedup_compare_kind(nd_ctx* ctx) {
  if (!ctx) return "";
  if (is_group(ctx)) return ctx->multi.last_valid ? ctx->shards[0]->dedup.compare_kind : "";
  return ctx->dedup.valid ? ctx->dedup.compare_kind : "";
}

int nd_signatures(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                  uint32_t bands, uint32_t rows, uint32_t K, uint32_t* sig_out,
                  uint32_t* band_out) {
  return guarded_impl(ctx, [&] {
    if (is_group(ctx)) {
      ctx->require_family();
      multi_signatures(ctx, bytes, offsets, n, bands, rows, K, sig_out, band_out);
      return;
    }
    signatures_host(ctx, bytes, offsets, n, bands, rows, K, sig_out, band_out);
  });
}

int nd_text_units(nd_ctx* ctx, const uint8_t* bytes, const uint64_t* offsets, uint64_t n,
                  uint32_t unit, uint64_t* unit_offsets, uint32_t* units_out) {
  return guarded_impl(ctx, [&] {
    if (unit > 1) fail(ND_ERR_CONFIG, "unknown shingle unit");
    if (!unit_offsets) fail(ND_ERR_CONFIG, "null unit_offsets");
    for (uint64_t i = 0; i < n; ++i)
      if (offsets[i + 1] < offsets[i]) fail(ND_ERR_CONFIG, "offsets must be non-decreasing");
    const uint64_t nb = n ? offsets[n] - offsets[0] : 0;
    if (unit == 0) {  // byte units: the counts are the lengths
      for (uint64_t i = 0; i <= n; ++i) unit_offsets[i] = offsets[i] - offsets[0];
      if (units_out)
        for (uint64_t i = 0; i < nb; ++i) units_out[i] = bytes[offsets[0] + i];
      return;
    }
    unit_offsets[0] = 0;
    if (n == 0) return;
    cudaStream_t s = ctx->stream;
    uint8_t* dt = ctx->sig_in_text.as<uint8_t>(nb + 16);
    uint64_t* doff = ctx->sig_in_off.as<uint64_t>(n + 1);
    std::vector<uint64_t> rel(n + 1);
    for (uint64_t i = 0; i <= n; ++i) rel[i] = offsets[i] - offsets[0];
    ND_CUDA(cudaMemcpyAsync(dt, bytes + offsets[0], nb, cudaMemcpyHostToDevice, s));
    ND_CUDA(cudaMemcpyAsync(doff, rel.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    const uint32_t* units = nullptr;
    const uint64_t* uoff = nullptr;
    SigScratch& sc = ctx->sig_scratch;
    decode_codepoints_device(dt, doff, n, sc.units, sc.unit_off, sc.unit_cnt, sc.scan_tmp, s,
                             &units, &uoff);
    ND_CUDA(cudaMemcpyAsync(unit_offsets, uoff, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
    if (units_out && unit_offsets[n])
      ND_CUDA(cudaMemcpyAsync(units_out, units, unit_offsets[n] * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, s));
    ND_CUDA(cudaStreamSynchronize(s));
  });
}

int nd_signatures_device(nd_ctx* ctx, const uint8_t* d_bytes, const uint64_t* d_offsets,
                         uint64_t n, uint32_t bands, uint32_t rows, uint32_t K, uint32_t* d_sig,
                         uint32_t* d_band) {
  return guarded_impl(ctx, [&] {
    ctx->require_family();
    if (d_band && (bands == 0 || rows == 0 || static_cast<uint64_t>(bands) * rows != ctx->fam.H))
      fail(ND_ERR_CONFIG, "banding shape does not match the hash count");
    launch_signatures(ctx->fam, d_bytes, d_offsets, n, bands, rows, K, d_sig, d_band,
                      ctx->sig_scratch, ctx->stream, /*check_short=*/true, nullptr);
  });
}

}  // extern "C"
