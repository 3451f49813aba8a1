// C-ABI of the compare / union / dedup stages (filled in by k_cells.cu,
// k_compare.cu, k_pairs.cu, k_components.cu).
#include "nd_capi_impl.cuh"

using namespace ndb;

extern "C" {

int nd_compare_cells(nd_ctx* ctx, const uint32_t*, uint64_t, uint32_t, const uint64_t*,
                     const uint32_t*, uint64_t, uint64_t, uint64_t, uint64_t*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_pairs_fetch(nd_ctx* ctx, uint32_t*, uint32_t*, uint32_t*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_union(nd_ctx* ctx, const uint32_t*, const uint32_t*, uint64_t, uint32_t, uint64_t*,
             uint64_t*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_groups_fetch(nd_ctx* ctx, uint32_t*, uint64_t*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_dedup(nd_ctx* ctx, const uint8_t*, const uint64_t*, const uint64_t*, uint64_t,
             const nd_params*, nd_dedup_stats*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_dedup_device(nd_ctx* ctx, const uint8_t*, const uint64_t*, const uint64_t*, uint64_t,
                    const nd_params*, nd_dedup_stats*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_dedup_fetch_pairs(nd_ctx* ctx, uint64_t*, uint64_t*, uint32_t*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_dedup_fetch_groups(nd_ctx* ctx, uint64_t*, uint64_t*) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}
int nd_dedup_write_report(nd_ctx* ctx, const char*, uint64_t) {
  return guarded_impl(ctx, [&] { fail(ND_ERR_INTERNAL, "not implemented"); });
}

}  // extern "C"
