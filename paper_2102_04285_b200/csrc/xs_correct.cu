// xs_correct.cu -- placeholder (correction pipeline lands next)
#include "xs_engine.cuh"
namespace xs {
int stage_transitions(xs_ctx* ctx, const EventView&, int, int, cudaStream_t) {
  ctx->err = "not yet built";
  return XS_UNSUPPORTED;
}
int stage_correct(xs_ctx* ctx, const EventView&, const xs_profile_t*, int64_t*, int64_t*, bool, cudaStream_t) {
  ctx->err = "not yet built";
  return XS_UNSUPPORTED;
}
}  // namespace xs
extern "C" {
int xs_transition_sites(xs_ctx_t* ctx, const xs_events_t*, int, int64_t*, xs_stream_t) { return XS_UNSUPPORTED; }
int xs_transition_fetch(xs_ctx_t* ctx, int32_t*, int64_t*, xs_stream_t) { return XS_UNSUPPORTED; }
int xs_remap(xs_ctx_t* ctx, int64_t, const int32_t*, const int64_t*, int64_t*, xs_stream_t) { return XS_UNSUPPORTED; }
}
