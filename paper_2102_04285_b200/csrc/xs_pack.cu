// xs_pack.cu -- widen the packed upload format (include/xstrace_b200.h,
// xs_packed_t) into the engine's columnar layout, on the device.
//
// The host keeps a trace in pinned memory in the narrowest exact widths
// (ColumnarTrace.pinned, columnar.py): the PCIe upload is the e2e bottleneck
// at 1M events (38 B/event at ~55 GB/s is ~0.7 ms against a ~0.9 ms
// analysis), so the wire carries ~17-22 B/event and this kernel -- one HBM
// pass, ~60 B/event of traffic -- restores the 38-byte columns.  Values are
// reproduced bit for bit (the host only narrows a column when every value
// fits), so parity with the reference is unaffected.
#include "xs_engine.cuh"

namespace xs {

__device__ __forceinline__ int64_t ld_index(const void* p, int w, int64_t i) {
  if (w == 1) return ((const uint8_t*)p)[i];
  if (w == 2) return ((const uint16_t*)p)[i];
  return ((const int32_t*)p)[i];
}

__device__ __forceinline__ int64_t ld_wide(const void* p, int w, int64_t i) {
  if (w == 4) return (int64_t)((const uint32_t*)p)[i];
  return ((const int64_t*)p)[i];
}

__global__ void __launch_bounds__(XS_BLOCK) k_unpack(xs_packed_t pk, int64_t* start, int64_t* dur, int32_t* pid,
                                                     int32_t* tid, uint8_t* cat, int32_t* name, int64_t* corr,
                                                     uint8_t* has_corr) {
  const int64_t blk0 = pk.row0 >> 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pk.n; i += (int64_t)gridDim.x * blockDim.x) {
    if (pk.start_w == 4)
      start[i] = pk.start_base[((pk.row0 + i) >> 8) - blk0] + (int64_t)((const uint32_t*)pk.start)[i];
    else
      start[i] = ((const int64_t*)pk.start)[i];
    dur[i] = ld_wide(pk.dur, pk.dur_w, i);
    pid[i] = (int32_t)ld_index(pk.pid, pk.pid_w, i);
    tid[i] = (int32_t)ld_index(pk.tid, pk.tid_w, i);
    name[i] = (int32_t)ld_index(pk.name, pk.name_w, i);
    corr[i] = ld_wide(pk.corr, pk.corr_w, i);
    const uint8_t cf = pk.catf[i];
    cat[i] = cf & 0x7f;
    has_corr[i] = cf >> 7;
  }
}

// values that did not fit their 32-bit slot, scattered after the widening
__global__ void k_unpack_exc(xs_packed_t pk, int64_t* start, int64_t* dur, int64_t* corr) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < pk.n_exc;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = pk.exc_row[j] - pk.row0;
    if (r < 0 || r >= pk.n) continue;
    const int c = pk.exc_col[j];
    int64_t* dst = c == 0 ? start : c == 1 ? dur : corr;
    dst[r] = pk.exc_val[j];
  }
}

}  // namespace xs

using namespace xs;

extern "C" int xs_unpack(xs_ctx_t* ctx, const xs_packed_t* pk, int64_t* start, int64_t* dur, int32_t* pid,
                         int32_t* tid, uint8_t* cat, int32_t* name, int64_t* corr, uint8_t* has_corr,
                         xs_stream_t stream) {
  if (!ctx || !pk || pk->n < 0) return XS_BAD_ARGUMENT;
  auto idx_ok = [](int w) { return w == 1 || w == 2 || w == 4; };
  auto wide_ok = [](int w) { return w == 4 || w == 8; };
  if (!wide_ok(pk->start_w) || !wide_ok(pk->dur_w) || !wide_ok(pk->corr_w) || !idx_ok(pk->pid_w) ||
      !idx_ok(pk->tid_w) || !idx_ok(pk->name_w) || (pk->start_w == 4 && !pk->start_base) ||
      (pk->n_exc > 0 && (!pk->exc_row || !pk->exc_val || !pk->exc_col)))
    return XS_BAD_ARGUMENT;
  if (pk->n == 0) return XS_OK;
  cudaSetDevice(ctx->device);
  const int grid = (int)std::min<int64_t>(grid_for(pk->n), (int64_t)148 * 8);
  XS_LAUNCH(ctx, k_unpack, grid, XS_BLOCK, 0, (cudaStream_t)stream, *pk, start, dur, pid, tid, cat, name, corr,
            has_corr);
  if (pk->n_exc > 0)
    XS_LAUNCH(ctx, k_unpack_exc, (int)std::min<int64_t>(grid_for(pk->n_exc), 1184), XS_BLOCK, 0,
              (cudaStream_t)stream, *pk, start, dur, corr);
  return XS_OK;
}
