// Host-to-host *_L product (linalg.py:34-43) as one pipelined native call.
//
// The numpy-in / numpy-out l_product is bound by the host link, not by the
// 50 us of device work: the inputs (A, B) must come in and C must go out.  The
// rows of A (and of C) are independent, so A is cut into row chunks and three
// streams overlap the link in both directions with the compute:
//   copy_in  : B, then A chunk 0, 1, ...                      (host -> device)
//   compute  : K1(B); per chunk K1(A_c) -> K2 -> K1'(C_c)     (ctx->stream)
//   copy_out : C chunk 0, 1, ...                              (device -> host)
// With pinned host buffers the end-to-end time approaches max(in, out) + one
// chunk; with pageable buffers the copies serialise but stay correct.
#include <algorithm>

#include "ltb_dispatch.cuh"

namespace {

int ensure_copy_streams(ltb_ctx* ctx) {
  if (!ctx->copy_in) LTB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
  if (!ctx->copy_out) LTB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
  return LTB_OK;
}

struct EventPool {  // events of one call, destroyed on exit
  cudaEvent_t ev[64];
  int n = 0;
  ~EventPool() {
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
  cudaEvent_t make() {
    cudaEvent_t e = nullptr;
    if (n < 64 && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) ev[n++] = e;
    return e;
  }
};

}  // namespace

int g_lprod_chunks = 8;  // maximum row chunks (test / tuning hook)
extern "C" void ltb_debug_set_lprod_chunks(int v) { g_lprod_chunks = v < 1 ? 1 : v; }

extern "C" int ltb_l_product_host(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype,
                                  const void* h_a, const void* h_b, void* h_c) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  if (I1 < 0 || L < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "l_product: negative dimension");
  if ((dtype != LTB_F32 && dtype != LTB_F64) || spec->is_complex || spec->nmodes == 0)
    return LTB_EUNSUPPORTED;  // complex transform domains take the generic path (real-output check)
  const int64_t P = spec->P;
  if (I1 == 0 || I2 == 0 || P == 0) return LTB_OK;
  const size_t es = dtype == LTB_F32 ? 4 : 8;
  LTB_TRY(ensure_copy_streams(ctx));
  // row chunks of A / C: up to 8, at least 32 rows each (the tensor-core GEMM tile side)
  const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(g_lprod_chunks, I1 / 32));
  const int64_t rows = (I1 + nch - 1) / nch;
  void *dA = nullptr, *dB = nullptr, *hA = nullptr, *hB = nullptr, *hC = nullptr, *dC = nullptr;
  LTB_TRY(ltb_ws_alloc(ctx, es * I1 * L * P + 16, &dA));
  LTB_TRY(ltb_ws_alloc(ctx, es * L * I2 * P + 16, &dB));
  LTB_TRY(ltb_ws_alloc(ctx, es * I1 * L * P + 16, &hA));
  LTB_TRY(ltb_ws_alloc(ctx, es * L * I2 * P + 16, &hB));
  LTB_TRY(ltb_ws_alloc(ctx, es * I1 * I2 * P + 16, &hC));
  LTB_TRY(ltb_ws_alloc(ctx, es * I1 * I2 * P + 16, &dC));
  EventPool pool;
  cudaEvent_t ready = pool.make();  // the stream-ordered allocations above are usable everywhere
  if (!ready) return ltb_set_error(ctx, LTB_ECUDA, "l_product: event creation failed");
  LTB_CUDA_TRY(ctx, cudaEventRecord(ready, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_in, ready, 0));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_out, ready, 0));
  // B in, K1(B)
  cudaEvent_t eb = pool.make();
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(dB, h_b, es * L * I2 * P, cudaMemcpyHostToDevice, ctx->copy_in));
  LTB_CUDA_TRY(ctx, cudaEventRecord(eb, ctx->copy_in));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, eb, 0));
  LTB_TRY(ltb_transform_impl(ctx, spec, L * I2, 0, dtype, LTB_TUBE_MAJOR, dB, dtype, LTB_SLICE_MAJOR, hB, nullptr));
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t r0 = c * rows, r = std::min(rows, I1 - r0);
    if (r <= 0) break;
    cudaEvent_t ea = pool.make(), ec = pool.make();
    if (!ea || !ec) return ltb_set_error(ctx, LTB_ECUDA, "l_product: event creation failed");
    char* a_c = (char*)dA + es * r0 * L * P;
    char* ha_c = (char*)hA + es * r0 * L * P;  // chunk-major: chunk c's slice stack (P x r x L)
    char* hc_c = (char*)hC + es * r0 * I2 * P;
    char* c_c = (char*)dC + es * r0 * I2 * P;
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(a_c, (const char*)h_a + es * r0 * L * P, es * r * L * P,
                                      cudaMemcpyHostToDevice, ctx->copy_in));
    LTB_CUDA_TRY(ctx, cudaEventRecord(ea, ctx->copy_in));
    LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ea, 0));
    LTB_TRY(ltb_transform_impl(ctx, spec, r * L, 0, dtype, LTB_TUBE_MAJOR, a_c, dtype, LTB_SLICE_MAJOR, ha_c,
                               nullptr));
    LTB_TRY(ltb_gemm_impl(ctx, dtype, P, r, I2, L, LTB_OP_N, ha_c, L, r * L, LTB_OP_N, hB, I2, L * I2, hc_c, I2,
                          r * I2, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
    LTB_TRY(ltb_transform_impl(ctx, spec, r * I2, 1, dtype, LTB_SLICE_MAJOR, hc_c, dtype, LTB_TUBE_MAJOR, c_c,
                               nullptr));
    LTB_CUDA_TRY(ctx, cudaEventRecord(ec, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_out, ec, 0));
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync((char*)h_c + es * r0 * I2 * P, c_c, es * r * I2 * P, cudaMemcpyDeviceToHost,
                                      ctx->copy_out));
  }
  // join the copy streams back into the compute stream, release, wait for the host copy
  cudaEvent_t done_in = pool.make(), done_out = pool.make();
  LTB_CUDA_TRY(ctx, cudaEventRecord(done_in, ctx->copy_in));
  LTB_CUDA_TRY(ctx, cudaEventRecord(done_out, ctx->copy_out));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, done_in, 0));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, done_out, 0));
  for (void* p : {dA, dB, hA, hB, hC, dC}) ltb_ws_free(ctx, p);
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return LTB_OK;
}
