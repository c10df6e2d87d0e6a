// Host-to-host *_L product (linalg.py:34-43) as one pipelined native call.
//
// The numpy-in / numpy-out l_product is bound by the host link, not by the
// 50 us of device work: the inputs (A, B) must come in and C must go out.  The
// rows of A (and of C) are independent, so A is cut into row chunks and three
// streams overlap the link in both directions with the compute:
//   copy_in  : B, then A chunk 0, 1, ...                      (host -> device)
//   compute  : K1(B); per chunk K1(A_c) -> K2 -> K1'(C_c)     (ctx->stream)
//   copy_out : C chunk 0, 1, ...                              (device -> host)
// Pinned host buffers go straight to the DMA engines.  A pageable buffer (a
// plain numpy array, what the drop-in receives) is staged through a pinned
// per-context buffer: the host thread copies the next chunk in (8 threads)
// while the DMA of the previous one runs, and copies C out chunk by chunk as
// the device finishes it.  Every return path waits for both copy streams
// before releasing the workspace, so no DMA touches caller memory after the
// call returns, error or not.
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

namespace {
// Resources of one call.  The destructor runs on every return path: it waits for the
// copy streams (they may still read the caller's A / B or write C) and only then
// releases the stream-ordered workspace.
struct HostCall {
  ltb_ctx* ctx;
  void* ws[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  EventPool pool;
  explicit HostCall(ltb_ctx* c) : ctx(c) {}
  ~HostCall() {
    if (ctx->copy_in) cudaStreamSynchronize(ctx->copy_in);
    if (ctx->copy_out) cudaStreamSynchronize(ctx->copy_out);
    for (void* p : ws) ltb_ws_free(ctx, p);
  }
};

// host -> device of [off, off + n) of one operand: straight from pinned memory, else a
// multi-threaded copy into the pinned stage followed by the DMA from there
int copy_in_range(ltb_ctx* ctx, char* d, const char* h, char* stage, size_t off, size_t n) {
  if (stage) {
    ltb_host_copy(stage + off, h + off, n);
    h = stage;
  }
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(d + off, h + off, n, cudaMemcpyHostToDevice, ctx->copy_in));
  return LTB_OK;
}
}  // namespace

constexpr int g_lprod_chunks = 8;  // maximum row chunks

extern "C" int ltb_l_product_host(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype,
                                  const void* h_a, const void* h_b, void* h_c) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  if (I1 < 0 || L < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "l_product: negative dimension");
  if ((dtype != LTB_F32 && dtype != LTB_F64) || spec->is_complex || spec->nmodes == 0)
    return LTB_EUNSUPPORTED;  // complex transform domains take the generic path (real-output check)
  const int64_t P = spec->P;
  if (I1 == 0 || I2 == 0 || P == 0) return LTB_OK;
  const size_t es = dtype == LTB_F32 ? 4 : 8;
  const size_t bytes_a = es * I1 * L * P, bytes_b = es * L * I2 * P, bytes_c = es * I1 * I2 * P;
  LTB_TRY(ensure_copy_streams(ctx));
  HostCall call(ctx);
  // pageable operands: one pinned stage region each
  const bool pin_a = ltb_is_pinned(h_a), pin_b = ltb_is_pinned(h_b), pin_c = ltb_is_pinned(h_c);
  const size_t need = (pin_a ? 0 : bytes_a) + (pin_b ? 0 : bytes_b) + (pin_c ? 0 : bytes_c);
  char *st_a = nullptr, *st_b = nullptr, *st_c = nullptr;
  if (need) {
    void* base = nullptr;
    LTB_TRY(ltb_pinned_scratch(ctx, need, &base));
    char* q = (char*)base;
    if (!pin_a) st_a = q, q += bytes_a;
    if (!pin_b) st_b = q, q += bytes_b;
    if (!pin_c) st_c = q;
  }
  // row chunks of A / C: up to 8, at least 32 rows each (the tensor-core GEMM tile side)
  const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(g_lprod_chunks, I1 / 32));
  const int64_t rows = (I1 + nch - 1) / nch;
  void *&dA = call.ws[0], *&dB = call.ws[1], *&hA = call.ws[2], *&hB = call.ws[3], *&hC = call.ws[4],
       *&dC = call.ws[5];
  LTB_TRY(ltb_ws_alloc(ctx, bytes_a + 16, &dA));
  LTB_TRY(ltb_ws_alloc(ctx, bytes_b + 16, &dB));
  LTB_TRY(ltb_ws_alloc(ctx, bytes_a + 16, &hA));
  LTB_TRY(ltb_ws_alloc(ctx, bytes_b + 16, &hB));
  LTB_TRY(ltb_ws_alloc(ctx, bytes_c + 16, &hC));
  LTB_TRY(ltb_ws_alloc(ctx, bytes_c + 16, &dC));
  EventPool& pool = call.pool;
  cudaEvent_t ready = pool.make();  // the stream-ordered allocations above are usable everywhere
  if (!ready) return ltb_set_error(ctx, LTB_ECUDA, "l_product: event creation failed");
  LTB_CUDA_TRY(ctx, cudaEventRecord(ready, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_in, ready, 0));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->copy_out, ready, 0));
  // B in (in quarters when staged, so the host copy of one overlaps the DMA of the last), K1(B)
  cudaEvent_t eb = pool.make();
  {
    const int nb = st_b ? 4 : 1;
    const size_t per = ((bytes_b + nb - 1) / nb + 4095) & ~size_t(4095);
    for (size_t off = 0; off < bytes_b; off += per)
      LTB_TRY(copy_in_range(ctx, (char*)dB, (const char*)h_b, st_b, off, std::min(per, bytes_b - off)));
  }
  LTB_CUDA_TRY(ctx, cudaEventRecord(eb, ctx->copy_in));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, eb, 0));
  LTB_TRY(ltb_transform_impl(ctx, spec, L * I2, 0, dtype, LTB_TUBE_MAJOR, dB, dtype, LTB_SLICE_MAJOR, hB, nullptr));
  cudaEvent_t c_done[64];
  int64_t issued = 0;
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t r0 = c * rows, r = std::min(rows, I1 - r0);
    if (r <= 0) break;
    cudaEvent_t ea = pool.make(), ec = pool.make();
    if (!ea || !ec) return ltb_set_error(ctx, LTB_ECUDA, "l_product: event creation failed");
    char* a_c = (char*)dA + es * r0 * L * P;
    char* ha_c = (char*)hA + es * r0 * L * P;  // chunk-major: chunk c's slice stack (P x r x L)
    char* hc_c = (char*)hC + es * r0 * I2 * P;
    char* c_c = (char*)dC + es * r0 * I2 * P;
    LTB_TRY(copy_in_range(ctx, (char*)dA, (const char*)h_a, st_a, es * r0 * L * P, es * r * L * P));
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
    char* dst = st_c ? st_c : (char*)h_c;
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(dst + es * r0 * I2 * P, c_c, es * r * I2 * P, cudaMemcpyDeviceToHost,
                                      ctx->copy_out));
    if (st_c) {
      c_done[c] = pool.make();
      if (!c_done[c]) return ltb_set_error(ctx, LTB_ECUDA, "l_product: event creation failed");
      LTB_CUDA_TRY(ctx, cudaEventRecord(c_done[c], ctx->copy_out));
    }
    issued = c + 1;
  }
  // staged C: copy each chunk out of the pinned stage as soon as its DMA lands
  if (st_c) {
    for (int64_t c = 0; c < issued; ++c) {
      const int64_t r0 = c * rows, r = std::min(rows, I1 - r0);
      LTB_CUDA_TRY(ctx, cudaEventSynchronize(c_done[c]));
      ltb_host_copy((char*)h_c + es * r0 * I2 * P, st_c + es * r0 * I2 * P, es * r * I2 * P);
    }
  }
  // join the copy streams back into the compute stream (the workspace is released behind them)
  cudaEvent_t done_in = pool.make(), done_out = pool.make();
  LTB_CUDA_TRY(ctx, cudaEventRecord(done_in, ctx->copy_in));
  LTB_CUDA_TRY(ctx, cudaEventRecord(done_out, ctx->copy_out));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, done_in, 0));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, done_out, 0));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return LTB_OK;
}

// ---------------------------------------------------------------- device-resident product
// l_product (linalg.py:34-43) on device buffers: the fused one-launch kernel for fp32 real
// specs (ltb_lprod_fused.cuh), otherwise K1(A), K1(B), K2, K1' through the workspace.
extern "C" int64_t ltb_l_product_ws_bytes(const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype) {
  if (!spec || I1 < 0 || L < 0 || I2 < 0) return 0;
  const int64_t P = spec->P;
  const int64_t hs = dtype_size(spec->is_complex ? (dtype_is_double(dtype) ? LTB_C128 : LTB_C64) : dtype);
  const int64_t three = hs * P * (I1 * L + L * I2 + I1 * I2) + 256;
  return std::max<int64_t>(three, dtype == LTB_F32 ? ltb_lprod_fused_ws_bytes(P, I1, L, I2) : 0);
}

extern "C" int ltb_l_product_device(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, int dtype,
                                    const void* d_a, const void* d_b, void* d_c, void* d_ws, int64_t ws_bytes,
                                    int fused) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  if (I1 < 0 || L < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "l_product: negative dimension");
  if (dtype != LTB_F32 && dtype != LTB_F64) return ltb_set_error(ctx, LTB_EPARAM, "l_product: real dtype expected");
  if (spec->is_complex) return LTB_EUNSUPPORTED;  // complex transform domains: the generic path
  if (ws_bytes < ltb_l_product_ws_bytes(spec, I1, L, I2, dtype))
    return ltb_set_error(ctx, LTB_EPARAM, "l_product: workspace too small");
  const int64_t P = spec->P;
  if (I1 == 0 || I2 == 0 || P == 0) return LTB_OK;
  if ((fused & 1) && dtype == LTB_F32) {
    const int st = ltb_lprod_fused_f32(ctx, spec, I1, L, I2, (const float*)d_a, (const float*)d_b, (float*)d_c, d_ws,
                                       (fused & 2) != 0);
    if (st != LTB_EUNSUPPORTED) return st;
  }
  const size_t es = dtype == LTB_F32 ? 4 : 8;
  char* hA = (char*)d_ws;
  char* hB = hA + es * P * I1 * L;
  char* hC = hB + es * P * L * I2;
  if (I1 * L == L * I2)
    LTB_TRY(ltb_transform_pair_impl(ctx, spec, I1 * L, 0, dtype, LTB_TUBE_MAJOR, d_a, d_b, dtype, LTB_SLICE_MAJOR, hA,
                                    hB));
  else {
    LTB_TRY(ltb_transform_impl(ctx, spec, I1 * L, 0, dtype, LTB_TUBE_MAJOR, d_a, dtype, LTB_SLICE_MAJOR, hA, nullptr));
    LTB_TRY(ltb_transform_impl(ctx, spec, L * I2, 0, dtype, LTB_TUBE_MAJOR, d_b, dtype, LTB_SLICE_MAJOR, hB, nullptr));
  }
  LTB_TRY(ltb_gemm_impl(ctx, dtype, P, I1, I2, L, LTB_OP_N, hA, L, I1 * L, LTB_OP_N, hB, I2, L * I2, hC, I2, I1 * I2,
                        nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
  return ltb_transform_impl(ctx, spec, I1 * I2, 1, dtype, LTB_SLICE_MAJOR, hC, dtype, LTB_TUBE_MAJOR, d_c, nullptr);
}
