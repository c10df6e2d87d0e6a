// Deterministic reductions: sum |x - y|^2 and max Re(x) (fro_norm core.py:38-40,
// rse / psnr completion.py:45-78).  Two fixed-order stages in float64.
#include <cfloat>

#include "ltb_dispatch.cuh"

namespace {

constexpr int kRedThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kRedThreads) sumsq_max_partials(int64_t n, const T* __restrict__ x,
                                                                  const T* __restrict__ y, double* __restrict__ part) {
  double s = 0.0, mx = -DBL_MAX;
  for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedThreads) {
    T v = x[i];
    mx = fmax(mx, (double)re_v(v));
    if (y) v = v - y[i];
    s += (double)abs2_v(v);
  }
  __shared__ double rs[kRedThreads / 32], rm[kRedThreads / 32];
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    rs[wid] = s;
    rm[wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = -DBL_MAX;
    for (int k = 0; k < kRedThreads / 32; ++k) {
      a += rs[k];
      b = fmax(b, rm[k]);
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void sumsq_max_finalize(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double rs[32], rm[32];
  double s = 0.0, mx = -DBL_MAX;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    s += part[2 * i];
    mx = fmax(mx, part[2 * i + 1]);
  }
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    rs[wid] = s;
    rm[wid] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = -DBL_MAX;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      a += rs[k];
      b = fmax(b, rm[k]);
    }
    out[0] = a;
    out[1] = b;
  }
}

}  // namespace

int ltb_reduce_sumsq_dev(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y, double* d_out) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "reduce: bad dtype");
  // a fixed block count keeps the summation order independent of the device
  const int nb = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (n + kRedThreads - 1) / kRedThreads));
  double* part = nullptr;
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * 2 * nb, (void**)&part));
  int st = dispatch_dtype(dtype, [&](auto tg) {
    using T = typename decltype(tg)::type;
    sumsq_max_partials<T><<<nb, kRedThreads, 0, ctx->stream>>>(n, (const T*)d_x, (const T*)d_y, part);
    LTB_LAUNCH_CHECK(ctx);
    sumsq_max_finalize<<<1, 256, 0, ctx->stream>>>(part, nb, d_out);
    LTB_LAUNCH_CHECK(ctx);
    return (int)LTB_OK;
  });
  ltb_ws_free(ctx, part);
  return st;
}
