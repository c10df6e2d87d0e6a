// Small slice-stack helpers used by the *_L algebra wrappers:
//   ltb_embed_diag       _embed_diag (linalg.py:93-99) and identity_tensor's eye stack (linalg.py:46-51)
//   ltb_slice_transpose  l_transpose's conj(swapaxes(hat, 1, 2)) (linalg.py:54-59)
//   ltb_project_omega    project_omega (completion.py:23-29)
//   ltb_reduce_dot       inner_product's vdot (core.py:26-35)
#include <algorithm>

#include "ltb_dispatch.cuh"

namespace {

template <typename T, typename R>
__global__ void embed_diag_kernel(int64_t batch, int64_t m, int64_t n, int64_t k, const R* __restrict__ vals,
                                  T* __restrict__ out) {
  const int64_t total = batch * m * n;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = l / (m * n);
    const int64_t r = l - b * m * n;
    const int64_t i = r / n, j = r - (r / n) * n;
    out[l] = (i == j && i < k) ? cvt<T>(vals[b * k + i]) : zero_v<T>();
  }
}

template <typename T>
__global__ void slice_transpose_kernel(int64_t m, int64_t n, int conj, const T* __restrict__ in, T* __restrict__ out) {
  __shared__ T tile[32][33];
  const int64_t b = blockIdx.z;
  const T* src = in + b * m * n;
  T* dst = out + b * m * n;
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < m && c < n) {
      T v = src[r * n + c];
      tile[k][threadIdx.x] = conj ? conj_v(v) : v;
    }
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < m && c < n) dst[c * m + r] = tile[threadIdx.x][k];
  }
}

template <typename T>
__global__ void project_omega_kernel(int64_t n, const T* __restrict__ x, const uint8_t* __restrict__ mask,
                                     T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mask[i] ? x[i] : zero_v<T>();
}

template <typename T>
__global__ void dot_partials_kernel(int64_t n, const T* __restrict__ x, const T* __restrict__ y,
                                    double* __restrict__ part) {
  double a = 0.0, c = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T v = conj_v(x[i]) * y[i];
    a += (double)re_v(v);
    c += (double)im_v(v);
  }
  __shared__ double ra[32], rc[32];
  a = warp_sum(a);
  c = warp_sum(c);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    ra[wid] = a;
    rc[wid] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      s += ra[k];
      t += rc[k];
    }
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = t;
  }
}

// PGA gradient point (completion.py:170-171) on a row shard, same rounding as the fused path:
// y = x + beta (x - x_prev), g = y - (where(mask, y, 0) - p_obs)
template <typename R>
__global__ void pga_gradient_kernel(int64_t n, const R* __restrict__ xc, const R* __restrict__ xp,
                                    const R* __restrict__ pobs, const uint8_t* __restrict__ mask, R beta,
                                    R* __restrict__ y, R* __restrict__ g) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    R yi;
    if constexpr (std::is_same<R, double>::value) {
      yi = __dadd_rn(xc[i], __dmul_rn(beta, __dsub_rn(xc[i], xp[i])));
      g[i] = __dsub_rn(yi, __dsub_rn(mask[i] ? yi : 0.0, pobs[i]));
    } else {
      yi = __fadd_rn(xc[i], __fmul_rn(beta, __fsub_rn(xc[i], xp[i])));
      g[i] = __fsub_rn(yi, __fsub_rn(mask[i] ? yi : 0.f, pobs[i]));
    }
    if (y) y[i] = yi;
  }
}

}  // namespace

__global__ void finalize_partials_kernel(const double* __restrict__ partials, int64_t nblocks, int nacc,
                                         unsigned maxmask, double* __restrict__ out);

// TLT1 payloads are generalized column-major (io.py:1-10): the device copy is
// reordered to C order, dst[c-index(i)] = src[f-index(i)], for element sizes
// 1, 4, 8, 16 bytes.  Each thread owns one destination element (coalesced
// writes; the source gather is strided).
struct FDims {
  int nd;
  int64_t d[8];
};

template <typename E>
__global__ void fortran_to_c_kernel(int64_t total, FDims g, const E* __restrict__ src, E* __restrict__ dst) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = l, f = 0, stride = 1;
    int64_t idx[8];
    for (int a = g.nd - 1; a >= 0; --a) {  // C-order decode
      idx[a] = r % g.d[a];
      r /= g.d[a];
    }
    for (int a = 0; a < g.nd; ++a) {  // Fortran-order encode
      f += idx[a] * stride;
      stride *= g.d[a];
    }
    dst[l] = src[f];
  }
}

extern "C" {

int ltb_fortran_to_c(ltb_ctx* ctx, int ndim, const int64_t* dims, int elem_bytes, const void* d_src, void* d_dst) {
  if (ndim < 1 || ndim > 8) return ltb_set_error(ctx, LTB_ESHAPE, "fortran_to_c: order %d outside 1..8", ndim);
  FDims g{};
  g.nd = ndim;
  int64_t total = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 0) return ltb_set_error(ctx, LTB_ESHAPE, "fortran_to_c: negative dim");
    g.d[a] = dims[a];
    total *= dims[a];
  }
  if (total == 0) return LTB_OK;
  const unsigned grid = grid_for(total, 256, ctx->num_sms * 16);
  switch (elem_bytes) {
    case 1:
      fortran_to_c_kernel<uint8_t><<<grid, 256, 0, ctx->stream>>>(total, g, (const uint8_t*)d_src, (uint8_t*)d_dst);
      break;
    case 4:
      fortran_to_c_kernel<float><<<grid, 256, 0, ctx->stream>>>(total, g, (const float*)d_src, (float*)d_dst);
      break;
    case 8:
      fortran_to_c_kernel<double><<<grid, 256, 0, ctx->stream>>>(total, g, (const double*)d_src, (double*)d_dst);
      break;
    case 16:
      fortran_to_c_kernel<double2><<<grid, 256, 0, ctx->stream>>>(total, g, (const double2*)d_src, (double2*)d_dst);
      break;
    default:
      return ltb_set_error(ctx, LTB_EPARAM, "fortran_to_c: element size %d not in {1, 4, 8, 16}", elem_bytes);
  }
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

int ltb_embed_diag(ltb_ctx* ctx, int dtype_out, int64_t batch, int64_t m, int64_t n, const void* d_vals,
                   void* d_out) {
  if (!dtype_valid(dtype_out)) return ltb_set_error(ctx, LTB_EPARAM, "embed_diag: bad dtype");
  const int64_t total = batch * m * n;
  if (total <= 0) return LTB_OK;
  const int64_t k = std::min(m, n);
  return dispatch_dtype(dtype_out, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    using R = typename scalar_traits<T>::real;
    embed_diag_kernel<T, R><<<grid_for(total, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(batch, m, n, k,
                                                                                            (const R*)d_vals, (T*)d_out);
    LTB_LAUNCH_CHECK(ctx);
    return LTB_OK;
  });
}

int ltb_slice_transpose(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, int conj, const void* d_in,
                        void* d_out) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "slice_transpose: bad dtype");
  if (batch <= 0 || m <= 0 || n <= 0) return LTB_OK;
  if (batch > 65535) return ltb_set_error(ctx, LTB_ESHAPE, "slice_transpose: batch too large");
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    dim3 g((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32), (unsigned)batch);
    slice_transpose_kernel<T><<<g, dim3(32, 8), 0, ctx->stream>>>(m, n, conj, (const T*)d_in, (T*)d_out);
    LTB_LAUNCH_CHECK(ctx);
    return LTB_OK;
  });
}

int ltb_project_omega(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const uint8_t* d_mask, void* d_out) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "project_omega: bad dtype");
  if (n <= 0) return LTB_OK;
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    project_omega_kernel<T><<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(n, (const T*)d_x, d_mask,
                                                                                        (T*)d_out);
    LTB_LAUNCH_CHECK(ctx);
    return LTB_OK;
  });
}

int ltb_pga_gradient(ltb_ctx* ctx, int dtype, int64_t n, const void* d_xc, const void* d_xp, const void* d_pobs,
                     const uint8_t* d_mask, double beta, void* d_y, void* d_g) {
  if (dtype != LTB_F32 && dtype != LTB_F64) return ltb_set_error(ctx, LTB_EPARAM, "pga_gradient: real dtype only");
  if (n <= 0) return LTB_OK;
  const int blocks = grid_for(n, 256, ctx->num_sms * 8);
  if (dtype == LTB_F64)
    pga_gradient_kernel<double><<<blocks, 256, 0, ctx->stream>>>(n, (const double*)d_xc, (const double*)d_xp,
                                                                 (const double*)d_pobs, d_mask, beta, (double*)d_y,
                                                                 (double*)d_g);
  else
    pga_gradient_kernel<float><<<blocks, 256, 0, ctx->stream>>>(n, (const float*)d_xc, (const float*)d_xp,
                                                                (const float*)d_pobs, d_mask, (float)beta,
                                                                (float*)d_y, (float*)d_g);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

int ltb_reduce_dot(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y, double* h_out) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "reduce_dot: bad dtype");
  const int nb = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (n + 255) / 256));
  double* part = nullptr;
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * 2 * nb, (void**)&part));
  int st = dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    dot_partials_kernel<T><<<nb, 256, 0, ctx->stream>>>(n, (const T*)d_x, (const T*)d_y, part);
    LTB_LAUNCH_CHECK(ctx);
    finalize_partials_kernel<<<1, 64, 0, ctx->stream>>>(part, nb, 2, 0u, ctx->d_scratch);
    LTB_LAUNCH_CHECK(ctx);
    return LTB_OK;
  });
  ltb_ws_free(ctx, part);
  if (st != LTB_OK) return st;
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scratch, ctx->d_scratch, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  h_out[0] = ctx->h_scratch[0];
  h_out[1] = ctx->h_scratch[1];
  return LTB_OK;
}

}  // extern "C"
