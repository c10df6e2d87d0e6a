// K1 / K1': the transform L and its inverse as mode products over tubes.
//
// Reference semantics: apply_l / apply_l_inv (pkg/src/ltensor/transforms.py:176-226)
// apply M_k along each transformed mode in ascending order (inverse: M_k^{-1}
// in reverse order).  In C-order every tube x[i1, i2, :, ..., :] is P
// contiguous elements and L acts on each tube independently
// (mode_n_product, core.py:110-122).
//
// B200 design: the shared-memory tube-tile engine of ltb_xform_tile.cuh — one
// CTA owns TT consecutive tubes, all mode products run out of shared memory,
// and the epilogue writes either tube-major (apply_l's layout) or slice-major
// (the transform-domain slice stack fed to the slice GEMM / SVD), i.e. the
// layout change of as_rep_stack (core.py:70-74) is fused into the store.  HBM
// traffic is one read and one write of the tensor.  Tiles that cannot fit in
// shared memory (P beyond ~6K complex doubles) fall back to one global pass
// per mode.
#include <algorithm>

#include "ltb_xform_tile.cuh"

__global__ void finalize_partials_kernel(const double* __restrict__ partials, int64_t nblocks, int nacc,
                                         unsigned maxmask, double* __restrict__ out) {
  // one warp per slot, fixed order
  const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (slot >= nacc) return;
  const bool mx = (maxmask >> slot) & 1;
  double v = mx ? -1.0e308 : 0.0;
  for (int64_t i = lane; i < nblocks; i += 32) {
    const double w = partials[i * nacc + slot];
    v = mx ? fmax(v, w) : v + w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = mx ? fmax(v, w) : v + w;
  }
  if (lane == 0) out[slot] = v;
}

namespace {

// ------------------------------------------------------------------ generic global kernels
template <typename Tin, typename Tm, typename Tout, typename Tc>
__global__ void mode_product_kernel(int64_t outer, int64_t nin, int64_t inner, int64_t nout, const Tin* __restrict__ x,
                                    const Tm* __restrict__ M, Tout* __restrict__ y) {
  const int64_t total = outer * nout * inner;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = idx % inner;
    const int64_t r = idx / inner;
    const int64_t i = r % nout;
    const int64_t o = r / nout;
    Tc acc = zero_v<Tc>();
    const Tin* xb = x + o * nin * inner + l;
    const Tm* mr = M + i * nin;
    for (int64_t j = 0; j < nin; ++j) fma_acc(acc, mr[j], cvt<Tc>(xb[j * inner]));
    y[idx] = cvt<Tout>(acc);
  }
}

template <typename Tin, typename Tout>
__global__ void convert_kernel(int64_t n, const Tin* __restrict__ x, Tout* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = cvt<Tout>(x[i]);
}

// out[c, r] = in[r, c] (rows x cols -> cols x rows), with conversion
template <typename Tin, typename Tout>
__global__ void transpose_convert_kernel(int64_t rows, int64_t cols, const Tin* __restrict__ in, Tout* __restrict__ out) {
  __shared__ Tout tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = cvt<Tout>(in[r * cols + c]);
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
  }
}

template <typename T>
__global__ void sumsq_im_partials_kernel(int64_t n, const T* __restrict__ x, double* __restrict__ partials) {
  double a = 0.0, b = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    a += (double)abs2_v(x[i]);
    const double im = (double)im_v(x[i]);
    b += im * im;
  }
  __shared__ double red[2][32];
  a = warp_sum(a);
  b = warp_sum(b);
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][wid] = a;
    red[1][wid] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x0 = 0.0, y0 = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      x0 += red[0][k];
      y0 += red[1][k];
    }
    partials[2 * blockIdx.x] = x0;
    partials[2 * blockIdx.x + 1] = y0;
  }
}

// fallback: one global pass per mode (P too large for a shared-memory tile)
template <typename Tc, typename Tm, typename Tin, typename Tout>
int run_global(ltb_ctx* ctx, const XformParams& p, const void* in, int layout_in, void* out, int layout_out,
               const Tm* mats, double* d_sumsq) {
  const int64_t E = p.NT * (int64_t)p.P;
  Tc *a = nullptr, *b = nullptr;
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(Tc) * std::max<int64_t>(E, 1), (void**)&a));
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(Tc) * std::max<int64_t>(E, 1), (void**)&b));
  const int blocks = grid_for(E, 256, ctx->num_sms * 16);
  if (layout_in == LTB_TUBE_MAJOR) {
    convert_kernel<Tin, Tc><<<blocks, 256, 0, ctx->stream>>>(E, (const Tin*)in, a);
  } else {  // (P x NT) -> (NT x P)
    dim3 g((unsigned)((p.NT + 31) / 32), (unsigned)((p.P + 31) / 32));
    transpose_convert_kernel<Tin, Tc><<<g, dim3(32, 8), 0, ctx->stream>>>(p.P, p.NT, (const Tin*)in, a);
  }
  LTB_LAUNCH_CHECK(ctx);
  for (int s = 0; s < p.nsteps; ++s) {
    const ModeStep& st = p.step[s];
    mode_product_kernel<Tc, Tm, Tc, Tc><<<blocks, 256, 0, ctx->stream>>>(p.NT * st.hi, st.n, st.lo, st.n, a,
                                                                         mats + st.mat_off, b);
    LTB_LAUNCH_CHECK(ctx);
    std::swap(a, b);
  }
  constexpr bool residual = scalar_traits<Tc>::is_complex && !scalar_traits<Tout>::is_complex;
  if (d_sumsq) {
    if (residual) {
      const int nb = grid_for(E, 256, 1024);
      double* partials = nullptr;
      LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * 2 * nb, (void**)&partials));
      sumsq_im_partials_kernel<Tc><<<nb, 256, 0, ctx->stream>>>(E, a, partials);
      LTB_LAUNCH_CHECK(ctx);
      finalize_partials_kernel<<<1, 64, 0, ctx->stream>>>(partials, nb, 2, 0u, d_sumsq);
      LTB_LAUNCH_CHECK(ctx);
      ltb_ws_free(ctx, partials);
    } else {
      LTB_CUDA_TRY(ctx, cudaMemsetAsync(d_sumsq, 0, 2 * sizeof(double), ctx->stream));
    }
  }
  if (layout_out == LTB_TUBE_MAJOR) {
    convert_kernel<Tc, Tout><<<blocks, 256, 0, ctx->stream>>>(E, a, (Tout*)out);
  } else {
    dim3 g((unsigned)((p.P + 31) / 32), (unsigned)((p.NT + 31) / 32));
    transpose_convert_kernel<Tc, Tout><<<g, dim3(32, 8), 0, ctx->stream>>>(p.NT, p.P, a, (Tout*)out);
  }
  LTB_LAUNCH_CHECK(ctx);
  ltb_ws_free(ctx, a);
  ltb_ws_free(ctx, b);
  return LTB_OK;
}

template <typename R, bool IC, bool OC, bool CM>
int run_transform(ltb_ctx* ctx, XformParams p, const void* in, int layout_in, void* out, int layout_out,
                  const void* mats_v, double* d_sumsq) {
  using Tc = pick<R, IC || CM>;
  using Tin = pick<R, IC>;
  using Tout = pick<R, OC>;
  using Tm = pick<R, CM>;
  constexpr bool residual = (IC || CM) && !OC;
  const Tm* mats = (const Tm*)mats_v;
  size_t smem = 0;
  const int TT = plan_tile<Tc, Tm>(p, &smem);
  if (!TT) return run_global<Tc, Tm, Tin, Tout>(ctx, p, in, layout_in, out, layout_out, mats, d_sumsq);
  const int64_t nblocks = (p.NT + TT - 1) / TT;
  double* partials = nullptr;
  if (residual && d_sumsq) LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * 2 * nblocks, (void**)&partials));
  LoadPlain<Tin> ld{(const Tin*)in, layout_in};
  StorePlain<Tout, residual> st{(Tout*)out, layout_out};
  int64_t grid = 0;
  LTB_TRY((launch_xform_tile<Tc, Tm>(ctx, p, ld, st, mats, partials, nullptr, smem, &grid)));
  if (d_sumsq) {
    if (partials) {
      finalize_partials_kernel<<<1, 64, 0, ctx->stream>>>(partials, grid, 2, 0u, d_sumsq);
      LTB_LAUNCH_CHECK(ctx);
      ltb_ws_free(ctx, partials);
    } else {
      LTB_CUDA_TRY(ctx, cudaMemsetAsync(d_sumsq, 0, 2 * sizeof(double), ctx->stream));
    }
  }
  return LTB_OK;
}

template <typename R, bool IC, bool OC>
int dispatch_cm(ltb_ctx* ctx, bool cm, XformParams p, const void* in, int li, void* out, int lo, const void* mats,
                double* d) {
  if (cm) return run_transform<R, IC, OC, true>(ctx, p, in, li, out, lo, mats, d);
  return run_transform<R, IC, OC, false>(ctx, p, in, li, out, lo, mats, d);
}

template <typename R>
int dispatch_io(ltb_ctx* ctx, bool ic, bool oc, bool cm, XformParams p, const void* in, int li, void* out, int lo,
                const void* mats, double* d) {
  if (ic && oc) return dispatch_cm<R, true, true>(ctx, cm, p, in, li, out, lo, mats, d);
  if (ic && !oc) return dispatch_cm<R, true, false>(ctx, cm, p, in, li, out, lo, mats, d);
  if (!ic && oc) return dispatch_cm<R, false, true>(ctx, cm, p, in, li, out, lo, mats, d);
  return dispatch_cm<R, false, false>(ctx, cm, p, in, li, out, lo, mats, d);
}

}  // namespace

// 0: force the CUDA-core tile engine for fp32 real specs (A/B measurements)
constexpr int g_xform_tc = 1;

int ltb_transform_impl(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse, int dtype_in, int layout_in,
                       const void* d_in, int dtype_out, int layout_out, void* d_out, double* d_sumsq) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  if (!dtype_valid(dtype_in) || !dtype_valid(dtype_out))
    return ltb_set_error(ctx, LTB_EPARAM, "transform: bad dtype");
  if (dtype_is_double(dtype_in) != dtype_is_double(dtype_out))
    return ltb_set_error(ctx, LTB_EPARAM, "transform: input and output precision differ");
  if (ntubes < 0) return ltb_set_error(ctx, LTB_ESHAPE, "transform: negative tube count");
  if (spec->P > 0x7fffffff / 64) return ltb_set_error(ctx, LTB_ESHAPE, "transform: tube too long");
  XformParams p{};
  build_steps(spec, inverse, p);
  p.NT = ntubes;
  const bool ic = dtype_is_complex(dtype_in), oc = dtype_is_complex(dtype_out), cm = spec->is_complex != 0;
  const bool dbl = dtype_is_double(dtype_in);
  const void* mats = spec->d_mats[dbl ? 1 : 0][inverse ? 1 : 0];
  if (ntubes == 0) {
    if (d_sumsq) LTB_CUDA_TRY(ctx, cudaMemsetAsync(d_sumsq, 0, 2 * sizeof(double), ctx->stream));
    return LTB_OK;
  }
  // fp32 real specs: the transform as one dense Kronecker GEMM on the tensor
  // cores (tcgen05 kind::tf32, 3xTF32 split), with the tube<->slice layout
  // change folded into the operand / output orientation
  if (g_xform_tc && !dbl && !ic && !oc && !cm && spec->d_kron[0] && spec->nmodes > 0 &&
      !(layout_in == LTB_SLICE_MAJOR && layout_out == LTB_SLICE_MAJOR)) {
    const int64_t P = spec->P, NT = ntubes;
    const float* K = spec->d_kron[inverse ? 1 : 0];
    const float* Klo = K + P * P;  // precomputed 3xTF32 lo part (ltb_ctx.cu)
    const float* X = (const float*)d_in;
    float* Y = (float*)d_out;
    int st;
    // every orientation is D(NT x P) = X(NT x P) * K^T with tubes on the 128-row MMA side
    // and K (constant, pre-split) resident in shared memory when P <= 96
    if (layout_in == LTB_TUBE_MAJOR && layout_out == LTB_SLICE_MAJOR)  // Y(P x NT) = D^T
      st = ltb_tc_gemm_f32(ctx, 1, NT, P, P, false, X, P, 0, false, K, P, 0, Y, NT, 0, 3, true, Klo);
    else if (layout_in == LTB_SLICE_MAJOR)  // X stored P x NT (MN-major A), Y(NT x P) = D
      st = ltb_tc_gemm_f32(ctx, 1, NT, P, P, true, X, NT, 0, false, K, P, 0, Y, P, 0, 3, false, Klo);
    else  // tube -> tube: Y(NT x P) = D
      st = ltb_tc_gemm_f32(ctx, 1, NT, P, P, false, X, P, 0, false, K, P, 0, Y, P, 0, 3, false, Klo);
    if (st != LTB_EUNSUPPORTED) {
      if (st == LTB_OK && d_sumsq) LTB_CUDA_TRY(ctx, cudaMemsetAsync(d_sumsq, 0, 2 * sizeof(double), ctx->stream));
      return st;
    }
  }
  if (dbl) return dispatch_io<double>(ctx, ic, oc, cm, p, d_in, layout_in, d_out, layout_out, mats, d_sumsq);
  return dispatch_io<float>(ctx, ic, oc, cm, p, d_in, layout_in, d_out, layout_out, mats, d_sumsq);
}

// K1 of two tensors with equal tube counts: one batched tensor-core launch when
// the pair can be addressed as a batch of two (same sign of the input and
// output pointer offsets, 16-byte multiples); otherwise two launches.
int ltb_transform_pair_impl(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse, int dtype_in,
                            int layout_in, const void* d_in0, const void* d_in1, int dtype_out, int layout_out,
                            void* d_out0, void* d_out1) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  const bool real32 = dtype_in == LTB_F32 && dtype_out == LTB_F32 && !spec->is_complex;
  if (g_xform_tc && real32 && spec->d_kron[0] && spec->nmodes > 0 && ntubes > 0 && spec->P <= 96 &&
      layout_in == LTB_TUBE_MAJOR && layout_out == LTB_SLICE_MAJOR) {
    int64_t din = (const char*)d_in1 - (const char*)d_in0;
    int64_t dout = (const char*)d_out1 - (const char*)d_out0;
    const float* X = (const float*)d_in0;
    float* Y = (float*)d_out0;
    if (din < 0 && dout < 0) {  // address the pair from the lower pointers
      din = -din;
      dout = -dout;
      X = (const float*)d_in1;
      Y = (float*)d_out1;
    }
    const int64_t P = spec->P, NT = ntubes;
    if (din > 0 && dout > 0 && din % 16 == 0 && dout % 16 == 0 && din < (int64_t(1) << 40) &&
        dout < (int64_t(1) << 40) && din / 4 >= NT * P && dout / 4 >= NT * P) {
      const float* K = spec->d_kron[inverse ? 1 : 0];
      const int st =
          ltb_tc_gemm_f32(ctx, 2, NT, P, P, false, X, P, din / 4, false, K, P, 0, Y, NT, dout / 4, 3, true, K + P * P);
      if (st != LTB_EUNSUPPORTED) return st;
    }
  }
  LTB_TRY(ltb_transform_impl(ctx, spec, ntubes, inverse, dtype_in, layout_in, d_in0, dtype_out, layout_out, d_out0,
                             nullptr));
  return ltb_transform_impl(ctx, spec, ntubes, inverse, dtype_in, layout_in, d_in1, dtype_out, layout_out, d_out1,
                            nullptr);
}

extern "C" int ltb_mode_product(ltb_ctx* ctx, int64_t outer, int64_t nin, int64_t inner, int64_t nout, int dtype_in,
                                const void* d_in, int dtype_mat, const void* d_mat, int dtype_out, void* d_out) {
  if (!dtype_valid(dtype_in) || !dtype_valid(dtype_mat) || !dtype_valid(dtype_out))
    return ltb_set_error(ctx, LTB_EPARAM, "mode_product: bad dtype");
  if (outer < 0 || nin < 0 || inner < 0 || nout < 0) return ltb_set_error(ctx, LTB_ESHAPE, "mode_product: bad shape");
  const int64_t total = outer * nout * inner;
  if (total == 0) return LTB_OK;
  const bool dbl = dtype_is_double(dtype_out);
  if (dtype_is_double(dtype_in) != dbl || dtype_is_double(dtype_mat) != dbl)
    return ltb_set_error(ctx, LTB_EPARAM, "mode_product: mixed precision");
  if (dtype_in == dtype_mat && dtype_in == dtype_out && nin > 0) {
    // y[o, :, l] = M x[o, :, l] is a GEMM (core.py:110-122 unfolds to the same product):
    //   inner == 1  one GEMM  Y (outer x nout) = X (outer x nin) M^T
    //   otherwise   outer GEMMs Y_o (nout x inner) = M (nout x nin) X_o (nin x inner), M shared
    // through the shared-memory tiled / tcgen05 engine of ltb_gemm.cu (batches of <= 65535)
    const size_t es = dtype_size(dtype_in);
    if (inner == 1)
      return ltb_gemm_impl(ctx, dtype_in, 1, outer, nout, nin, LTB_OP_N, d_in, nin, 0, LTB_OP_T, d_mat, nin, 0, d_out,
                           nout, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    if (inner >= 16) {
      for (int64_t o0 = 0; o0 < outer; o0 += 65535) {
        const int64_t nb = std::min<int64_t>(65535, outer - o0);
        LTB_TRY(ltb_gemm_impl(ctx, dtype_in, nb, nout, inner, nin, LTB_OP_N, d_mat, nin, 0, LTB_OP_N,
                              (const char*)d_in + es * o0 * nin * inner, inner, nin * inner,
                              (char*)d_out + es * o0 * nout * inner, inner, nout * inner, nullptr, nullptr, nullptr,
                              nullptr, nullptr, nullptr));
      }
      return LTB_OK;
    }
  }
  // short inner runs (2..15) or mixed real / complex operands: one output per thread
  const int blocks = grid_for(total, 256, ctx->num_sms * 16);
  return dispatch_dtype(dtype_in, [&](auto ti) {
    using Tin = typename decltype(ti)::type;
    return dispatch_dtype(dtype_mat, [&](auto tm) {
      using Tm = typename decltype(tm)::type;
      return dispatch_dtype(dtype_out, [&](auto to) {
        using Tout = typename decltype(to)::type;
        using R = typename scalar_traits<Tout>::real;
        constexpr bool cc = scalar_traits<Tin>::is_complex || scalar_traits<Tm>::is_complex;
        using Tc = pick<R, cc>;
        if constexpr (!std::is_same<typename scalar_traits<Tin>::real, R>::value ||
                      !std::is_same<typename scalar_traits<Tm>::real, R>::value) {
          return ltb_set_error(ctx, LTB_EPARAM, "mode_product: mixed precision");
        } else {
          mode_product_kernel<Tin, Tm, Tout, Tc><<<blocks, 256, 0, ctx->stream>>>(
              outer, nin, inner, nout, (const Tin*)d_in, (const Tm*)d_mat, (Tout*)d_out);
          LTB_LAUNCH_CHECK(ctx);
          return (int)LTB_OK;
        }
      });
    });
  });
}

extern "C" int ltb_convert(ltb_ctx* ctx, int64_t n, int dtype_in, const void* d_in, int dtype_out, void* d_out) {
  if (!dtype_valid(dtype_in) || !dtype_valid(dtype_out)) return ltb_set_error(ctx, LTB_EPARAM, "convert: bad dtype");
  if (n <= 0) return LTB_OK;
  const int blocks = grid_for(n, 256, ctx->num_sms * 16);
  return dispatch_dtype(dtype_in, [&](auto ti) {
    using Tin = typename decltype(ti)::type;
    return dispatch_dtype(dtype_out, [&](auto to) {
      using Tout = typename decltype(to)::type;
      convert_kernel<Tin, Tout><<<blocks, 256, 0, ctx->stream>>>(n, (const Tin*)d_in, (Tout*)d_out);
      LTB_LAUNCH_CHECK(ctx);
      return (int)LTB_OK;
    });
  });
}
