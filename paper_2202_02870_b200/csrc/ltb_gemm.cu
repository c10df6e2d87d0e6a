// K2: batched transform-domain GEMM (facewise_product core.py:125-134,
// l_product linalg.py:42) and the SVT recomposition GEMMs (linalg.py:180).
//
// C[b] = op_a(A[b]) * op_b(B[b]) (* optional per-row / per-column real scale),
// with optional per-batch limits on m / n / k read from device memory (the
// SVT recomposition only multiplies the singular directions that survive
// the threshold; the kept count differs per slice and is known only on the
// device).  Shared-memory tiled CUDA-core kernel, register-blocked; fp32,
// fp64, complex64, complex128.
#include "ltb_dispatch.cuh"

namespace {

template <typename T>
__device__ __forceinline__ T load_op(const T* __restrict__ base, int op, int64_t ld, int64_t r, int64_t c) {
  // element (r, c) of op(X)
  T v = (op == LTB_OP_N || op == LTB_OP_C) ? base[r * ld + c] : base[c * ld + r];
  if (op == LTB_OP_C || op == LTB_OP_H) v = conj_v(v);
  return v;
}

template <typename T, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    gemm_kernel(int64_t M, int64_t N, int64_t K, int op_a, const T* __restrict__ A, int64_t lda, int64_t sa, int op_b,
                const T* __restrict__ B, int64_t ldb, int64_t sb, T* __restrict__ C, int64_t ldc, int64_t sc,
                const int* __restrict__ mlim, const int* __restrict__ nlim, const int* __restrict__ klim,
                const typename scalar_traits<T>::real* __restrict__ row_scale,
                const typename scalar_traits<T>::real* __restrict__ col_scale, const int* __restrict__ skip) {
  if (skip && *skip) return;
  constexpr int DX = BN / TN, DY = BM / TM, NTH = DX * DY;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int64_t b = blockIdx.z;
  const int64_t Mb = mlim ? min(M, (int64_t)mlim[b]) : M;
  const int64_t Nb = nlim ? min(N, (int64_t)nlim[b]) : N;
  const int64_t Kb = klim ? min(K, (int64_t)klim[b]) : K;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  if (m0 >= Mb || n0 >= Nb) return;
  A += b * sa;
  B += b * sb;
  C += b * sc;
  const int tid = threadIdx.x;
  const int tx = tid % DX, ty = tid / DX;
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = zero_v<T>();

  const bool a_rowmajor = (op_a == LTB_OP_N || op_a == LTB_OP_C);
  const bool b_rowmajor = (op_b == LTB_OP_N || op_b == LTB_OP_C);
  for (int64_t k0 = 0; k0 < Kb; k0 += BK) {
    for (int l = tid; l < BM * BK; l += NTH) {
      int i, kk;
      if (a_rowmajor) {  // contiguous along k
        i = l / BK;
        kk = l % BK;
      } else {
        kk = l / BM;
        i = l % BM;
      }
      const int64_t gi = m0 + i, gk = k0 + kk;
      As[kk][i] = (gi < Mb && gk < Kb) ? load_op(A, op_a, lda, gi, gk) : zero_v<T>();
    }
    for (int l = tid; l < BN * BK; l += NTH) {
      int j, kk;
      if (b_rowmajor) {  // contiguous along n
        kk = l / BN;
        j = l % BN;
      } else {
        j = l / BK;
        kk = l % BK;
      }
      const int64_t gj = n0 + j, gk = k0 + kk;
      Bs[kk][j] = (gj < Nb && gk < Kb) ? load_op(B, op_b, ldb, gk, gj) : zero_v<T>();
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty + i * DY];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx + j * DX];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) fma_acc(acc[i][j], a[i], bv[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t gi = m0 + ty + i * DY;
    if (gi >= Mb) continue;
    const auto rs = row_scale ? row_scale[b * M + gi] : (typename scalar_traits<T>::real)1;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t gj = n0 + tx + j * DX;
      if (gj >= Nb) continue;
      T v = acc[i][j];
      if (row_scale) v = v * rs;
      if (col_scale) v = v * col_scale[b * N + gj];
      C[gi * ldc + gj] = v;
    }
  }
}

template <typename T, int BM, int BN, int BK, int TM, int TN>
int launch_gemm(ltb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t k, int op_a, const T* a, int64_t lda,
                int64_t sa, int op_b, const T* b, int64_t ldb, int64_t sb, T* c, int64_t ldc, int64_t sc,
                const int* mlim, const int* nlim, const int* klim, const void* rs, const void* cs,
                const int* skip) {
  using R = typename scalar_traits<T>::real;
  dim3 grid((unsigned)((n + BN - 1) / BN), (unsigned)((m + BM - 1) / BM), (unsigned)batch);
  if (grid.y > 65535 || grid.z > 65535) return ltb_set_error(ctx, LTB_ESHAPE, "gemm: grid too large");
  gemm_kernel<T, BM, BN, BK, TM, TN><<<grid, (BM / TM) * (BN / TN), 0, ctx->stream>>>(
      m, n, k, op_a, a, lda, sa, op_b, b, ldb, sb, c, ldc, sc, mlim, nlim, klim, (const R*)rs, (const R*)cs, skip);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

// zero-fill C when k == 0 (numpy returns zeros for an empty inner dimension)
template <typename T>
__global__ void zero_c_kernel(int64_t batch, int64_t m, int64_t n, T* c, int64_t ldc, int64_t sc) {
  const int64_t total = batch * m * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i % n, r = (i / n) % m, b = i / (m * n);
    c[b * sc + r * ldc + j] = zero_v<T>();
  }
}

// complex64 on the tensor cores: the real 2 x 2 representation of the right operand.
// With X (m x k complex, K contiguous) viewed as a real m x 2k matrix [re, im interleaved
// along K], X Y = X' Y~ where Y~ (2k x 2n real) holds, for every y = Y[l][j], the block
//   rows 2l, 2l+1 / columns 2j, 2j+1:  [ re  im ; -im  re ]      (row 2l meets Re x, row 2l+1 Im x)
// and conj(X) Y uses [ re  im ; im  -re ].  The real product X' Y~ (m x 2n) is the complex
// result in its usual interleaved layout, so one fp32 tensor-core GEMM (3xTF32) with the
// same 8 m n k real multiply-adds as the 4M scheme computes it.  `in` is stored rows x cols
// complex (ld elements): kn == true, rows = k and cols = n (the block is written as above, the
// result is the MN-major B operand); kn == false, rows = n and cols = k (the block is written
// transposed: the K-major B operand).
__global__ void cexpand_kernel(int rows, int cols, int64_t ld, int64_t sin, const cplx<float>* __restrict__ in,
                               float* __restrict__ out, int kn, int conj_in, int conj_left,
                               const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t b = blockIdx.z;
  const int r = blockIdx.y;
  const cplx<float>* src = in + b * sin + (int64_t)r * ld;
  float2* o0 = reinterpret_cast<float2*>(out + (b * 4 * rows + (int64_t)(2 * r) * 2) * cols);
  float2* o1 = o0 + cols;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(src + c));
    const float re = v.x, im = conj_in ? -v.y : v.y;
    // E = [e00 e01; e10 e11]
    const float e00 = re, e01 = im, e10 = conj_left ? im : -im, e11 = conj_left ? -re : re;
    if (kn) {
      o0[c] = make_float2(e00, e01);
      o1[c] = make_float2(e10, e11);
    } else {
      o0[c] = make_float2(e00, e10);
      o1[c] = make_float2(e01, e11);
    }
  }
}

}  // namespace

// C = op(A) op(B) for complex64 on the tcgen05 engine through the real representation above.
// A: m x k, K contiguous (conj_a: conj(A)); B: stored k x n (b_kn) or n x k, conj_b conjugates
// its elements.  rscale: optional real scale per row of C (batch x m).  LTB_EUNSUPPORTED when
// the shape / alignment does not fit (the caller falls back to the CUDA-core kernel).
int ltb_cgemm_tc(ltb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t k, bool conj_a, const void* d_a,
                 int64_t lda, int64_t sa, bool b_kn, bool conj_b, const void* d_b, int64_t ldb, int64_t sb,
                 void* d_c, int64_t ldc, int64_t sc, const float* rscale, const int* skip) {
  if (batch < 1 || batch > 65535 || m < 32 || n < 16 || k < 4) return LTB_EUNSUPPORTED;
  const int64_t rows = b_kn ? k : n, cols = b_kn ? n : k;
  if (rows > 65535 || cols > (1 << 28)) return LTB_EUNSUPPORTED;
  const int64_t nb = (sb == 0) ? 1 : batch;  // a B shared by the batch is expanded once
  WsScope ws(ctx);
  float* be = nullptr;
  LTB_TRY(ws.alloc(sizeof(float) * (size_t)nb * 4 * rows * cols, &be));
  {
    const dim3 grid((unsigned)std::min<int64_t>((cols + 255) / 256, 64), (unsigned)rows, (unsigned)nb);
    cexpand_kernel<<<grid, 256, 0, ctx->stream>>>((int)rows, (int)cols, ldb, sb, (const cplx<float>*)d_b, be,
                                                  b_kn ? 1 : 0, conj_b ? 1 : 0, conj_a ? 1 : 0, skip);
    LTB_LAUNCH_CHECK(ctx);
  }
  return ltb_tc_gemm_f32(ctx, batch, m, 2 * n, 2 * k, false, (const float*)d_a, 2 * lda, 2 * sa, b_kn, be, 2 * cols,
                         sb == 0 ? 0 : 4 * rows * cols, (float*)d_c, 2 * ldc, 2 * sc, 3, false, nullptr, nullptr,
                         rscale, nullptr, skip);
}

int ltb_gemm_impl(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, int64_t k, int op_a, const void* d_a,
                  int64_t lda, int64_t sa, int op_b, const void* d_b, int64_t ldb, int64_t sb, void* d_c, int64_t ldc,
                  int64_t sc, const int* d_mlim, const int* d_nlim, const int* d_klim, const void* d_row_scale,
                  const void* d_col_scale, const int* d_skip) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "gemm: bad dtype");
  if (batch < 0 || m < 0 || n < 0 || k < 0) return ltb_set_error(ctx, LTB_ESHAPE, "gemm: negative dimension");
  if (op_a < 0 || op_a > 3 || op_b < 0 || op_b > 3) return ltb_set_error(ctx, LTB_EPARAM, "gemm: bad op");
  if (batch == 0 || m == 0 || n == 0) return LTB_OK;
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    const T* a = (const T*)d_a;
    const T* b = (const T*)d_b;
    T* c = (T*)d_c;
    if (k == 0) {
      zero_c_kernel<T><<<grid_for(batch * m * n, 256, 4096), 256, 0, ctx->stream>>>(batch, m, n, c, ldc, sc);
      LTB_LAUNCH_CHECK(ctx);
      return LTB_OK;
    }
    // fp32 without m / n limits: tcgen05 kind::tf32 with the 3xTF32 split (per-slice K
    // limits, row / column scaling and the skip flag are handled by the tensor-core kernel)
    if constexpr (std::is_same<T, float>::value) {
      if (!d_mlim && !d_nlim && m >= 32 && n >= 32 && k >= 8) {
        // op N: A stored m x k (K-major); op T: stored k x m (MN-major).  B: op N stored k x n (MN-major).
        const bool a_mn = (op_a == LTB_OP_T || op_a == LTB_OP_H);
        const bool b_mn = (op_b == LTB_OP_N || op_b == LTB_OP_C);
        const int st = ltb_tc_gemm_f32(ctx, batch, m, n, k, a_mn, a, lda, sa, b_mn, b, ldb, sb, c, ldc, sc, 3,
                                       false, nullptr, d_klim, (const float*)d_row_scale,
                                       (const float*)d_col_scale, d_skip);
        if (st != LTB_EUNSUPPORTED) return st;
      }
    }
    // complex64 without limits / column scaling and with A's K contiguous: one 3xTF32
    // tensor-core GEMM on the real 2 x 2 representation of B (ltb_cgemm_tc)
    if constexpr (std::is_same<T, cplx<float>>::value) {
      if (!d_mlim && !d_nlim && !d_klim && !d_col_scale && (op_a == LTB_OP_N || op_a == LTB_OP_C) && m >= 64 &&
          n >= 32 && k >= 16) {
        const bool b_kn = (op_b == LTB_OP_N || op_b == LTB_OP_C);
        const bool conj_b = (op_b == LTB_OP_C || op_b == LTB_OP_H);
        const int st = ltb_cgemm_tc(ctx, batch, m, n, k, op_a == LTB_OP_C, a, lda, sa, b_kn, conj_b, b, ldb, sb, c,
                                    ldc, sc, (const float*)d_row_scale, d_skip);
        if (st != LTB_EUNSUPPORTED) return st;
      }
    }
    const bool small = (m <= 32 && n <= 32);
    if constexpr (std::is_same<T, float>::value) {
      if (!small)
        return launch_gemm<T, 128, 128, 8, 8, 8>(ctx, batch, m, n, k, op_a, a, lda, sa, op_b, b, ldb, sb, c, ldc, sc,
                                                 d_mlim, d_nlim, d_klim, d_row_scale, d_col_scale, d_skip);
    } else if constexpr (!std::is_same<T, cplx<double>>::value) {
      if (!small)
        return launch_gemm<T, 64, 64, 8, 4, 4>(ctx, batch, m, n, k, op_a, a, lda, sa, op_b, b, ldb, sb, c, ldc, sc,
                                               d_mlim, d_nlim, d_klim, d_row_scale, d_col_scale, d_skip);
    }
    return launch_gemm<T, 32, 32, 8, 2, 2>(ctx, batch, m, n, k, op_a, a, lda, sa, op_b, b, ldb, sb, c, ldc, sc,
                                           d_mlim, d_nlim, d_klim, d_row_scale, d_col_scale, d_skip);
  });
}
