// Shared device/host helpers for libltb (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/ltb.h"

// ------------------------------------------------------------------ complex
template <typename R>
struct cplx {
  R re, im;
};

template <typename T> struct scalar_traits {
  using real = T;
  static constexpr bool is_complex = false;
};
template <typename R> struct scalar_traits<cplx<R>> {
  using real = R;
  static constexpr bool is_complex = true;
};

template <typename R> __host__ __device__ __forceinline__ cplx<R> operator+(cplx<R> a, cplx<R> b) {
  return {a.re + b.re, a.im + b.im};
}
template <typename R> __host__ __device__ __forceinline__ cplx<R> operator-(cplx<R> a, cplx<R> b) {
  return {a.re - b.re, a.im - b.im};
}
template <typename R> __host__ __device__ __forceinline__ cplx<R> operator*(cplx<R> a, cplx<R> b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
template <typename R> __host__ __device__ __forceinline__ cplx<R> operator*(R a, cplx<R> b) {
  return {a * b.re, a * b.im};
}
template <typename R> __host__ __device__ __forceinline__ cplx<R> operator*(cplx<R> b, R a) {
  return {a * b.re, a * b.im};
}

// value helpers usable for both real and complex
template <typename T> __host__ __device__ __forceinline__ T zero_v() { return T(0); }
template <> __host__ __device__ __forceinline__ cplx<float> zero_v<cplx<float>>() { return {0.f, 0.f}; }
template <> __host__ __device__ __forceinline__ cplx<double> zero_v<cplx<double>>() { return {0.0, 0.0}; }

__host__ __device__ __forceinline__ float conj_v(float a) { return a; }
__host__ __device__ __forceinline__ double conj_v(double a) { return a; }
template <typename R> __host__ __device__ __forceinline__ cplx<R> conj_v(cplx<R> a) { return {a.re, -a.im}; }

__host__ __device__ __forceinline__ float abs2_v(float a) { return a * a; }
__host__ __device__ __forceinline__ double abs2_v(double a) { return a * a; }
template <typename R> __host__ __device__ __forceinline__ R abs2_v(cplx<R> a) { return a.re * a.re + a.im * a.im; }

__host__ __device__ __forceinline__ float re_v(float a) { return a; }
__host__ __device__ __forceinline__ double re_v(double a) { return a; }
template <typename R> __host__ __device__ __forceinline__ R re_v(cplx<R> a) { return a.re; }
__host__ __device__ __forceinline__ float im_v(float) { return 0.f; }
__host__ __device__ __forceinline__ double im_v(double) { return 0.0; }
template <typename R> __host__ __device__ __forceinline__ R im_v(cplx<R> a) { return a.im; }

// acc += a * b  (mixed real/complex); fused where the types allow
__device__ __forceinline__ void fma_acc(float& acc, float a, float b) { acc = fmaf(a, b, acc); }
__device__ __forceinline__ void fma_acc(double& acc, double a, double b) { acc = fma(a, b, acc); }
template <typename R> __device__ __forceinline__ void fma_acc(cplx<R>& acc, R a, cplx<R> b) {
  acc.re = fma(a, b.re, acc.re);
  acc.im = fma(a, b.im, acc.im);
}
template <typename R> __device__ __forceinline__ void fma_acc(cplx<R>& acc, cplx<R> a, R b) {
  acc.re = fma(a.re, b, acc.re);
  acc.im = fma(a.im, b, acc.im);
}
template <typename R> __device__ __forceinline__ void fma_acc(cplx<R>& acc, cplx<R> a, cplx<R> b) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(-a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(a.im, b.re, acc.im);
}

// conversion between element types (complex -> real keeps the real part)
template <typename To, typename From> struct conv;
template <> struct conv<float, float> { __host__ __device__ static float f(float a) { return a; } };
template <> struct conv<double, double> { __host__ __device__ static double f(double a) { return a; } };
template <> struct conv<float, double> { __host__ __device__ static float f(double a) { return (float)a; } };
template <> struct conv<double, float> { __host__ __device__ static double f(float a) { return (double)a; } };
template <typename R, typename S> struct conv<cplx<R>, S> {
  __host__ __device__ static cplx<R> f(S a) { return {(R)a, (R)0}; }
};
template <typename R, typename S> struct conv<cplx<R>, cplx<S>> {
  __host__ __device__ static cplx<R> f(cplx<S> a) { return {(R)a.re, (R)a.im}; }
};
template <typename S> struct conv<float, cplx<S>> {
  __host__ __device__ static float f(cplx<S> a) { return (float)a.re; }
};
template <typename S> struct conv<double, cplx<S>> {
  __host__ __device__ static double f(cplx<S> a) { return (double)a.re; }
};
template <typename To, typename From> __host__ __device__ __forceinline__ To cvt(From a) {
  return conv<To, From>::f(a);
}

// read-only cached loads for real and complex element types
__device__ __forceinline__ float ldg_v(const float* p) { return __ldg(p); }
__device__ __forceinline__ double ldg_v(const double* p) { return __ldg(p); }
__device__ __forceinline__ cplx<float> ldg_v(const cplx<float>* p) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(p));
  return {v.x, v.y};
}
__device__ __forceinline__ cplx<double> ldg_v(const cplx<double>* p) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}

// ------------------------------------------------------------------ warp
template <typename R> __device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ context
struct ltb_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  std::string last_error;
  int64_t launches = 0;
  // small pinned host scratch for reduction results
  double* h_scratch = nullptr;
  double* d_scratch = nullptr;  // 64 doubles
  unsigned int* d_counter = nullptr;
  unsigned long long* d_stats = nullptr;  // [0] Jacobi slices, [1] Jacobi sweeps
  // copy streams of the pipelined host-to-host l_product (created on first use)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  // split batched SVT (ltb_svt_carry_impl): a high- and a low-priority stream (first use)
  cudaStream_t split_hi = nullptr, split_hi2 = nullptr, split_lo = nullptr;
  // pageable host copies: two pinned staging buffers and their DMA events (first use)
  void* h_stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  // pinned staging of whole pageable operands (host-to-host l_product), grown on demand
  void* h_big = nullptr;
  size_t h_big_bytes = 0;
  // per-context test / profiling options (ltb_ctx_set_option)
  int opt_force_blocked = 0;                       // route every SVD through the blocked Jacobi tier
  unsigned long long* opt_tc_timeline = nullptr;   // tcgen05 kernels: per-tile clock stamps (CTA 0)
  unsigned long long* opt_qr_timeline = nullptr;   // QR-preconditioned Jacobi: stage stamps (CTA 0)
  int opt_full_sweeps = 0;   // carried complex SVT: no truncated sweeps
  int opt_jacobi_pairs = 0;  // warm Cholesky Jacobi: 0 / 2 two-column blocks, 1 one pair per team, 3 four-column blocks
};

struct ltb_spec {
  ltb_ctx* ctx = nullptr;
  int ntrail = 0;
  int64_t trail_dims[16] = {0};
  int64_t P = 1;
  int nmodes = 0;
  int axes[16] = {0};
  int sizes[16] = {0};
  int is_complex = 0;
  // device copies: [precision 0=f32,1=f64] x [0=fwd,1=inv]; element type
  // is real or complex according to is_complex; per-mode offsets (elements)
  void* d_mats[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int64_t mat_off[16] = {0};
  int64_t mat_total = 0;
  // real specs, per direction [0=fwd,1=inv] and mode: the mode matrix A (n even) has the
  // even/odd symmetry of the DCT-II (1: A[i][n-1-j] = (-1)^i A[i][j]) or of its transpose
  // (2: A[n-1-i][j] = (-1)^j A[i][j]), 0 none; the fp32 tile engine then halves the mode
  // product's multiply-adds (xform_tile: mode_step_f2_sym*)
  int sym[2][16] = {{0}, {0}};
  // real specs with P <= kKronMax: the dense Kronecker matrix of L and of L^{-1}
  // (C-order trailing index), fp32, for the tensor-core transform path
  float* d_kron[2] = {nullptr, nullptr};  // [P*P raw fp32 | P*P 3xTF32 lo part]
  // complex specs whose modes are real or have exactly Hermitian rows (the
  // DFT): slice q of a REAL tensor's transform is the conjugate of slice
  // partner[q]; uniq lists one slice of every pair (q <= partner[q])
  int64_t n_unique = 0;
  int* d_uniq = nullptr;
  int* d_partner = nullptr;
};

constexpr int64_t kKronMax = 512;

// fp32 tensor-core GEMM (ltb_tc_gemm.cu); LTB_EUNSUPPORTED when the shape /
// alignment cannot take the tcgen05 path
int ltb_tc_gemm_f32(ltb_ctx* ctx, int64_t batch, int64_t M, int64_t N, int64_t K, bool a_mn, const float* A,
                    int64_t lda, int64_t sa, bool b_mn, const float* B, int64_t ldb, int64_t sb, float* C,
                    int64_t ldc, int64_t sc, int split, bool c_trans = false, const float* b_lo = nullptr,
                    const int* klim = nullptr, const float* rscale = nullptr, const float* cscale = nullptr,
                    const int* skip = nullptr);

// fused one-launch fp32 *_L product (ltb_lprod_fused.cuh): workspace bytes, and the launch
// (LTB_EUNSUPPORTED when the shape / spec does not fit; the caller then runs three launches)
int64_t ltb_lprod_fused_ws_bytes(int64_t P, int64_t I1, int64_t L, int64_t I2);
int ltb_lprod_fused_f32(ltb_ctx* ctx, const ltb_spec* spec, int64_t I1, int64_t L, int64_t I2, const float* A,
                        const float* B, float* C, void* ws, bool ws_clean);

// ------------------------------------------------------------------ errors
int ltb_set_error(ltb_ctx* ctx, int code, const char* fmt, ...);

#define LTB_CUDA_TRY(ctx, expr)                                                              \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      return ltb_set_error((ctx), _e == cudaErrorMemoryAllocation ? LTB_EOOM : LTB_ECUDA,    \
                           "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                           __LINE__);                                                        \
    }                                                                                        \
  } while (0)

#define LTB_LAUNCH_CHECK(ctx)                                                          \
  do {                                                                                 \
    (ctx)->launches++;                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess)                                                             \
      return ltb_set_error((ctx), LTB_ECUDA, "kernel launch failed: %s (%s:%d)",       \
                           cudaGetErrorString(_e), __FILE__, __LINE__);                \
  } while (0)

#define LTB_TRY(expr)           \
  do {                          \
    int _s = (expr);            \
    if (_s != LTB_OK) return _s; \
  } while (0)

inline size_t dtype_size(int dt) {
  switch (dt) {
    case LTB_F32: return 4;
    case LTB_F64: return 8;
    case LTB_C64: return 8;
    case LTB_C128: return 16;
  }
  return 0;
}
inline bool dtype_is_complex(int dt) { return dt == LTB_C64 || dt == LTB_C128; }
inline bool dtype_is_double(int dt) { return dt == LTB_F64 || dt == LTB_C128; }
inline bool dtype_valid(int dt) { return dt >= 0 && dt <= 3; }

// raise a kernel's dynamic shared-memory limit (and optionally prefer the max
// smem carveout) only the first time a larger size is needed: the attribute
// calls cost host time on every launch otherwise
int ltb_ensure_smem(ltb_ctx* ctx, const void* kern, size_t smem, bool carveout = false);
template <typename K> inline int ensure_smem(ltb_ctx* ctx, K kern, size_t smem, bool carveout = false) {
  return ltb_ensure_smem(ctx, reinterpret_cast<const void*>(kern), smem, carveout);
}
// cached cudaOccupancyMaxActiveBlocksPerMultiprocessor
int ltb_occupancy(const void* kern, int threads, size_t smem);

// host side of pageable copies (ltb_ctx.cu): pinned test, multi-threaded memcpy, and a
// per-context pinned scratch buffer grown on demand
extern "C" {
bool ltb_is_pinned(const void* p);
void ltb_host_copy(void* dst, const void* src, size_t n);
int ltb_pinned_scratch(ltb_ctx* ctx, size_t bytes, void** out);
}

// stream-ordered scratch allocation
int ltb_ws_alloc(ltb_ctx* ctx, size_t bytes, void** out);
void ltb_ws_free(ltb_ctx* ctx, void* p);

// Workspace of one call: every buffer is released (stream-ordered) when the scope ends,
// on the success path and on every early error return alike.
struct WsScope {
  ltb_ctx* ctx;
  void* p[24];
  int n = 0;
  explicit WsScope(ltb_ctx* c) : ctx(c) {}
  WsScope(const WsScope&) = delete;
  WsScope& operator=(const WsScope&) = delete;
  ~WsScope() {
    while (n > 0) ltb_ws_free(ctx, p[--n]);
  }
  template <typename T> int alloc(size_t bytes, T** out) {
    if (n == 24) return ltb_set_error(ctx, LTB_EOOM, "too many workspace buffers in one call");
    void* q = nullptr;
    const int st = ltb_ws_alloc(ctx, bytes, &q);
    if (st != LTB_OK) return st;
    p[n++] = q;
    *out = (T*)q;
    return LTB_OK;
  }
};

// internal entry points shared between translation units
int ltb_transform_impl(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse, int dtype_in,
                       int layout_in, const void* d_in, int dtype_out, int layout_out, void* d_out,
                       double* d_sumsq /* device, 2 doubles, may be null */);
int ltb_svt_carry_impl(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* G, double tau, float* out,
                       float* V, int warm, const int* skip);
int ltb_svt_carry64_impl(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const double* G, double tau,
                         double* out, double* V, int warm, const int* skip);
int ltb_svt_carry_c64_impl(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const void* d_g, double tau,
                           void* d_out, void* d_vt, int warm, const int* skip);
int ltb_svt_mirror_carry_c64_impl(ltb_ctx* ctx, const ltb_spec* spec, int64_t batch, int64_t I1, int64_t I2,
                                  const void* d_a, double tau, void* d_out, void* d_vt, int warm, const int* d_skip);
int ltb_svt_mirror_impl(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t batch, int64_t I1, int64_t I2,
                        const void* d_a, double tau, void* d_out, const int* d_skip);
int ltb_transform_pair_impl(ltb_ctx* ctx, const ltb_spec* spec, int64_t ntubes, int inverse, int dtype_in,
                            int layout_in, const void* d_in0, const void* d_in1, int dtype_out, int layout_out,
                            void* d_out0, void* d_out1);
int ltb_reduce_sumsq_dev(ltb_ctx* ctx, int dtype, int64_t n, const void* d_x, const void* d_y,
                         double* d_out /* 2 doubles */);
int ltb_gemm_impl(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, int64_t k, int op_a,
                  const void* d_a, int64_t lda, int64_t sa, int op_b, const void* d_b, int64_t ldb,
                  int64_t sb, void* d_c, int64_t ldc, int64_t sc, const int* d_mlim, const int* d_nlim,
                  const int* d_klim, const void* d_row_scale, const void* d_col_scale, const int* d_skip = nullptr);
// complex64 GEMM on the tcgen05 engine (ltb_gemm.cu): C = [conj] A * op(B), A m x k with K
// contiguous, B stored k x n (b_kn) or n x k; LTB_EUNSUPPORTED when it does not fit
int ltb_cgemm_tc(ltb_ctx* ctx, int64_t batch, int64_t m, int64_t n, int64_t k, bool conj_a, const void* d_a,
                 int64_t lda, int64_t sa, bool b_kn, bool conj_b, const void* d_b, int64_t ldb, int64_t sb,
                 void* d_c, int64_t ldc, int64_t sc, const float* rscale, const int* skip);
int ltb_svt_impl(ltb_ctx* ctx, int dtype, int64_t batch, int64_t m, int64_t n, const void* d_a,
                 double tau, const double* d_tau /* optional per-call device tau */, void* d_out,
                 const int* d_skip /* optional device flag: nonzero -> kernels return */);
