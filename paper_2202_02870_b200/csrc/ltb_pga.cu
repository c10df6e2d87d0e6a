// K4 + the PGA completion loop (pga_complete, completion.py:141-202).
//
// Per iteration k the device runs, with no host round trip:
//   1. xform tile kernel, prologue = the PGA gradient step fused into the load
//        y = x + beta_k (x - x_prev)                       (completion.py:170)
//        g = y - (P_Omega(y) - P_Omega(m))                 (completion.py:171)
//      (bit-packed observation mask, coalesced tube loads), forward transform,
//      slice-major store of the transform-domain stack;
//   2. the slice SVT (ltb_svd.cu) with tau = mu_k;
//   3. xform tile kernel, inverse transform, epilogue = real part + the fused
//      reductions sum (y - x+)^2, sum x+^2, sum (x+ - gt)^2, max x+,
//      sum Im^2 (completion.py:174-189, transforms.py:217-225);
//   4. a one-warp finalisation that reduces the per-CTA partials in fixed
//      order, computes rel exactly as completion.py:174-181 and raises the
//      device stop flag when rel <= tol (completion.py:195-197).
// Every kernel first checks the stop flag, so a chunk of iterations can be
// enqueued back to back; the host only reads the records at chunk end.
// The scalar recurrences (mu_k, t_k) stay on the host, exactly as the reference
// computes them, and arrive as per-iteration arrays.
#include <algorithm>
#include <vector>

#include "ltb_xform_tile.cuh"

struct ltb_pga {
  ltb_ctx* ctx = nullptr;
  const ltb_spec* spec = nullptr;
  int dtype = LTB_F64;  // real compute dtype
  int hat_dtype = LTB_F64;
  int64_t I1 = 0, I2 = 0, P = 1, NT = 0, E = 0;
  void* x[3] = {nullptr, nullptr, nullptr};
  void* pobs = nullptr;
  void* gt = nullptr;
  uint32_t* mask = nullptr;
  void* hat_a = nullptr;
  void* hat_b = nullptr;
  double* partials = nullptr;
  int64_t nblocks = 0;
  double* d_records = nullptr;  // chunk x 5
  int* d_state = nullptr;       // [0] stop flag, [1] executed iterations
  double* d_scalars = nullptr;  // [0] sum pobs^2
  int records_cap = 0;
  int done = 0;  // iterations executed so far
  bool converged = false;
  double pobs_sumsq = 0.0;
  // fp32 real transform domain: right singular bases carried between iterations
  // (ltb_svt_carry_impl); allocated on first use, warm after the first SVT
  float* vcarry = nullptr;
  double* vcarry64 = nullptr;  // the same for an fp64 real transform domain
  void* vcarry_c = nullptr;    // complex64 domain, blocked tier: VT of the unique slices (ltb_svt_carry_c64_impl)
  int warm = 0;
  bool carry_off = false;
  bool tc_off = false;        // the tensor-core transform path declined this shape
  int64_t nblocks_cap = 0;    // partials capacity (blocks x 5 doubles)
};

// 1: fp32 PGA carries the right singular bases between iterations (warm-started SVT)
constexpr int g_pga_carry = 1;
// 1: fp32 real specs with a Kronecker matrix transform on the tensor cores inside PGA.
// Off by default: 3xTF32 keeps ~21 mantissa bits per product, and over ~90 iterations of
// the momentum recursion the iterate drifts to 1.0e-4 of the fp64 oracle (the fp32 tile
// engine stays below it); +8% it/s on config 3 when enabled
constexpr int g_pga_tc = 0;

namespace {

// buffer roles for iteration k (1-based): x_cur, x_prev, x_next
constexpr int kCur[3] = {0, 2, 1}, kPrev[3] = {1, 0, 2}, kNext[3] = {2, 1, 0};
inline int cur_of(int k) { return kCur[(k - 1) % 3]; }
inline int prev_of(int k) { return kPrev[(k - 1) % 3]; }
inline int next_of(int k) { return kNext[(k - 1) % 3]; }

template <typename R> __device__ __forceinline__ R momentum(R xc, R xp, R beta);
template <> __device__ __forceinline__ double momentum<double>(double xc, double xp, double beta) {
  // x_cur + beta * (x_cur - x_prev), no contraction (mirrors numpy's rounding)
  return __dadd_rn(xc, __dmul_rn(beta, __dsub_rn(xc, xp)));
}
template <> __device__ __forceinline__ float momentum<float>(float xc, float xp, float beta) {
  return __fadd_rn(xc, __fmul_rn(beta, __fsub_rn(xc, xp)));
}
template <typename R> __device__ __forceinline__ R gradient_point(R y, R pobs, bool observed);
template <> __device__ __forceinline__ double gradient_point<double>(double y, double pobs, bool observed) {
  return __dsub_rn(y, __dsub_rn(observed ? y : 0.0, pobs));
}
template <> __device__ __forceinline__ float gradient_point<float>(float y, float pobs, bool observed) {
  return __fsub_rn(y, __fsub_rn(observed ? y : 0.f, pobs));
}

// the PGA prologue: x_cur, x_prev, p_obs and the tile's packed mask words are staged by
// cp.async (all of a thread's copies in flight at once; x_cur in S0, x_prev in S1,
// p_obs in the extra tile, R views of S1 / extra when the tile is complex), then
// finish() forms the gradient point in place
template <typename R>
struct LoadPGA {
  static constexpr int kExtraBufs = 1;
  static constexpr bool kMaskWords = true;
  const R* xc;
  const R* xp;
  const R* pobs;
  const uint32_t* mask;
  R beta;
  template <typename Tc>
  __device__ __forceinline__ void stage(const XformParams& p, Tc* S0, Tc* S1, unsigned char* extra, R*& sx, R*& sp,
                                        R*& so, uint32_t*& sm) const {
    const size_t tile = (size_t)p.P * p.pitch;
    if constexpr (std::is_same<Tc, R>::value) {
      sx = S0;
      sp = S1;
    } else {
      sx = reinterpret_cast<R*>(S1);
      sp = sx + tile;
    }
    so = reinterpret_cast<R*>(extra);
    sm = reinterpret_cast<uint32_t*>(extra + tile * sizeof(Tc));
  }
  template <typename Tc>
  __device__ __forceinline__ void load(const XformParams& p, Tc* S0, Tc* S1, unsigned char* extra, int64_t tube0,
                                       int nt, int tid) const {
    const int P = p.P, pitch = p.pitch;
    const int64_t e0 = tube0 * P;
    const int cnt = nt * P;
    R *sx, *sp, *so;
    uint32_t* sm;
    stage(p, S0, S1, extra, sx, sp, so, sm);
    for (int l = tid; l < cnt; l += kXformThreads) {
      int t, q;
      split_tube(l, P, p.invP, t, q);
      const int i = q * pitch + t;
      cp_async<sizeof(R)>(sx + i, xc + e0 + l);
      cp_async<sizeof(R)>(sp + i, xp + e0 + l);
      cp_async<sizeof(R)>(so + i, pobs + e0 + l);
    }
    const int64_t w0 = e0 >> 5;
    const int nw = (int)(((e0 + cnt - 1) >> 5) - w0 + 1);
    for (int w = tid; w < nw; w += kXformThreads) cp_async<4>(sm + w, mask + w0 + w);
  }
  template <typename Tc>
  __device__ __forceinline__ void finish(const XformParams& p, Tc* S0, Tc* S1, unsigned char* extra, int64_t tube0,
                                         int nt, int tid) const {
    const int P = p.P, pitch = p.pitch;
    const int64_t e0 = tube0 * P;
    const int cnt = nt * P;
    const int b0 = (int)(e0 & 31);  // bit of element e0 in the first staged word
    R *sx, *sp, *so;
    uint32_t* sm;
    stage(p, S0, S1, extra, sx, sp, so, sm);
    for (int l = tid; l < cnt; l += kXformThreads) {
      int t, q;
      split_tube(l, P, p.invP, t, q);
      const int i = q * pitch + t;
      const R y = momentum<R>(sx[i], sp[i], beta);
      const int bit = b0 + l;
      const bool obs = (sm[bit >> 5] >> (bit & 31)) & 1u;
      S0[i] = cvt<Tc>(gradient_point<R>(y, so[i], obs));
    }
  }
};

// slots: 0 sum (y - x+)^2, 1 sum x+^2, 2 sum (x+ - gt)^2, 3 max x+, 4 sum Im^2
template <typename R>
struct StorePGA {
  static constexpr int NACC = 5;
  static constexpr unsigned MAXMASK = 1u << 3;
  R* xn;
  const R* xc;
  const R* xp;
  const R* gt;
  R beta;
  template <typename Tc>
  __device__ __forceinline__ void store(const XformParams& p, const Tc* S, int64_t tube0, int nt, int tid,
                                        double* acc) const {
    const int P = p.P, pitch = p.pitch;
    const int64_t e0 = tube0 * P;
    const int cnt = nt * P;
    constexpr int U = 8;  // U elements' global loads issued before any is used
    for (int l0 = tid; l0 < cnt; l0 += U * kXformThreads) {
      R c[U], pv[U], g[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = l0 + u * kXformThreads;
        if (l < cnt) {
          c[u] = xc[e0 + l];
          pv[u] = xp[e0 + l];
          g[u] = gt ? gt[e0 + l] : R(0);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int l = l0 + u * kXformThreads;
        if (l < cnt) {
          int t, q;
          split_tube(l, P, p.invP, t, q);
          const Tc v = S[q * pitch + t];
          const R x1 = re_v(v);
          const R y = momentum<R>(c[u], pv[u], beta);
          const double d = (double)y - (double)x1;
          acc[0] += d * d;
          acc[1] += (double)x1 * (double)x1;
          if (gt) {
            const double dg = (double)x1 - (double)g[u];
            acc[2] += dg * dg;
          }
          acc[3] = fmax(acc[3], (double)x1);
          acc[4] += (double)im_v(v) * (double)im_v(v);
          xn[e0 + l] = x1;
        }
      }
    }
  }
};

// fp32 real specs with a Kronecker matrix: the gradient step as its own pass (the tensor-core
// transform reads it with TMA) and the five norms of StorePGA as a pass after the inverse
__global__ void pga_grad_kernel(int64_t E, const float* __restrict__ xc, const float* __restrict__ xp,
                                const float* __restrict__ pobs, const uint32_t* __restrict__ mask, float beta,
                                float* __restrict__ g, const int* __restrict__ skip) {
  if (skip && *skip) return;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const float y = momentum<float>(xc[e], xp[e], beta);
    const bool obs = (mask[e >> 5] >> (e & 31)) & 1u;
    g[e] = gradient_point<float>(y, pobs[e], obs);
  }
}

// per-block partials in StorePGA's slot order (fixed grid: the reduction order is deterministic)
__global__ void pga_norms_kernel(int64_t E, const float* __restrict__ xn, const float* __restrict__ xc,
                                 const float* __restrict__ xp, const float* __restrict__ gt, float beta,
                                 double* __restrict__ partials, const int* __restrict__ skip) {
  if (skip && *skip) return;
  double acc[5] = {0.0, 0.0, 0.0, -1.0e308, 0.0};
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const float x1 = xn[e];
    const float y = momentum<float>(xc[e], xp[e], beta);
    const double d = (double)y - (double)x1;
    acc[0] += d * d;
    acc[1] += (double)x1 * (double)x1;
    if (gt) {
      const double dg = (double)x1 - (double)gt[e];
      acc[2] += dg * dg;
    }
    acc[3] = fmax(acc[3], (double)x1);
  }
  __shared__ double red[5][8];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = k == 3 ? fmax(v, w) : v + w;
    }
    if (lane == 0) red[k][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    const int k = threadIdx.x;
    double v = k == 3 ? -1.0e308 : 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = k == 3 ? fmax(v, red[k][w]) : v + red[k][w];
    partials[(int64_t)blockIdx.x * 5 + k] = v;
  }
}

// reduce the per-CTA partials of one iteration, record, and decide to stop
__global__ void pga_finalize_kernel(const double* __restrict__ partials, int64_t nblocks, double* __restrict__ rec,
                                    int* __restrict__ state, const double* __restrict__ scalars, double tol) {
  if (state[0]) return;
  const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ double vals[5];
  if (slot < 5) {
    const bool mx = slot == 3;
    double v = mx ? -1.0e308 : 0.0;
    for (int64_t i = lane; i < nblocks; i += 32) {
      const double w = partials[i * 5 + slot];
      v = mx ? fmax(v, w) : v + w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = mx ? fmax(v, w) : v + w;
    }
    if (lane == 0) vals[slot] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 5; ++k) rec[k] = vals[k];
    const double num = sqrt(vals[0]);
    const double den = sqrt(vals[1]);
    double rel;
    if (den > 0.0)
      rel = num / den;
    else if (scalars[0] == 0.0)
      rel = 0.0;
    else
      rel = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    state[1] += 1;
    if (rel <= tol) state[0] = 1;
  }
}

template <typename R>
__global__ void pga_setup_kernel(int64_t E, const double* __restrict__ m, const uint8_t* __restrict__ mask8,
                                 R* __restrict__ pobs) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    pobs[e] = mask8[e] ? (R)m[e] : (R)0;
}

__global__ void pack_mask_kernel(int64_t E, const uint8_t* __restrict__ mask8, uint32_t* __restrict__ bits) {
  const int64_t words = (E + 31) / 32;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t e = w * 32 + b;
      if (e < E && mask8[e]) v |= 1u << b;
    }
    bits[w] = v;
  }
}

template <typename R>
__global__ void pga_fetch_kernel(int64_t E, const R* __restrict__ x, const R* __restrict__ pobs,
                                 const uint32_t* __restrict__ bits, const double* __restrict__ m, int reimpose,
                                 double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const bool obs = (bits[e >> 5] >> (e & 31)) & 1u;
    out[e] = (reimpose && obs) ? m[e] : (double)x[e];
  }
}

// sharded PGA (multi-GPU): the local reduction of the fused inverse's per-CTA partials in a
// fixed order, laid out for the cross-rank all-reduces: [0..3] = sum (y - x+)^2, sum x+^2,
// sum (x+ - gt)^2, sum Im^2 (SUM), [4] = max x+ (MAX)
__global__ void pga_shard_sums_kernel(const double* __restrict__ partials, int64_t nblocks,
                                      double* __restrict__ sums, const int* __restrict__ state) {
  if (state && state[0]) return;
  const int slot = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (slot >= 5) return;
  const bool mx = slot == 3;
  double v = mx ? -1.0e308 : 0.0;
  for (int64_t i = lane; i < nblocks; i += 32) {
    const double w = partials[i * 5 + slot];
    v = mx ? fmax(v, w) : v + w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = mx ? fmax(v, w) : v + w;
  }
  if (lane == 0) sums[slot == 3 ? 4 : (slot == 4 ? 3 : slot)] = v;
}

// the stop rule of completion.py:174-181,195-197 on the all-reduced sums (identical on every
// rank); rec in ltb_pga_run's record order {sum (y-x+)^2, sum x+^2, sum (x+-gt)^2, max x+, sum Im^2}
__global__ void pga_shard_decide_kernel(const double* __restrict__ sums, double pobs_sumsq, double tol,
                                        double* __restrict__ rec, int* __restrict__ state) {
  if (state[0]) return;
  rec[0] = sums[0];
  rec[1] = sums[1];
  rec[2] = sums[2];
  rec[3] = sums[4];
  rec[4] = sums[3];
  const double num = sqrt(sums[0]), den = sqrt(sums[1]);
  double rel;
  if (den > 0.0)
    rel = num / den;
  else if (pobs_sumsq == 0.0)
    rel = 0.0;
  else
    rel = __longlong_as_double(0x7ff0000000000000LL);
  state[1] += 1;
  if (rel <= tol) state[0] = 1;
}

// tile plan of the fused transforms for this spec and compute type (0 if too long)
template <typename Tc, typename Tm>
int pga_plan(const ltb_spec* spec, int64_t NT, int inverse, XformParams& p, size_t* smem) {
  p = XformParams{};
  p.NT = NT;
  build_steps(spec, inverse, p);
  // the forward's LoadPGA stages p_obs in one extra tile plus the packed mask words
  return inverse ? plan_tile<Tc, Tm>(p, smem) : plan_tile<Tc, Tm>(p, smem, LoadPGA<float>::kExtraBufs, true);
}

// the SVT step of one iteration (hat_a -> hat_b): carried bases for fp32 real transform
// domains, otherwise the conjugate-mirrored / plain SVT
int pga_svt(ltb_pga* g, double mu, const int* skip) {
  ltb_ctx* ctx = g->ctx;
  // fp32 real transform domain: the SVT carries the slices' right bases between iterations
  int carry = LTB_EUNSUPPORTED;
  if (g->hat_dtype == LTB_F32 && !g->carry_off && g_pga_carry) {
    const int64_t n = std::min(g->I1, g->I2);
    if (!g->vcarry) LTB_TRY(ltb_ws_alloc(ctx, sizeof(float) * g->P * n * n, (void**)&g->vcarry));
    carry = ltb_svt_carry_impl(ctx, g->P, g->I1, g->I2, (const float*)g->hat_a, mu, (float*)g->hat_b, g->vcarry,
                               g->warm, skip);
    if (carry == LTB_OK) g->warm = 1;
    else if (carry == LTB_EUNSUPPORTED) g->carry_off = true;
    else return carry;
  }
  // fp64 real transform domain: the same carry with a warm-started resident Jacobi
  if (g->hat_dtype == LTB_F64 && !g->carry_off && g_pga_carry) {
    const int64_t n = std::min(g->I1, g->I2);
    if (!g->vcarry64) LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * g->P * n * n, (void**)&g->vcarry64));
    carry = ltb_svt_carry64_impl(ctx, g->P, g->I1, g->I2, (const double*)g->hat_a, mu, (double*)g->hat_b,
                                 g->vcarry64, g->warm, skip);
    if (carry == LTB_OK) g->warm = 1;
    else if (carry == LTB_EUNSUPPORTED) g->carry_off = true;
    else return carry;
  }
  // complex64 transform domain with slices beyond shared memory: carried bases for the
  // blocked Jacobi tier (one slice of every conjugate pair)
  if (g->hat_dtype == LTB_C64 && !g->carry_off && g_pga_carry) {
    const int64_t n = std::min(g->I1, g->I2);
    const int64_t nu = (g->spec->d_uniq && g->spec->P == g->P) ? g->spec->n_unique : g->P;
    if (!g->vcarry_c) LTB_TRY(ltb_ws_alloc(ctx, 2 * sizeof(float) * nu * n * n, &g->vcarry_c));
    carry = ltb_svt_mirror_carry_c64_impl(ctx, g->spec, g->P, g->I1, g->I2, g->hat_a, mu, g->hat_b, g->vcarry_c,
                                          g->warm, skip);
    if (carry == LTB_OK) g->warm = 1;
    else if (carry == LTB_EUNSUPPORTED) g->carry_off = true;
    else return carry;
  }
  // otherwise (conjugate slice pairs of the real iterate are solved once)
  if (carry != LTB_OK)
    LTB_TRY(ltb_svt_mirror_impl(ctx, g->spec, g->hat_dtype, g->P, g->I1, g->I2, g->hat_a, mu, g->hat_b, skip));
  return LTB_OK;
}

template <typename R, typename Tc, typename Tm>
int pga_transforms(ltb_pga* g, int k, double beta, double mu, double tol, double* rec) {
  ltb_ctx* ctx = g->ctx;
  const R* xc = (const R*)g->x[cur_of(k)];
  const R* xp = (const R*)g->x[prev_of(k)];
  R* xn = (R*)g->x[next_of(k)];
  const int* skip = g->d_state;
  const int dbl = std::is_same<R, double>::value ? 1 : 0;
  XformParams p;
  size_t smem = 0;
  // fp32 real specs with a Kronecker matrix: gradient pass + tensor-core transform (hat_b is
  // free until the SVT writes it, so it holds the gradient), then SVT, tensor-core inverse
  // and the norms pass; any shape the tcgen05 path declines takes the fused tile engine
  if constexpr (std::is_same<R, float>::value && std::is_same<Tc, float>::value) {
    if (g->spec->d_kron[0] && g_pga_tc && !g->tc_off) {
      const int64_t P = g->P, NT = g->NT, E = g->E;
      const float* Kf = g->spec->d_kron[0];
      const float* Ki = g->spec->d_kron[1];
      const unsigned eg = grid_for(E, 256, ctx->num_sms * 8);
      pga_grad_kernel<<<eg, 256, 0, ctx->stream>>>(E, xc, xp, (const float*)g->pobs, g->mask, (float)beta,
                                                   (float*)g->hat_b, skip);
      LTB_LAUNCH_CHECK(ctx);
      int st = ltb_tc_gemm_f32(ctx, 1, NT, P, P, false, (const float*)g->hat_b, P, 0, false, Kf, P, 0,
                               (float*)g->hat_a, NT, 0, 3, true, Kf + P * P, nullptr, nullptr, nullptr, skip);
      if (st == LTB_OK) {
        LTB_TRY(pga_svt(g, mu, skip));
        st = ltb_tc_gemm_f32(ctx, 1, NT, P, P, true, (const float*)g->hat_b, NT, 0, false, Ki, P, 0, xn, P, 0, 3,
                             false, Ki + P * P, nullptr, nullptr, nullptr, skip);
        if (st != LTB_OK) return st == LTB_EUNSUPPORTED ? ltb_set_error(ctx, LTB_ECUDA, "pga: inverse tc path") : st;
        const int nb = (int)std::min<int64_t>(g->nblocks_cap, 2 * ctx->num_sms);
        pga_norms_kernel<<<nb, 256, 0, ctx->stream>>>(E, xn, xc, xp, (const float*)g->gt, (float)beta,
                                                      g->partials, skip);
        LTB_LAUNCH_CHECK(ctx);
        g->nblocks = nb;
        pga_finalize_kernel<<<1, 160, 0, ctx->stream>>>(g->partials, g->nblocks, rec, g->d_state, g->d_scalars,
                                                        tol);
        LTB_LAUNCH_CHECK(ctx);
        return LTB_OK;
      }
      if (st != LTB_EUNSUPPORTED) return st;
      g->tc_off = true;  // this shape stays on the fused tile engine
    }
  }
  // forward: gradient step fused into the load, slice-major store
  if (!pga_plan<Tc, Tm>(g->spec, g->NT, 0, p, &smem))
    return ltb_set_error(ctx, LTB_ESHAPE, "pga: tube too long for the fused transform");
  {
    LoadPGA<R> ld{xc, xp, (const R*)g->pobs, g->mask, (R)beta};
    StorePlain<Tc, false> st{(Tc*)g->hat_a, LTB_SLICE_MAJOR};
    LTB_TRY((launch_xform_tile<Tc, Tm>(ctx, p, ld, st, (const Tm*)g->spec->d_mats[dbl][0], nullptr, skip, smem)));
  }
  // slice SVT with tau = mu_k
  LTB_TRY(pga_svt(g, mu, skip));
  // inverse with the fused norms epilogue
  if (!pga_plan<Tc, Tm>(g->spec, g->NT, 1, p, &smem))
    return ltb_set_error(ctx, LTB_ESHAPE, "pga: tube too long for the fused transform");
  {
    StorePGA<R> st{xn, xc, xp, (const R*)g->gt, (R)beta};
    LoadPlain<Tc> ld{(const Tc*)g->hat_b, LTB_SLICE_MAJOR};
    LTB_TRY((launch_xform_tile<Tc, Tm>(ctx, p, ld, st, (const Tm*)g->spec->d_mats[dbl][1], g->partials, skip, smem,
                                       &g->nblocks)));
  }
  pga_finalize_kernel<<<1, 160, 0, ctx->stream>>>(g->partials, g->nblocks, rec, g->d_state, g->d_scalars, tol);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

template <typename R>
int pga_iteration(ltb_pga* g, int k, double beta, double mu, double tol, double* rec) {
  if (g->spec->is_complex) return pga_transforms<R, cplx<R>, cplx<R>>(g, k, beta, mu, tol, rec);
  return pga_transforms<R, R, R>(g, k, beta, mu, tol, rec);
}

}  // namespace

extern "C" {

int ltb_pga_create(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t i1, int64_t i2, const double* h_m,
                   const uint8_t* h_mask, const double* h_gt, ltb_pga** out) {
  *out = nullptr;
  if (dtype != LTB_F32 && dtype != LTB_F64) return ltb_set_error(ctx, LTB_EPARAM, "pga: compute dtype must be real");
  if (i1 < 1 || i2 < 1) return ltb_set_error(ctx, LTB_ESHAPE, "pga: empty slice");
  ltb_pga* g = new ltb_pga();
  g->ctx = ctx;
  g->spec = spec;
  g->dtype = dtype;
  const bool cm = spec->is_complex != 0;
  g->hat_dtype = cm ? (dtype == LTB_F64 ? LTB_C128 : LTB_C64) : dtype;
  g->I1 = i1;
  g->I2 = i2;
  g->P = spec->P;
  g->NT = i1 * i2;
  g->E = g->NT * g->P;
  const size_t rs = dtype_size(dtype), hs = dtype_size(g->hat_dtype);
  const int64_t E = g->E;
  size_t smem = 0;
  XformParams plan;
  const int tt = cm ? (dtype == LTB_F64 ? pga_plan<cplx<double>, cplx<double>>(spec, g->NT, 1, plan, &smem)
                                        : pga_plan<cplx<float>, cplx<float>>(spec, g->NT, 1, plan, &smem))
                    : (dtype == LTB_F64 ? pga_plan<double, double>(spec, g->NT, 1, plan, &smem)
                                        : pga_plan<float, float>(spec, g->NT, 1, plan, &smem));
  if (!tt) {
    delete g;
    return ltb_set_error(ctx, LTB_ESHAPE, "pga: tube of %lld elements does not fit the fused transform tile",
                         (long long)spec->P);
  }
  const int64_t nb = (g->NT + tt - 1) / tt;
  int st = LTB_OK;
  auto alloc = [&](size_t bytes, void** p) {
    if (st == LTB_OK) st = ltb_ws_alloc(ctx, bytes, p);
  };
  for (int k = 0; k < 3; ++k) alloc(rs * E, &g->x[k]);
  alloc(rs * E, &g->pobs);
  alloc(sizeof(uint32_t) * ((E + 31) / 32), (void**)&g->mask);
  alloc(hs * E, &g->hat_a);
  alloc(hs * E, &g->hat_b);
  alloc(sizeof(double) * 5 * nb, (void**)&g->partials);
  g->nblocks_cap = nb;
  alloc(sizeof(int) * 4, (void**)&g->d_state);
  alloc(sizeof(double) * 4, (void**)&g->d_scalars);
  if (h_gt) alloc(rs * E, &g->gt);
  double* d_m = nullptr;
  uint8_t* d_mask8 = nullptr;
  alloc(sizeof(double) * E, (void**)&d_m);
  alloc(E, (void**)&d_mask8);
  if (st != LTB_OK) {
    ltb_pga_destroy(g);
    return st;
  }
  cudaStream_t s = ctx->stream;
  cudaMemcpyAsync(d_m, h_m, sizeof(double) * E, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_mask8, h_mask, E, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(g->x[0], 0, rs * E, s);
  cudaMemsetAsync(g->x[1], 0, rs * E, s);
  cudaMemsetAsync(g->d_state, 0, sizeof(int) * 4, s);
  const int blocks = grid_for(E, 256, ctx->num_sms * 8);
  pack_mask_kernel<<<grid_for((E + 31) / 32, 256, ctx->num_sms * 8), 256, 0, s>>>(E, d_mask8, g->mask);
  ctx->launches++;
  if (dtype == LTB_F64) {
    pga_setup_kernel<double><<<blocks, 256, 0, s>>>(E, d_m, d_mask8, (double*)g->pobs);
  } else {
    pga_setup_kernel<float><<<blocks, 256, 0, s>>>(E, d_m, d_mask8, (float*)g->pobs);
  }
  ctx->launches++;
  if (h_gt) {
    cudaMemcpyAsync(d_m, h_gt, sizeof(double) * E, cudaMemcpyHostToDevice, s);
    st = ltb_convert(ctx, E, LTB_F64, d_m, dtype, g->gt);
  }
  if (st == LTB_OK) st = ltb_reduce_sumsq_dev(ctx, dtype, E, g->pobs, nullptr, ctx->d_scratch);
  if (st == LTB_OK) {
    cudaMemcpyAsync(g->d_scalars, ctx->d_scratch, sizeof(double), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(&g->pobs_sumsq, ctx->d_scratch, sizeof(double), cudaMemcpyDeviceToHost, s);
  }
  ltb_ws_free(ctx, d_m);
  ltb_ws_free(ctx, d_mask8);
  cudaError_t e = cudaStreamSynchronize(s);
  if (st == LTB_OK && e != cudaSuccess) st = ltb_set_error(ctx, LTB_ECUDA, "pga setup: %s", cudaGetErrorString(e));
  if (st != LTB_OK) {
    ltb_pga_destroy(g);
    return st;
  }
  *out = g;
  return LTB_OK;
}

int ltb_pga_pobs_sumsq(ltb_pga* g, double* h_out) {
  *h_out = g->pobs_sumsq;
  return LTB_OK;
}

int ltb_pga_run(ltb_pga* g, int k0, int count, const double* h_beta, const double* h_mu, double tol,
                double* h_records, int* h_done, int* h_converged) {
  ltb_ctx* ctx = g->ctx;
  *h_done = 0;
  *h_converged = g->converged ? 1 : 0;
  if (count <= 0 || g->converged) return LTB_OK;
  if (k0 != g->done + 1) return ltb_set_error(ctx, LTB_EPARAM, "pga: iterations must be run in order");
  if (count > g->records_cap) {
    if (g->d_records) ltb_ws_free(ctx, g->d_records);
    g->d_records = nullptr;
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * 5 * count, (void**)&g->d_records));
    g->records_cap = count;
  }
  for (int i = 0; i < count; ++i) {
    const int k = k0 + i;
    int st = g->dtype == LTB_F64 ? pga_iteration<double>(g, k, h_beta[i], h_mu[i], tol, g->d_records + 5 * i)
                                 : pga_iteration<float>(g, k, h_beta[i], h_mu[i], tol, g->d_records + 5 * i);
    if (st != LTB_OK) return st;
  }
  int state[2] = {0, 0};
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(state, g->d_state, sizeof(int) * 2, cudaMemcpyDeviceToHost, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(h_records, g->d_records, sizeof(double) * 5 * count, cudaMemcpyDeviceToHost,
                                    ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  LTB_CUDA_TRY(ctx, cudaGetLastError());
  const int executed = state[1] - g->done;
  g->done = state[1];
  g->converged = state[0] != 0;
  *h_done = executed;
  *h_converged = g->converged ? 1 : 0;
  return LTB_OK;
}

int ltb_pga_current(ltb_pga* g, void** d_x) {
  *d_x = g->x[cur_of(g->done + 1)];
  return LTB_OK;
}

int ltb_pga_fetch(ltb_pga* g, int reimpose_observed, double* h_x) {
  ltb_ctx* ctx = g->ctx;
  const int64_t E = g->E;
  double* d_out = nullptr;
  double* d_m = nullptr;
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * E, (void**)&d_out));
  const void* xc = g->x[cur_of(g->done + 1)];
  const int blocks = grid_for(E, 256, ctx->num_sms * 8);
  if (reimpose_observed) {
    // observed entries come back as m itself: p_obs holds m there in compute precision,
    // so re-upload is avoided only when the compute dtype is float64
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(double) * E, (void**)&d_m));
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(d_m, h_x, sizeof(double) * E, cudaMemcpyHostToDevice, ctx->stream));
  }
  if (g->dtype == LTB_F64)
    pga_fetch_kernel<double><<<blocks, 256, 0, ctx->stream>>>(E, (const double*)xc, (const double*)g->pobs, g->mask,
                                                              d_m, reimpose_observed, d_out);
  else
    pga_fetch_kernel<float><<<blocks, 256, 0, ctx->stream>>>(E, (const float*)xc, (const float*)g->pobs, g->mask,
                                                             d_m, reimpose_observed, d_out);
  LTB_LAUNCH_CHECK(ctx);
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(h_x, d_out, sizeof(double) * E, cudaMemcpyDeviceToHost, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ltb_ws_free(ctx, d_out);
  if (d_m) ltb_ws_free(ctx, d_m);
  return LTB_OK;
}

void ltb_pga_destroy(ltb_pga* g) {
  if (!g) return;
  ltb_ctx* ctx = g->ctx;
  for (int k = 0; k < 3; ++k) ltb_ws_free(ctx, g->x[k]);
  ltb_ws_free(ctx, g->pobs);
  ltb_ws_free(ctx, g->gt);
  ltb_ws_free(ctx, g->mask);
  ltb_ws_free(ctx, g->hat_a);
  ltb_ws_free(ctx, g->hat_b);
  ltb_ws_free(ctx, g->partials);
  ltb_ws_free(ctx, g->d_records);
  ltb_ws_free(ctx, g->d_state);
  ltb_ws_free(ctx, g->d_scalars);
  ltb_ws_free(ctx, g->vcarry);
  ltb_ws_free(ctx, g->vcarry64);
  ltb_ws_free(ctx, g->vcarry_c);
  cudaStreamSynchronize(ctx->stream);
  delete g;
}

// ---------------------------------------------------------------- sharded PGA steps
int ltb_pack_mask(ltb_ctx* ctx, int64_t n, const uint8_t* d_mask, uint32_t* d_bits) {
  if (n < 0) return ltb_set_error(ctx, LTB_ESHAPE, "pack_mask: negative length");
  if (n == 0) return LTB_OK;
  pack_mask_kernel<<<grid_for((n + 31) / 32, 256, ctx->num_sms * 8), 256, 0, ctx->stream>>>(n, d_mask, d_bits);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

int ltb_pga_shard_forward(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t ntubes, double beta,
                          const void* d_xc, const void* d_xp, const void* d_pobs, const uint32_t* d_bits,
                          void* d_hat, const int* d_state) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  if (dtype != LTB_F32 && dtype != LTB_F64) return ltb_set_error(ctx, LTB_EPARAM, "pga shard: real dtype expected");
  if (ntubes <= 0) return LTB_OK;
  auto run = [&](auto rt, auto ct) -> int {
    using R = decltype(rt);
    using Tc = decltype(ct);
    XformParams p;
    size_t smem = 0;
    if (!pga_plan<Tc, Tc>(spec, ntubes, 0, p, &smem))
      return ltb_set_error(ctx, LTB_ESHAPE, "pga shard: tube too long for the fused transform");
    LoadPGA<R> ld{(const R*)d_xc, (const R*)d_xp, (const R*)d_pobs, d_bits, (R)beta};
    StorePlain<Tc, false> st{(Tc*)d_hat, LTB_SLICE_MAJOR};
    const int dbl = std::is_same<R, double>::value ? 1 : 0;
    return launch_xform_tile<Tc, Tc>(ctx, p, ld, st, (const Tc*)spec->d_mats[dbl][0], nullptr, d_state, smem);
  };
  if (spec->is_complex)
    return dtype == LTB_F64 ? run(double(), cplx<double>()) : run(float(), cplx<float>());
  return dtype == LTB_F64 ? run(double(), double()) : run(float(), float());
}

int ltb_pga_shard_svt(ltb_ctx* ctx, int dtype, int64_t batch, int64_t I1, int64_t I2, const void* d_hat, double tau,
                      void* d_out, void* d_v, int warm, const int* d_state) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "pga shard svt: bad dtype");
  if (!(tau >= 0)) return ltb_set_error(ctx, LTB_EPARAM, "tau must be >= 0, got %g", tau);
  if (batch <= 0 || I1 <= 0 || I2 <= 0) return LTB_OK;
  if (d_v && dtype == LTB_F32) {
    const int st = ltb_svt_carry_impl(ctx, batch, I1, I2, (const float*)d_hat, tau, (float*)d_out, (float*)d_v, warm,
                                      d_state);
    if (st != LTB_EUNSUPPORTED) return st;
  }
  if (d_v && dtype == LTB_F64) {
    const int st = ltb_svt_carry64_impl(ctx, batch, I1, I2, (const double*)d_hat, tau, (double*)d_out,
                                        (double*)d_v, warm, d_state);
    if (st != LTB_EUNSUPPORTED) return st;
  }
  if (d_v && dtype == LTB_C64) {  // slices beyond the shared-memory tier: carried blocked Jacobi (d_v holds V^T)
    const int st = ltb_svt_carry_c64_impl(ctx, batch, I1, I2, d_hat, tau, d_out, d_v, warm, d_state);
    if (st != LTB_EUNSUPPORTED) return st;
  }
  return ltb_svt_impl(ctx, dtype, batch, I1, I2, d_hat, tau, nullptr, d_out, d_state);
}

int ltb_pga_shard_inverse(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t ntubes, double beta,
                          const void* d_hat, const void* d_xc, const void* d_xp, const void* d_gt, void* d_xn,
                          double* d_sums, const int* d_state) {
  if (!spec) return ltb_set_error(ctx, LTB_ETRANSFORM, "null spec");
  if (dtype != LTB_F32 && dtype != LTB_F64) return ltb_set_error(ctx, LTB_EPARAM, "pga shard: real dtype expected");
  if (ntubes <= 0) {  // an empty shard contributes zero sums and no maximum
    const double z[5] = {0.0, 0.0, 0.0, 0.0, -1.0e308};
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(d_sums, z, sizeof(z), cudaMemcpyHostToDevice, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return LTB_OK;
  }
  WsScope ws(ctx);
  auto run = [&](auto rt, auto ct) -> int {
    using R = decltype(rt);
    using Tc = decltype(ct);
    XformParams p;
    size_t smem = 0;
    if (!pga_plan<Tc, Tc>(spec, ntubes, 1, p, &smem))
      return ltb_set_error(ctx, LTB_ESHAPE, "pga shard: tube too long for the fused transform");
    double* partials = nullptr;  // one slot set per CTA: the grid never exceeds the tile count
    LTB_TRY(ws.alloc(sizeof(double) * 5 * ((ntubes + p.TT - 1) / p.TT), &partials));
    StorePGA<R> st{(R*)d_xn, (const R*)d_xc, (const R*)d_xp, (const R*)d_gt, (R)beta};
    LoadPlain<Tc> ld{(const Tc*)d_hat, LTB_SLICE_MAJOR};
    const int dbl = std::is_same<R, double>::value ? 1 : 0;
    int64_t nb = 0;
    LTB_TRY((launch_xform_tile<Tc, Tc>(ctx, p, ld, st, (const Tc*)spec->d_mats[dbl][1], partials, d_state, smem, &nb)));
    pga_shard_sums_kernel<<<1, 160, 0, ctx->stream>>>(partials, nb, d_sums, d_state);
    LTB_LAUNCH_CHECK(ctx);
    return LTB_OK;
  };
  if (spec->is_complex)
    return dtype == LTB_F64 ? run(double(), cplx<double>()) : run(float(), cplx<float>());
  return dtype == LTB_F64 ? run(double(), double()) : run(float(), float());
}

int ltb_pga_shard_decide(ltb_ctx* ctx, const double* d_sums, double pobs_sumsq, double tol, double* d_rec,
                         int* d_state) {
  pga_shard_decide_kernel<<<1, 1, 0, ctx->stream>>>(d_sums, pobs_sumsq, tol, d_rec, d_state);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

}  // extern "C"
