// K3: batched one-sided (Hestenes) Jacobi SVD of transform-domain slices,
// the SVT fused recomposition and the full-matrices SVD for t_svd.
//
// Reference semantics:
//   svt   linalg.py:168-181  u, s, vh = svd(hat, full_matrices=False);
//                            out = (u * max(s - tau, 0)) @ vh
//   t_svd linalg.py:102-118  u, s, vh = svd(hat, full_matrices=True)
//   ranks / spectral_norm / nuclear_norm  linalg.py:132-165 (values only)
//
// B200 design (one CTA per slice, the slice resident in shared memory):
//   * the slice is loaded once, oriented so that it has n = min(I1, I2)
//     columns of length m = max(I1, I2) (A itself, or A^H), column-contiguous
//     with an odd pitch (bank-conflict-free strided fills);
//   * a round-robin (circle-method) ordering gives n/2 disjoint column pairs
//     per round; each warp takes pairs, reduces the 2x2 Gram entries with
//     warp shuffles, and applies the (complex-phased) Jacobi rotation in
//     place; one __syncthreads per round, sweeps until no pair exceeds
//     tol * sqrt(alpha * beta);
//   * the columns are then sorted by norm (descending, like LAPACK) and the
//     SVT is recomposed WITHOUT accumulating V:
//        out = sum_{sigma_j > tau} (sigma_j - tau) / sigma_j^2 * w_j (w_j^H A)
//     as two batched GEMMs whose inner dimension is limited per slice to the
//     number of surviving singular values (ltb_gemm.cu).
// Slices that do not fit in shared memory run the block-cyclic tier below
// (column blocks paired through shared memory, one launch per outer round).
#include <cfloat>

#include "ltb_dispatch.cuh"

namespace {

constexpr int kJacobiMaxThreads = 1024;

template <typename R> struct eps_of;
template <> struct eps_of<float> {
  static constexpr float value = FLT_EPSILON;
};
template <> struct eps_of<double> {
  static constexpr double value = DBL_EPSILON;
};

template <typename R> __device__ __forceinline__ R warp_sum_r(R v) { return warp_sum(v); }

// MUFU approximations (flush-to-zero) for the fp32 rotation parameters.  The
// rotation stays orthogonal to rounding whatever the accuracy of t (c = (1 +
// t^2)^-1/2 is refined by one Newton step, s = c t); t itself only decides how
// completely the pair's Gram entry is annihilated.  Pairs whose norms or Gram
// entry are below FLT_MIN are left alone (they cannot move an fp32 result).
__device__ __forceinline__ float sqrt_apx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_apx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_apx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// fp64 MUFU approximations (MUFU.RCP64H / RSQ64H, ~20-bit): Jacobi rotation parameters only
__device__ __forceinline__ double rcp_apx64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rsqrt_apx64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// two consecutive elements, one vector shared-memory access (LDS.64 / LDS.128)
template <typename T> struct alignas(2 * sizeof(T)) vec2 {
  T a, b;
};

struct JacobiOut {
  void* w_out;       // batch x n x m (column j contiguous, sorted) or null
  void* sv_out;      // batch x n real, descending, or null
  void* v_out;       // batch x n x n (column j contiguous, sorted) or null (WANT_V)
  int* kept_out;     // batch, number of sigma > tau, or null
  void* d_out;       // batch x n real: (sigma - tau)_+ / sigma^2 in sorted order, or null
  double tau;
  const int* skip;   // device flag: nonzero -> return immediately
  unsigned long long* stats;  // optional: [0] += slices, [1] += sweeps
  float tol_scale = 1.f;      // QR/Cholesky-preconditioned fp32 path: rotation threshold multiplier
  // QR/Cholesky path: stop after a sweep whose rotations all had |<w_p, w_q>| / (|w_p| |w_q|)
  // below this (0: stop only after a sweep without rotations)
  float early_stop = 0.f;
  // blocked tier: optional device flags (batch), 0 = the slice is known to have no singular
  // value above tau (||A||_F <= tau): it is not solved and reports kept = 0, sigma = 0
  const int* pre_active = nullptr;
  // blocked tier without WANT_V: optional batch x n x n array holding V^T (row j = the right
  // vector that belongs to working column j, in the Jacobi's own column order); every round
  // multiplies the rows of its block pair by the pair's accumulated rotations (V <- V J)
  void* v_acc = nullptr;
  int* rank_out = nullptr;  // blocked tier: optional batch x n, the sorted position of working column j
  // blocked tier, SVT of complex64 slices with sigma-sorted working columns (the carried path): only
  // block pairs that involve one of the slice's leading blocks are rotated; the untouched columns are
  // certified to have no singular value above tau (see block_certify), else the slice is finished
  // with full sweeps
  bool truncate = false;
  const int* lead = nullptr;  // (internal) batch: leading blocks of each slice
  float small2 = 0.f;         // (internal) pairs of two columns with squared norms <= small2 are left alone
};

template <typename T, bool WANT_V, bool GLOBAL, int TS, int MPL, int MINB>
__global__ void __launch_bounds__(MINB == 2 ? 576 : kJacobiMaxThreads, MINB)
    jacobi_kernel(int64_t I1, int64_t I2, const T* __restrict__ A, T* __restrict__ gws, JacobiOut o, int max_sweeps,
                  int mp) {
  using R = typename scalar_traits<T>::real;
  constexpr bool CPLX = scalar_traits<T>::is_complex;
  if (o.skip && *o.skip) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const bool trans = I1 < I2;
  const int m = (int)(trans ? I2 : I1);
  const int n = (int)(trans ? I1 : I2);
  const int np_v = n | 1;
  const int64_t b = blockIdx.x;
  const T* Ab = A + b * I1 * I2;

  T* W;
  T* V = nullptr;
  R* sig;
  int* flags;
  if constexpr (GLOBAL) {
    W = gws + b * ((int64_t)n * mp + (WANT_V ? (int64_t)n * np_v : 0));
    if (WANT_V) V = W + (int64_t)n * mp;
    sig = reinterpret_cast<R*>(smem_raw);
  } else {
    W = reinterpret_cast<T*>(smem_raw);
    if (WANT_V) V = W + (size_t)n * mp;
    sig = reinterpret_cast<R*>(W + (size_t)n * mp + (WANT_V ? (size_t)n * np_v : 0));
  }
  flags = reinterpret_cast<int*>(sig + n + 1);

  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;

  // ---- load the working columns
  if (!trans) {  // columns of A (strided in row-major storage)
    for (int l = tid; l < m * n; l += nth) {
      const int i = l / n, j = l - i * n;
      W[(size_t)j * mp + i] = Ab[l];
    }
  } else {  // columns of A^H = conjugated rows of A
    for (int l = tid; l < m * n; l += nth) {
      const int j = l / m, i = l - j * m;
      W[(size_t)j * mp + i] = conj_v(Ab[l]);
    }
  }
  if (mp > m) {  // zero padding rows: register tiles need no row predicates
    const int pad = mp - m;
    for (int l = tid; l < n * pad; l += nth) {
      const int j = l / pad, i = m + (l - j * pad);
      W[(size_t)j * mp + i] = zero_v<T>();
    }
  }
  if (WANT_V) {
    for (int l = tid; l < n * n; l += nth) {
      const int j = l / n, k = l - j * n;
      V[(size_t)j * np_v + k] = (j == k) ? cvt<T>((R)1) : zero_v<T>();
    }
  }
  if (tid < 2) flags[tid] = 0;
  __syncthreads();

  const R tol = eps_of<R>::value * sqrt((R)max(m, 1));
  const int npl = n + (n & 1);
  const int npairs = npl / 2;
  // teams of TS lanes each own one column pair per round (TPW teams per warp)
  constexpr int TPW = 32 / TS;
  const int tl = lane % TS;
  const int team = lane / TS;
  R* nrm = sig;  // squared column norms, exact at each sweep start, updated analytically
  int sweeps_done = 0;
  for (int sweep = 0; sweep < max_sweeps && n > 1; ++sweep) {
    int* rot = &flags[sweep & 1];
    for (int j = warp; j < n; j += nwarps) {
      const T* wj = W + (size_t)j * mp;
      R s2 = 0;
      for (int i = lane; i < m; i += 32) s2 += abs2_v(wj[i]);
      s2 = warp_sum_r(s2);
      if (lane == 0) nrm[j] = s2;
    }
    __syncthreads();
    if (sweep == 0 && o.tau > 0.0 && !o.sv_out && !o.v_out && !WANT_V) {
      // SVT-only call: sigma_max <= ||A||_F, so ||A||_F <= tau keeps nothing and the
      // output slice is exactly zero (the recomposition GEMMs see kept == 0)
      if (warp == 0) {
        R s = 0;
        for (int j = lane; j < n; j += 32) s += nrm[j];
        s = warp_sum_r(s);
        if (lane == 0) flags[3] = (s <= (R)o.tau * (R)o.tau) ? 1 : 0;
      }
      __syncthreads();
      if (flags[3]) {
        R* d_out = reinterpret_cast<R*>(o.d_out);
        if (d_out)
          for (int j = tid; j < n; j += nth) d_out[b * n + j] = (R)0;
        if (tid == 0) {
          if (o.kept_out) o.kept_out[b] = 0;
          if (o.stats) atomicAdd(&o.stats[0], 1ull);
        }
        return;
      }
    }
    for (int r = 0; r < npl - 1; ++r) {
      for (int base = warp * TPW; base < npairs; base += nwarps * TPW) {
        const int k = base + team;
        int p = 0, q = 0;
        if (k < npairs) {  // circle-method pairing without integer division
          const int m1 = npl - 1;
          if (k == 0) {
            p = m1;
            q = r;
          } else {
            p = r + k;
            p -= (p >= m1) ? m1 : 0;
            q = r - k;
            q += (q < 0) ? m1 : 0;
          }
        }
        const bool active = k < npairs && p < n && q < n;
        T* wp = W + (size_t)(active ? p : 0) * mp;
        T* wq = W + (size_t)(active ? q : 0) * mp;
        if constexpr (std::is_same<T, float>::value && MPL > 0) {
          // fp32: paired-lane FFMA2/FMUL2 on two rows at a time, MUFU rotation parameters
          float2 X[MPL / 2], Y[MPL / 2];
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int h = 0; h < MPL / 2; ++h) {
            const int i = 2 * tl + 2 * TS * h;
            X[h] = *reinterpret_cast<const float2*>(wp + i);
            Y[h] = *reinterpret_cast<const float2*>(wq + i);
            acc = __ffma2_rn(X[h], Y[h], acc);
          }
          float g = acc.x + acc.y;
#pragma unroll
          for (int o = TS / 2; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
          const float al = active ? nrm[p] : 0.f;
          const float be = active ? nrm[q] : 0.f;
          const float gabs = fabsf(g);
          if (!active || !(gabs > tol * sqrt_apx(al) * sqrt_apx(be)) || !(fminf(fminf(al, be), gabs) >= FLT_MIN)) continue;
          const float zeta = (be - al) * (0.5f * rcp_apx(gabs));
          const float az = fabsf(zeta);
          const float den = az < 1e18f ? az + sqrt_apx(fmaf(az, az, 1.f)) : 2.f * az;
          const float t = copysignf(rcp_apx(den), zeta);
          const float x1 = fmaf(t, t, 1.f);
          float c = rsqrt_apx(x1);
          c = c * fmaf(-0.5f * x1 * c, c, 1.5f);
          const float s = c * t;
          const float sg = g >= 0.f ? 1.f : -1.f;
          const float2 C2 = make_float2(c, c), S2 = make_float2(s, s);
          const float2 NSQ = make_float2(-s * sg, -s * sg), CQ = make_float2(c * sg, c * sg);
#pragma unroll
          for (int h = 0; h < MPL / 2; ++h) {
            const int i = 2 * tl + 2 * TS * h;
            *reinterpret_cast<float2*>(wp + i) = __ffma2_rn(C2, X[h], __fmul2_rn(NSQ, Y[h]));
            *reinterpret_cast<float2*>(wq + i) = __ffma2_rn(S2, X[h], __fmul2_rn(CQ, Y[h]));
          }
          if (WANT_V) {
            T* vp = V + (size_t)p * np_v;
            T* vq = V + (size_t)q * np_v;
            for (int i = tl; i < n; i += TS) {
              const float x = vp[i];
              const float y = sg * vq[i];
              vp[i] = c * x - s * y;
              vq[i] = s * x + c * y;
            }
          }
          if (tl == 0) {
            nrm[p] = fmaxf(al - t * gabs, 0.f);
            nrm[q] = be + t * gabs;
            *rot = 1;
          }
          continue;
        }
        T ga = zero_v<T>();
        T xr[MPL > 0 ? MPL : 1], yr[MPL > 0 ? MPL : 1];
        if constexpr (MPL > 0) {
          // two consecutive rows per vector access (rows >= m are zero padding)
#pragma unroll
          for (int e = 0; e < MPL; e += 2) {
            const int i = 2 * tl + TS * e;
            const vec2<T> vx = *reinterpret_cast<const vec2<T>*>(wp + i);
            const vec2<T> vy = *reinterpret_cast<const vec2<T>*>(wq + i);
            xr[e] = vx.a;
            xr[e + 1] = vx.b;
            yr[e] = vy.a;
            yr[e + 1] = vy.b;
            fma_acc(ga, conj_v(xr[e]), yr[e]);
            fma_acc(ga, conj_v(xr[e + 1]), yr[e + 1]);
          }
        } else {
          if (active)
            for (int i = tl; i < m; i += TS) fma_acc(ga, conj_v(wp[i]), wq[i]);
        }
        R gre = re_v(ga), gim = im_v(ga);
#pragma unroll
        for (int o = TS / 2; o > 0; o >>= 1) {
          gre += __shfl_xor_sync(0xffffffffu, gre, o);
          if (CPLX) gim += __shfl_xor_sync(0xffffffffu, gim, o);
        }
        const R al = active ? nrm[p] : (R)0;
        const R be = active ? nrm[q] : (R)0;
        const R gabs = CPLX ? hypot(gre, gim) : fabs(gre);
        // one square root for the test, and sqrt(1 + zeta^2) / rsqrt instead of hypot and a
        // division below |zeta| = 1e100 (the rotation chain is the latency of a round)
        constexpr bool DBL = sizeof(R) == 8;  // (fp32 keeps two roots: al * be may overflow)
        R sab, t, c;
        if constexpr (DBL) {
          // fp64: every lane of a team computes the parameters, so the IEEE sqrt / division
          // sequences (software, tens of DFMAs each) made the rotation chain FP64-throughput
          // bound.  The threshold test, zeta and t only need ~20 correct bits (an inexact t
          // leaves a ~1e-6 relative inner product for the next sweep; the rotation stays
          // orthogonal): MUFU approximations.  c = (1 + t^2)^-1/2 must be exact to fp64 for
          // orthogonality: MUFU rsqrt + three Newton steps.
          const double prod = al * be;
          sab = prod * rsqrt_apx64(prod);
          if (!active || !(gabs > tol * sab) || al == (R)0 || be == (R)0) continue;
          const double zeta = (be - al) * (0.5 * rcp_apx64(gabs));
          const double az = fabs(zeta);
          const double z1 = fma(az, az, 1.0);
          const double den = az < 1e18 ? az + z1 * rsqrt_apx64(z1) : 2.0 * az;
          t = copysign(rcp_apx64(den), zeta);
          const double x1 = fma(t, t, 1.0);
          double cc = rsqrt_apx64(x1);
#pragma unroll
          for (int it = 0; it < 3; ++it) cc = cc * fma(-0.5 * x1 * cc, cc, 1.5);
          c = cc;
        } else {
          sab = sqrt(al) * sqrt(be);
          if (!active || !(gabs > tol * sab) || al == (R)0 || be == (R)0) continue;
          const R zeta = (be - al) * ((R)0.5 / gabs);
          const R az = fabs(zeta);
          const R den = az < (R)1e18 ? az + sqrt(fma(az, az, (R)1)) : (R)2 * az;
          t = (zeta >= 0 ? (R)1 : (R)-1) / den;
          c = (R)1 / sqrt(fma(t, t, (R)1));
        }
        const R s = c * t;
        // phase e^{-i phi} applied to column q so the Gram entry becomes real
        T ph;
        if constexpr (CPLX) {
          ph = T{gre / gabs, -gim / gabs};
        } else {
          ph = (gre >= 0) ? (R)1 : (R)-1;
        }
        if constexpr (MPL > 0) {
          // real: fold the sign into the rotation; complex: phase the q column first
          R cq = c, sq = s;
          if constexpr (!CPLX) {
            cq = c * re_v(ph);
            sq = s * re_v(ph);
          }
#pragma unroll
          for (int e = 0; e < MPL; e += 2) {
            const int i = 2 * tl + TS * e;
            vec2<T> vx, vy;
            if constexpr (CPLX) {
              const T y0 = ph * yr[e], y1 = ph * yr[e + 1];
              vx.a = c * xr[e] - s * y0;
              vx.b = c * xr[e + 1] - s * y1;
              vy.a = s * xr[e] + c * y0;
              vy.b = s * xr[e + 1] + c * y1;
            } else {
              vx.a = c * xr[e] - sq * yr[e];
              vx.b = c * xr[e + 1] - sq * yr[e + 1];
              vy.a = s * xr[e] + cq * yr[e];
              vy.b = s * xr[e + 1] + cq * yr[e + 1];
            }
            *reinterpret_cast<vec2<T>*>(wp + i) = vx;
            *reinterpret_cast<vec2<T>*>(wq + i) = vy;
          }
        } else {
          for (int i = tl; i < m; i += TS) {
            const T x = wp[i];
            const T y = ph * wq[i];
            wp[i] = c * x - s * y;
            wq[i] = s * x + c * y;
          }
        }
        if (WANT_V) {
          T* vp = V + (size_t)p * np_v;
          T* vq = V + (size_t)q * np_v;
          for (int i = tl; i < n; i += TS) {
            const T x = vp[i];
            const T y = ph * vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
        }
        if (tl == 0) {
          // alpha' = alpha - t|gamma|, beta' = beta + t|gamma| for the rotation that zeroes gamma
          nrm[p] = fmax(al - t * gabs, (R)0);
          nrm[q] = be + t * gabs;
          // bit 0: the sweep rotated; bit 1: a rotation with |gamma| / sqrt(alpha beta) >= early_stop
          atomicOr(rot, (o.early_stop > 0.f && gabs >= (R)o.early_stop * sab) ? 3 : 1);
        }
      }
      __syncthreads();
    }
    const int any = *rot;
    __syncthreads();
    if (tid == 0) flags[(sweep + 1) & 1] = 0;
    __syncthreads();
    sweeps_done = sweep + 1;
    // without rotations the sweep changed nothing; with early_stop (the warm fp64 PGA SVT:
    // sqrt(tol)), a sweep whose rotations all had relative inner products below it leaves
    // inner products of order tol behind (quadratic convergence), as in jacobi_qr_kernel
    if (!(any & 1) || (o.early_stop > 0.f && !(any & 2))) break;
  }
  if (o.stats && tid == 0) {
    atomicAdd(&o.stats[0], 1ull);
    atomicAdd(&o.stats[1], (unsigned long long)sweeps_done);
  }

  // ---- singular values = column norms
  for (int j = warp; j < n; j += nwarps) {
    const T* wj = W + (size_t)j * mp;
    R s2 = 0;
    for (int i = lane; i < m; i += 32) s2 += abs2_v(wj[i]);
    s2 = warp_sum_r(s2);
    if (lane == 0) sig[j] = sqrt(s2);
  }
  __syncthreads();

  // ---- sort (descending, stable) and emit
  R* sv_out = reinterpret_cast<R*>(o.sv_out);
  R* d_out = reinterpret_cast<R*>(o.d_out);
  int* rank_sh = flags + 4;
  if (tid == 0) flags[2] = 0;
  __syncthreads();
  int kept_local = 0;
  for (int j = tid; j < n; j += nth) {
    const R sj = sig[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const R si = sig[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    rank_sh[j] = rank;
    if (sv_out) sv_out[b * n + rank] = sj;
    const bool keep = sj > (R)o.tau && sj > (R)0;
    kept_local += keep;
    // u_j u_j^H A / sigma_j scaled by (sigma_j - tau): w_j (w_j^H A) (sigma_j - tau) / sigma_j^3
    if (d_out) d_out[b * n + rank] = keep ? (((sj - (R)o.tau) / sj) / sj) / sj : (R)0;
  }
  if (kept_local) atomicAdd(&flags[2], kept_local);
  __syncthreads();
  if (o.kept_out && tid == 0) o.kept_out[b] = flags[2];
  if (o.w_out) {
    T* dst = reinterpret_cast<T*>(o.w_out) + b * (int64_t)n * m;
    for (int l = tid; l < n * m; l += nth) {
      const int j = l / m, i = l - j * m;
      dst[(int64_t)rank_sh[j] * m + i] = W[(size_t)j * mp + i];
    }
  }
  if (WANT_V && o.v_out) {
    T* dst = reinterpret_cast<T*>(o.v_out) + b * (int64_t)n * n;
    for (int l = tid; l < n * n; l += nth) {
      const int j = l / n, i = l - j * n;
      dst[(int64_t)rank_sh[j] * n + i] = V[(size_t)j * np_v + i];
    }
  }
}

// ---------------------------------------------------------------- t_svd helpers
// U (m x m, row-major output with leading dim m) from the sorted working
// columns: u_j = w_j / sigma_j where sigma_j is numerically nonzero, and a
// deterministic Gram-Schmidt completion for the remaining columns
// (rank-deficient slices, and the m - n extra columns of full_matrices=True).
// The completion candidate for each new column is the unit vector e_i whose
// residual (1 - |row i of the columns so far|^2) is largest: that residual
// is >= (m - slot) / m, so every candidate is accepted (no rejection loop).
template <typename T>
__global__ void complete_u_kernel(int m, int n, const T* __restrict__ w_sorted,
                                  const typename scalar_traits<T>::real* __restrict__ sv, T* __restrict__ U,
                                  int any_nonzero = 0) {
  using R = typename scalar_traits<T>::real;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  R* rn = reinterpret_cast<R*>(smem_raw);  // residual row norms, m entries
  const int64_t b = blockIdx.x;
  const T* Wb = w_sorted + b * (int64_t)n * m;
  const R* sb = sv + b * (int64_t)n;
  T* Ub = U + b * (int64_t)m * m;  // Ub[i * m + j] = column j, row i
  __shared__ R red[32];
  __shared__ int redi[32];
  __shared__ T redc[32];
  __shared__ int good_count;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  const R smax = n > 0 ? sb[0] : (R)0;
  // t_svd: columns above the rank threshold of numpy's matrix_rank; any_nonzero (the carried
  // PGA basis): every column with sigma > 0, since converged Jacobi columns are orthogonal
  // relative to their own norms and only an orthonormal basis is needed there
  const R thr = any_nonzero ? (R)0 : smax * (R)max(m, 1) * eps_of<R>::value;
  // number of leading good columns (sorted descending, so good ones are a prefix)
  if (tid == 0) {
    int g = 0;
    while (g < n && sb[g] > thr && sb[g] > (R)0) ++g;
    good_count = g;
  }
  __syncthreads();
  const int g0 = good_count;
  for (int j = tid; j < g0; j += nth) rn[j] = (R)1 / sb[j];
  __syncthreads();
  // row-major output, the column index fastest: coalesced stores; the column-major reads
  // revisit each 32-byte sector for 8 consecutive rows and stay in L1 (a 32 x 32 shared-
  // memory tile transpose measured slower: 25 tiles and 50 barriers per slice)
  for (int l = tid; l < m * g0; l += nth) {
    const int i = l / g0, j = l - i * g0;
    Ub[(int64_t)i * m + j] = Wb[(int64_t)j * m + i] * rn[j];
  }
  __syncthreads();
  if (g0 >= m) return;  // every column normalised: nothing to complete
  for (int i = tid; i < m; i += nth) {
    R acc = 0;
    for (int j = 0; j < g0; ++j) acc += abs2_v(Ub[(int64_t)i * m + j]);
    rn[i] = (R)1 - acc;
  }
  __syncthreads();
  auto block_sum_r = [&](R v) -> R {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    R s = 0;
    for (int k = 0; k < nw; ++k) s += red[k];
    return s;
  };
  auto block_sum_t = [&](T v) -> T {
    R a = warp_sum(re_v(v));
    R c = scalar_traits<T>::is_complex ? warp_sum(im_v(v)) : (R)0;
    __syncthreads();
    if (lane == 0) {
      if constexpr (scalar_traits<T>::is_complex) {
        redc[warp] = T{a, c};
      } else {
        redc[warp] = a;
      }
    }
    __syncthreads();
    T s = zero_v<T>();
    for (int k = 0; k < nw; ++k) s = s + redc[k];
    return s;
  };
  for (int slot = g0; slot < m; ++slot) {
    // pivot: the row with the largest residual (lowest index on ties)
    R best = -(R)1;
    int bi = m;
    for (int i = tid; i < m; i += nth)
      if (rn[i] > best) {
        best = rn[i];
        bi = i;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const R ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    __syncthreads();
    if (lane == 0) {
      red[warp] = best;
      redi[warp] = bi;
    }
    __syncthreads();
    int cand = redi[0];
    R cb = red[0];
    for (int k = 1; k < nw; ++k)
      if (red[k] > cb || (red[k] == cb && redi[k] < cand)) {
        cb = red[k];
        cand = redi[k];
      }
    for (int i = tid; i < m; i += nth) Ub[(int64_t)i * m + slot] = (i == cand) ? cvt<T>((R)1) : zero_v<T>();
    __syncthreads();
    for (int pass = 0; pass < 2; ++pass) {
      for (int g = 0; g < slot; ++g) {
        T part = zero_v<T>();
        for (int i = tid; i < m; i += nth) fma_acc(part, conj_v(Ub[(int64_t)i * m + g]), Ub[(int64_t)i * m + slot]);
        const T coef = block_sum_t(part);
        for (int i = tid; i < m; i += nth) Ub[(int64_t)i * m + slot] = Ub[(int64_t)i * m + slot] - coef * Ub[(int64_t)i * m + g];
        __syncthreads();
      }
    }
    R part = 0;
    for (int i = tid; i < m; i += nth) part += abs2_v(Ub[(int64_t)i * m + slot]);
    const R inv = (R)1 / sqrt(block_sum_r(part));
    for (int i = tid; i < m; i += nth) {
      const T u = Ub[(int64_t)i * m + slot] * inv;
      Ub[(int64_t)i * m + slot] = u;
      rn[i] -= abs2_v(u);
    }
    __syncthreads();
  }
}

// dst (row-major n x n, leading dim n): dst[i * n + j] = col_j[i], col-contiguous src
template <typename T>
__global__ void cols_to_rowmajor_kernel(int64_t batch, int n, const T* __restrict__ src, T* __restrict__ dst) {
  const int64_t total = batch * (int64_t)n * n;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = l / ((int64_t)n * n);
    const int64_t r = l - b * n * n;
    const int i = (int)(r / n), j = (int)(r - (int64_t)(r / n) * n);
    dst[l] = src[b * n * n + (int64_t)j * n + i];
  }
}

template <typename T>
size_t jacobi_smem_bytes(int m, int n, bool want_v, int mp_) {
  using R = typename scalar_traits<T>::real;
  const size_t mp = (size_t)mp_, np_v = (size_t)(n | 1);
  return ((size_t)n * mp + (want_v ? (size_t)n * np_v : 0)) * sizeof(T) + (n + 1) * sizeof(R) + (n + 8) * sizeof(int) + 16;
}

constexpr size_t kSmemLimit = 225 * 1024;

// one shared-memory variant: TS lanes per column pair, MPL rows per lane (0 =
// looped), MINB CTAs per SM (2 -> at most 576 threads and 56 registers)
template <typename T, bool WANT_V, int TS, int MPL, int MINB>
int launch_smem_variant(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const T* A, const JacobiOut& o,
                        int max_sweeps, int m, int n) {
  const int mp = MPL > 0 ? TS * MPL : (m | 1);
  const size_t smem = jacobi_smem_bytes<T>(m, n, WANT_V, mp);
  const int pairs = std::max(1, (n + 1) / 2);
  const int maxw = MINB == 2 ? 18 : 32;
  const int teams = std::max(1, (pairs * TS + 31) / 32);  // warps for one pair per team
  const int per_warp = (teams + maxw - 1) / maxw;
  const int nwarps = std::max(1, (teams + per_warp - 1) / per_warp);
  auto kern = jacobi_kernel<T, WANT_V, false, TS, MPL, MINB>;
  LTB_TRY(ensure_smem(ctx, kern, smem, true));
  kern<<<(unsigned)batch, 32 * nwarps, smem, ctx->stream>>>(I1, I2, A, nullptr, o, max_sweeps, mp);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

template <typename T, bool WANT_V, int TS, int MPL>
int launch_smem(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const T* A, const JacobiOut& o, int max_sweeps,
                int m, int n) {
  const int mp = MPL > 0 ? TS * MPL : (m | 1);
  // two CTAs per SM when two slices fit in shared memory (228 KB per SM, 1 KB reserved per CTA)
  if (2 * (jacobi_smem_bytes<T>(m, n, WANT_V, mp) + 1024) <= 228 * 1024)
    return launch_smem_variant<T, WANT_V, TS, MPL, 2>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  return launch_smem_variant<T, WANT_V, TS, MPL, 1>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
}

// ---------------------------------------------------------------- blocked tier
// Slices whose working columns do not fit in shared memory (config 4's
// 1024 x 1024 complex slices, config 5 at n >= 256) run a block-cyclic
// one-sided Jacobi: the n columns are cut into nb blocks of b; each outer
// round pairs the blocks by the circle method and one CTA per block pair
// loads its 2b columns into shared memory, orthogonalises every cross pair
// (on the first round of a sweep also the pairs inside the two blocks) with
// the same rotation as the resident kernel, and writes the columns back.
// A sweep is nb - 1 rounds (every column pair met at least once); a slice is
// converged after a sweep without rotations.  For t_svd, V rides along as n
// extra rows of every working column (rotated, never dotted).
struct BlockGeom {
  int m, n, mp, b, nb;
};

constexpr size_t kBlockSmem = 200 * 1024;
// early-stop scale (x sqrt(tol)) of the fp32 Jacobi for calls that do not set their own
// (QR path, blocked-tier svt / values; 0: run to a sweep without rotations)
constexpr float g_qr_early = 1.f;

__global__ void fill_int_kernel(int64_t n, int* __restrict__ p, int v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

template <typename T, bool WANT_V>
__global__ void block_load_kernel(int64_t I1, int64_t I2, const T* __restrict__ A, T* __restrict__ W, BlockGeom g) {
  using R = typename scalar_traits<T>::real;
  const int64_t s = blockIdx.y;
  const bool trans = I1 < I2;
  const T* Ab = A + s * I1 * I2;
  T* Ws = W + s * (int64_t)g.n * g.mp;
  const int64_t total = (int64_t)g.n * g.mp;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(l / g.mp), i = (int)(l - (int64_t)j * g.mp);
    T v = zero_v<T>();
    if (i < g.m) {
      v = trans ? conj_v(Ab[(int64_t)j * g.m + i]) : Ab[(int64_t)i * g.n + j];
    } else if (WANT_V && i < g.m + g.n && i - g.m == j) {
      v = cvt<T>((R)1);
    }
    Ws[l] = v;
  }
}

// rotation accumulation (JacobiOut::v_acc): blocks of at most ACCB / 2 columns (the 2b values of a
// V^T element index live in one thread's registers): 24 for complex64 / fp64, 32 for fp32
constexpr int kLeadMax = 8;  // truncated sweeps: most leading blocks of a slice (more: full sweeps)
template <typename T> struct acc_dim { static constexpr int value = 0; };
template <> struct acc_dim<cplx<float>> { static constexpr int value = 24; };
template <> struct acc_dim<float> { static constexpr int value = 32; };
template <> struct acc_dim<double> { static constexpr int value = 24; };
template <typename T> __host__ __device__ inline size_t block_acc_offset(int b, int mp) {
  using R = typename scalar_traits<T>::real;
  const size_t base = (size_t)2 * b * mp * sizeof(T) + (size_t)2 * b * sizeof(R) + 2 * sizeof(int);
  return (base + 15) / 16 * 16;
}

__device__ __forceinline__ bool jacobi_pair_params(float g, float al, float be, float tol, float& c, float& sn,
                                                   float& sg, float& tt, float& gabs, float& rel);

// Register-tile variants of complex64 keep the working columns PAIR-PLANAR in shared memory: every
// 16-byte group (two consecutive rows) holds (re0, re1, im0, im1) instead of (re0, im0, re1, im1),
// so that a lane's 16-byte access yields the packed operands (re0, re1) and (im0, im1) of
// FFMA2 / FMUL2 directly (the copies from and to global memory swap the two middle words).
template <typename T, int MPL> struct block_pair_planar {
  static constexpr bool value = MPL > 0 && std::is_same<T, cplx<float>>::value;
};
// two consecutive rows of a column as two elements, whatever the layout
template <bool PLANAR, typename T> __device__ __forceinline__ void ld_rows2(const T* p, T& a, T& b) {
  if constexpr (PLANAR) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    a = T{q.x, q.z};
    b = T{q.y, q.w};
  } else {
    const vec2<T> v = *reinterpret_cast<const vec2<T>*>(p);
    a = v.a;
    b = v.b;
  }
}
template <bool PLANAR, typename T> __device__ __forceinline__ void st_rows2(T* p, T a, T b) {
  if constexpr (PLANAR) {
    *reinterpret_cast<float4*>(p) = make_float4(a.re, b.re, a.im, b.im);
  } else {
    vec2<T> v;
    v.a = a;
    v.b = b;
    *reinterpret_cast<vec2<T>*>(p) = v;
  }
}

// MPL > 0: each lane holds rows lane + 32 e (e < MPL) of the pair in registers
// between the dot product and the rotation (mp == 32 MPL); MPL == 0 loops.
template <typename T, bool WANT_V, int MPL, int NTMAX, int ACCB = 0>
__global__ void __launch_bounds__(NTMAX, 1)
    jacobi_block_kernel(BlockGeom g, int round, int full, T* __restrict__ W, int* __restrict__ rot,
                        const int* __restrict__ active, const int* __restrict__ skip, unsigned* __restrict__ relmax,
                        T* __restrict__ Vacc, const int* __restrict__ lead, float small2, int compact) {
  using R = typename scalar_traits<T>::real;
  constexpr bool CPLX = scalar_traits<T>::is_complex;
  if (skip && *skip) return;
  const int64_t s = blockIdx.y;
  if (!active[s]) return;
  // block pair of this round (circle method over an even number of block slots)
  const int nbp = g.nb + (g.nb & 1), m1 = nbp - 1;
  const int k = blockIdx.x;
  int P, Q;
  if (compact) {
    // truncated sweeps, compacted grid: CTA i takes leading block i and its partner of this round
    // (the circle method pairs block m1 with `round` and blocks whose indices sum to 2 round mod m1);
    // a pair of two leading blocks is taken by the lower one; slices whose every block leads wait
    // for the full sweeps
    const int kl = lead[s];
    if (kl >= g.nb || k >= kl) return;
    P = k;
    Q = (k == round) ? m1 : (2 * round - k + 2 * m1) % m1;
    if (Q == P) Q = m1;  // (2 round = 2 k mod m1 with k != round cannot happen for odd m1; guard anyway)
    if (Q < kl && Q < P) return;
  } else if (k == 0) {
    P = m1;
    Q = round;
  } else {
    P = (round + k) % m1;
    Q = (round - k + m1) % m1;
  }
  // with an odd block count one block per round meets the empty slot: it still
  // needs its internal pairs on the first round of the sweep
  const bool pv = P < g.nb, qv = Q < g.nb;
  if (!(pv && qv) && !(full && (pv || qv))) return;
  if (lead) {  // truncated sweeps: pairs of two trailing blocks are left alone
    const int kl = lead[s];
    if ((!pv || P >= kl) && (!qv || Q >= kl)) return;
  }
  const int b = g.b, mp = g.mp, m = g.m;
  const int cp0 = P * b, cq0 = Q * b;
  const int np_ = pv ? min(b, g.n - cp0) : 0, nq_ = qv ? min(b, g.n - cq0) : 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* C = reinterpret_cast<T*>(smem_raw);
  R* nrm = reinterpret_cast<R*>(C + (size_t)2 * b * mp);
  int* flag = reinterpret_cast<int*>(nrm + 2 * b);
  unsigned* fmax_sh = reinterpret_cast<unsigned*>(flag + 1);  // largest relative rotated |gamma| (float bits)
  // Vacc: the rotations of this block pair accumulated as an ACCB x ACCB matrix (2b <= ACCB)
  constexpr bool ACC = ACCB > 0;
  constexpr int kAccB = ACCB > 0 ? ACCB : 1;
  T* Jb = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(C) + block_acc_offset<T>(b, mp));
  T* Ws = W + s * (int64_t)g.n * mp;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  auto gcol = [&](int l) { return l < b ? cp0 + l : cq0 + (l - b); };
  auto valid = [&](int l) { return l < b ? l < np_ : (l - b) < nq_; };
  const int vpc = (int)(mp * sizeof(T) / 16);  // 16-byte vectors per column
  constexpr bool PLANAR = block_pair_planar<T, MPL>::value;
  for (int l = warp; l < 2 * b; l += nwarps) {
    if (!valid(l)) continue;
    const int4* src = reinterpret_cast<const int4*>(Ws + (int64_t)gcol(l) * mp);
    int4* dst = reinterpret_cast<int4*>(C + (size_t)l * mp);
    for (int v = lane; v < vpc; v += 32) {
      const int4 t = src[v];
      dst[v] = PLANAR ? make_int4(t.x, t.z, t.y, t.w) : t;
    }
  }
  if (tid == 0) {
    *flag = 0;
    *fmax_sh = 0u;
  }
  if constexpr (ACC)
    for (int l = tid; l < kAccB * kAccB; l += nth) Jb[l] = cvt<T>((R)((l / kAccB == l % kAccB) ? 1 : 0));
  __syncthreads();
  const int m_even = min(mp, (m + 1) & ~1);  // (the pair-planar groups pair row m - 1 with a zero padding row)
  for (int l = warp; l < 2 * b; l += nwarps) {
    R s2 = 0;
    if (valid(l)) {
      const T* c = C + (size_t)l * mp;
      for (int i = lane; i < (PLANAR ? m_even : m); i += 32) s2 += abs2_v(c[i]);
    }
    s2 = warp_sum_r(s2);
    if (lane == 0) nrm[l] = s2;
  }
  __syncthreads();
  const R tol = eps_of<R>::value * sqrt((R)max(m, 1));
  const int rows = WANT_V ? m + g.n : m;  // rotated rows (padding rows stay zero)
  const int nrounds = full ? 2 * b - 1 : b;
  bool rounds_done = false;
  if constexpr (MPL > 0) {
    // cross rounds with one warp per column of block P: the warp's own column stays in
    // registers over all b inner rounds (only the columns of Q travel through shared memory,
    // half the shared-memory traffic per rotation)
    if (!full && nwarps == b) {
      const int p = warp;
      const bool pvld = valid(p);
      T* x = C + (size_t)p * mp;
      bool xdirty = false;
      if constexpr (std::is_same<R, float>::value) {
        // fp32 / complex64: packed FFMA2 / FMUL2 on two rows at a time (complex64: the pair-planar
        // layout gives (re0, re1) and (im0, im1) per 16-byte access), MUFU rotation parameters
        constexpr int H = MPL / 2;
        float2 XA[H], XB[CPLX ? H : 1];  // real: XA = rows; complex: XA = re pairs, XB = im pairs
        if (pvld) {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            if constexpr (CPLX) {
              const float4 q = *reinterpret_cast<const float4*>(x + 2 * lane + 64 * h);
              XA[h] = make_float2(q.x, q.y);
              XB[h] = make_float2(q.z, q.w);
            } else {
              XA[h] = *reinterpret_cast<const float2*>(x + 2 * lane + 64 * h);
            }
          }
        }
        for (int r = 0; r < b; ++r) {
          const int q = b + (p + r) % b;
          if (pvld && valid(q)) {
            T* y = C + (size_t)q * mp;
            float2 YA[H], YB[CPLX ? H : 1];
            float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
#pragma unroll
            for (int h = 0; h < H; ++h) {
              if constexpr (CPLX) {
                const float4 v = *reinterpret_cast<const float4*>(y + 2 * lane + 64 * h);
                YA[h] = make_float2(v.x, v.y);
                YB[h] = make_float2(v.z, v.w);
                a0 = __ffma2_rn(XA[h], YA[h], a0);  // xr yr
                a1 = __ffma2_rn(XB[h], YB[h], a1);  // xi yi
                a2 = __ffma2_rn(XA[h], YB[h], a2);  // xr yi
                a3 = __ffma2_rn(XB[h], YA[h], a3);  // xi yr
              } else {
                YA[h] = *reinterpret_cast<const float2*>(y + 2 * lane + 64 * h);
                if (h & 1) a1 = __ffma2_rn(XA[h], YA[h], a1);
                else a0 = __ffma2_rn(XA[h], YA[h], a0);
              }
            }
            float gre, gim = 0.f;
            if constexpr (CPLX) {
              gre = warp_sum_r((a0.x + a0.y) + (a1.x + a1.y));
              gim = warp_sum_r((a2.x + a2.y) - (a3.x + a3.y));
            } else {
              gre = warp_sum_r((a0.x + a0.y) + (a1.x + a1.y));
            }
            const float al = nrm[p], be = nrm[q];
            float gsig = gre, pr = 1.f, pi = 0.f;
            if constexpr (CPLX) {
              // |g| and the unit phase conj(g) / |g|: scaled by the larger component first (g^2 of a
              // tiny inner product underflows: a flushed rsqrt input gave an infinite |g| and a
              // rotation by NaN), one Newton step on the MUFU rsqrt so that |ph| = 1 to rounding
              const float smax = fmaxf(fabsf(gre), fabsf(gim));
              const bool tiny = !(smax >= FLT_MIN);
              const float k = rcp_apx(tiny ? 1.f : smax);
              const float gr = gre * k, gi = gim * k;
              const float g2 = fmaf(gr, gr, gi * gi);  // in [1, 2]
              float rinv = rsqrt_apx(g2);
              rinv = rinv * fmaf(-0.5f * g2 * rinv, rinv, 1.5f);
              gsig = tiny ? 0.f : smax * (g2 * rinv);
              pr = gr * rinv;
              pi = -gi * rinv;
            }
            float c, sn, sg, tt, gabs, rel;
            if (!(al <= small2 && be <= small2) && jacobi_pair_params(gsig, al, be, tol, c, sn, sg, tt, gabs, rel)) {
              if constexpr (CPLX) {
                // x' = c x + a y, y' = sn x + bb y with a = -sn ph, bb = c ph
                const float ar = -sn * pr, ai = -sn * pi, br = c * pr, bi = c * pi;
                const float2 C2 = make_float2(c, c), S2 = make_float2(sn, sn);
                const float2 AR = make_float2(ar, ar), AI = make_float2(ai, ai), NAI = make_float2(-ai, -ai);
                const float2 BR = make_float2(br, br), BI = make_float2(bi, bi), NBI = make_float2(-bi, -bi);
#pragma unroll
                for (int h = 0; h < H; ++h) {
                  const float2 yr2 = __ffma2_rn(NBI, YB[h], __ffma2_rn(BR, YA[h], __fmul2_rn(S2, XA[h])));
                  const float2 yi2 = __ffma2_rn(BI, YA[h], __ffma2_rn(BR, YB[h], __fmul2_rn(S2, XB[h])));
                  const float2 xr2 = __ffma2_rn(NAI, YB[h], __ffma2_rn(AR, YA[h], __fmul2_rn(C2, XA[h])));
                  const float2 xi2 = __ffma2_rn(AI, YA[h], __ffma2_rn(AR, YB[h], __fmul2_rn(C2, XB[h])));
                  XA[h] = xr2;
                  XB[h] = xi2;
                  *reinterpret_cast<float4*>(y + 2 * lane + 64 * h) = make_float4(yr2.x, yr2.y, yi2.x, yi2.y);
                }
              } else {
                const float2 C2 = make_float2(c, c), S2 = make_float2(sn, sn);
                const float2 NSQ = make_float2(-sn * sg, -sn * sg), CQ = make_float2(c * sg, c * sg);
#pragma unroll
                for (int h = 0; h < H; ++h) {
                  const float2 yn = __ffma2_rn(S2, XA[h], __fmul2_rn(CQ, YA[h]));
                  XA[h] = __ffma2_rn(C2, XA[h], __fmul2_rn(NSQ, YA[h]));
                  *reinterpret_cast<float2*>(y + 2 * lane + 64 * h) = yn;
                }
              }
              xdirty = true;
              if (ACC && lane < kAccB) {
                T ph;
                if constexpr (CPLX) ph = T{pr, pi};
                else ph = sg;
                const T jp = Jb[lane * kAccB + p];
                const T jq = ph * Jb[lane * kAccB + q];
                Jb[lane * kAccB + p] = c * jp - sn * jq;
                Jb[lane * kAccB + q] = sn * jp + c * jq;
              }
              if (lane == 0) {
                nrm[p] = fmaxf(al - tt * gabs, 0.f);
                nrm[q] = be + tt * gabs;
                *flag = 1;
                if (relmax) atomicMax(fmax_sh, __float_as_uint(rel));
              }
            }
          }
          __syncthreads();
        }
        if (xdirty) {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            if constexpr (CPLX)
              *reinterpret_cast<float4*>(x + 2 * lane + 64 * h) = make_float4(XA[h].x, XA[h].y, XB[h].x, XB[h].y);
            else
              *reinterpret_cast<float2*>(x + 2 * lane + 64 * h) = XA[h];
          }
        }
      } else {
        T xr[MPL];
        if (pvld) {
#pragma unroll
          for (int e = 0; e < MPL; e += 2) ld_rows2<PLANAR>(x + 2 * lane + 32 * e, xr[e], xr[e + 1]);
        }
        for (int r = 0; r < b; ++r) {
          const int q = b + (p + r) % b;
          if (pvld && valid(q)) {
            T* y = C + (size_t)q * mp;
            T yr[MPL];
            T ga = zero_v<T>();
#pragma unroll
            for (int e = 0; e < MPL; e += 2) {
              ld_rows2<PLANAR>(y + 2 * lane + 32 * e, yr[e], yr[e + 1]);
              fma_acc(ga, conj_v(xr[e]), yr[e]);
              fma_acc(ga, conj_v(xr[e + 1]), yr[e + 1]);
            }
            const R gre = warp_sum_r(re_v(ga));
            const R gim = CPLX ? warp_sum_r(im_v(ga)) : (R)0;
            const R al = nrm[p], be = nrm[q];
            const R gabs = CPLX ? hypot(gre, gim) : fabs(gre);
            if (gabs > tol * sqrt(al) * sqrt(be) && al != (R)0 && be != (R)0 &&
                !((float)al <= small2 && (float)be <= small2)) {
              const R zeta = (be - al) / (2 * gabs);
              const R t = (zeta >= 0 ? (R)1 : (R)-1) / (fabs(zeta) + hypot((R)1, zeta));
              const R c = (R)1 / sqrt((R)1 + t * t);
              const R sn = c * t;
              T ph;
              if constexpr (CPLX) {
                ph = T{gre / gabs, -gim / gabs};
              } else {
                ph = (gre >= 0) ? (R)1 : (R)-1;
              }
#pragma unroll
              for (int e = 0; e < MPL; e += 2) {
                const T y0 = ph * yr[e], y1 = ph * yr[e + 1];
                st_rows2<PLANAR>(y + 2 * lane + 32 * e, sn * xr[e] + c * y0, sn * xr[e + 1] + c * y1);
                xr[e] = c * xr[e] - sn * y0;
                xr[e + 1] = c * xr[e + 1] - sn * y1;
              }
              xdirty = true;
              if (ACC && lane < kAccB) {
                const T jp = Jb[lane * kAccB + p];
                const T jq = ph * Jb[lane * kAccB + q];
                Jb[lane * kAccB + p] = c * jp - sn * jq;
                Jb[lane * kAccB + q] = sn * jp + c * jq;
              }
              if (lane == 0) {
                nrm[p] = fmax(al - t * gabs, (R)0);
                nrm[q] = be + t * gabs;
                *flag = 1;
                if (relmax) atomicMax(fmax_sh, __float_as_uint((float)(gabs / (sqrt(al) * sqrt(be)))));
              }
            }
          }
          __syncthreads();
        }
        if (xdirty) {
#pragma unroll
          for (int e = 0; e < MPL; e += 2) st_rows2<PLANAR>(x + 2 * lane + 32 * e, xr[e], xr[e + 1]);
        }
      }
      __syncthreads();
      rounds_done = true;
    }
  }
  for (int r = 0; r < nrounds && !rounds_done; ++r) {
    for (int pi = warp; pi < b; pi += nwarps) {
      int p, q;
      if (full) {  // every pair of the 2b columns: circle method over 2b slots
        const int mm = 2 * b - 1;
        if (pi == 0) {
          p = mm;
          q = r;
        } else {
          p = (r + pi) % mm;
          q = (r - pi + mm) % mm;
        }
      } else {  // cross pairs only: column pi of block P with column (pi + r) mod b of block Q
        p = pi;
        q = b + (pi + r) % b;
      }
      if (!valid(p) || !valid(q)) continue;
      T* x = C + (size_t)p * mp;
      T* y = C + (size_t)q * mp;
      T ga = zero_v<T>();
      T xr[MPL > 0 ? MPL : 1], yr[MPL > 0 ? MPL : 1];
      if constexpr (MPL > 0) {  // rows past m are zero padding; two consecutive rows per vector access
#pragma unroll
        for (int e = 0; e < MPL; e += 2) {
          const int i = 2 * lane + 32 * e;
          ld_rows2<PLANAR>(x + i, xr[e], xr[e + 1]);
          ld_rows2<PLANAR>(y + i, yr[e], yr[e + 1]);
          fma_acc(ga, conj_v(xr[e]), yr[e]);
          fma_acc(ga, conj_v(xr[e + 1]), yr[e + 1]);
        }
      } else {
        for (int i = lane; i < m; i += 32) fma_acc(ga, conj_v(x[i]), y[i]);
      }
      R gre = warp_sum_r(re_v(ga));
      R gim = CPLX ? warp_sum_r(im_v(ga)) : (R)0;
      const R al = nrm[p], be = nrm[q];
      const R gabs = CPLX ? hypot(gre, gim) : fabs(gre);
      if (!(gabs > tol * sqrt(al) * sqrt(be)) || al == (R)0 || be == (R)0) continue;
      if ((float)al <= small2 && (float)be <= small2) continue;  // truncated sweeps: two small columns
      const R zeta = (be - al) / (2 * gabs);
      const R t = (zeta >= 0 ? (R)1 : (R)-1) / (fabs(zeta) + hypot((R)1, zeta));
      const R c = (R)1 / sqrt((R)1 + t * t);
      const R sn = c * t;
      T ph;
      if constexpr (CPLX) {
        ph = T{gre / gabs, -gim / gabs};
      } else {
        ph = (gre >= 0) ? (R)1 : (R)-1;
      }
      if constexpr (MPL > 0) {
#pragma unroll
        for (int e = 0; e < MPL; e += 2) {
          const int i = 2 * lane + 32 * e;
          const T y0 = ph * yr[e], y1 = ph * yr[e + 1];
          st_rows2<PLANAR>(x + i, c * xr[e] - sn * y0, c * xr[e + 1] - sn * y1);
          st_rows2<PLANAR>(y + i, sn * xr[e] + c * y0, sn * xr[e + 1] + c * y1);
        }
      } else {
        for (int i = lane; i < rows; i += 32) {
          const T xv = x[i];
          const T yv = ph * y[i];
          x[i] = c * xv - sn * yv;
          y[i] = sn * xv + c * yv;
        }
      }
      if (ACC && lane < kAccB) {  // the same rotation on columns p, q of the accumulated J (row `lane`)
        const T jp = Jb[lane * kAccB + p];
        const T jq = ph * Jb[lane * kAccB + q];
        Jb[lane * kAccB + p] = c * jp - sn * jq;
        Jb[lane * kAccB + q] = sn * jp + c * jq;
      }
      if (lane == 0) {
        nrm[p] = fmax(al - t * gabs, (R)0);
        nrm[q] = be + t * gabs;
        *flag = 1;
        if (relmax) atomicMax(fmax_sh, __float_as_uint((float)(gabs / (sqrt(al) * sqrt(be)))));
      }
    }
    __syncthreads();
  }
  for (int l = warp; l < 2 * b; l += nwarps) {
    if (!valid(l)) continue;
    const int4* src = reinterpret_cast<const int4*>(C + (size_t)l * mp);
    int4* dst = reinterpret_cast<int4*>(Ws + (int64_t)gcol(l) * mp);
    for (int v = lane; v < vpc; v += 32) {
      const int4 t = src[v];
      dst[v] = PLANAR ? make_int4(t.x, t.z, t.y, t.w) : t;
    }
  }
  if constexpr (ACC) if (*flag) {
    // V^T rows of the pair's columns times J: one thread per element index, the 2b values in
    // registers, J broadcast from shared memory (rows past 2b are identity rows meeting zeros)
    T* Vs = Vacc + s * (int64_t)g.n * g.n;
    const int n = g.n;
    for (int i = tid; i < n; i += nth) {
      T v[kAccB];
#pragma unroll
      for (int l = 0; l < kAccB; ++l) v[l] = (l < 2 * b && valid(l)) ? Vs[(int64_t)gcol(l) * n + i] : zero_v<T>();
      for (int l2 = 0; l2 < 2 * b; ++l2) {
        if (!valid(l2)) continue;
        T acc = zero_v<T>();
#pragma unroll
        for (int l = 0; l < kAccB; ++l) fma_acc(acc, v[l], Jb[l * kAccB + l2]);
        Vs[(int64_t)gcol(l2) * n + i] = acc;
      }
    }
  }
  if (tid == 0 && *flag) {
    rot[s] = 1;
    if (relmax) atomicMax(&relmax[s], *fmax_sh);
  }
}

// after a sweep: a slice without rotations is converged; count the rest.  relmax (svt /
// values): so is a slice whose rotations all had relative inner products below `early`
// (the inner products they left behind are ~early^2, as in jacobi_qr_kernel)
__global__ void block_sweep_update_kernel(int64_t batch, int* __restrict__ rot, int* __restrict__ active,
                                          int* __restrict__ count, unsigned long long* stats,
                                          unsigned* __restrict__ relmax, float early) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int local = 0;
  for (int64_t s = threadIdx.x; s < batch; s += blockDim.x) {
    const int a = active[s];
    local += a;  // this slice took part in the sweep
    const bool small = relmax && __uint_as_float(relmax[s]) < early;
    active[s] = a && rot[s] && !small;
    rot[s] = 0;
    if (relmax) relmax[s] = 0u;
  }
  atomicAdd(&cnt, local);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (stats) atomicAdd(&stats[1], (unsigned long long)cnt);
    int c = 0;
    for (int64_t s = 0; s < batch; ++s) c += active[s];
    *count = c;
  }
}

// singular values, descending stable ranks and the outputs of JacobiOut
template <typename T, bool WANT_V>
__global__ void block_finalize_kernel(BlockGeom g, const T* __restrict__ W, JacobiOut o) {
  using R = typename scalar_traits<T>::real;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  R* sig = reinterpret_cast<R*>(smem_raw);
  int* rank_sh = reinterpret_cast<int*>(sig + g.n);
  int* kept_sh = rank_sh + g.n;
  const int64_t s = blockIdx.x;
  const int n = g.n, m = g.m, mp = g.mp;
  const T* Ws = W + s * (int64_t)n * mp;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  if (tid == 0) *kept_sh = 0;
  const bool dead = o.pre_active && !o.pre_active[s];
  for (int j = warp; j < n; j += nwarps) {
    R s2 = 0;
    if (!dead)
      for (int i = lane; i < m; i += 32) s2 += abs2_v(Ws[(int64_t)j * mp + i]);
    s2 = warp_sum_r(s2);
    if (lane == 0) sig[j] = sqrt(s2);
  }
  __syncthreads();
  R* sv_out = reinterpret_cast<R*>(o.sv_out);
  R* d_out = reinterpret_cast<R*>(o.d_out);
  int kept_local = 0;
  for (int j = tid; j < n; j += nth) {
    const R sj = sig[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const R si = sig[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    rank_sh[j] = rank;
    if (o.rank_out) o.rank_out[s * n + j] = rank;
    if (sv_out) sv_out[s * n + rank] = sj;
    const bool keep = sj > (R)o.tau && sj > (R)0;
    kept_local += keep;
    if (d_out) d_out[s * n + rank] = keep ? (((sj - (R)o.tau) / sj) / sj) / sj : (R)0;
  }
  if (kept_local) atomicAdd(kept_sh, kept_local);
  __syncthreads();
  if (o.kept_out && tid == 0) o.kept_out[s] = *kept_sh;
  if (o.stats && tid == 0) atomicAdd(&o.stats[0], 1ull);
  if (o.w_out && !dead) {
    T* dst = reinterpret_cast<T*>(o.w_out) + s * (int64_t)n * m;
    for (int j = warp; j < n; j += nwarps) {
      T* dj = dst + (int64_t)rank_sh[j] * m;
      const T* sj = Ws + (int64_t)j * mp;
      for (int i = lane; i < m; i += 32) dj[i] = sj[i];
    }
  }
  if (!WANT_V && o.v_out && o.v_acc) {  // accumulated rotations: row j of V^T goes to its sorted place
    T* dst = reinterpret_cast<T*>(o.v_out) + s * (int64_t)n * n;
    const T* src = reinterpret_cast<const T*>(o.v_acc) + s * (int64_t)n * n;
    for (int j = warp; j < n; j += nwarps) {
      T* dj = dst + (int64_t)rank_sh[j] * n;
      const T* sj = src + (int64_t)j * n;
      for (int i = lane; i < n; i += 32) dj[i] = sj[i];
    }
  }
  if (WANT_V && o.v_out) {
    T* dst = reinterpret_cast<T*>(o.v_out) + s * (int64_t)n * n;
    for (int j = warp; j < n; j += nwarps) {
      T* dj = dst + (int64_t)rank_sh[j] * n;
      const T* sj = Ws + (int64_t)j * mp + m;
      for (int i = lane; i < n; i += 32) dj[i] = sj[i];
    }
  }
}

// the sweep loop of the blocked tier for one kernel variant
template <typename T, bool WANT_V, int MPL, int NTMAX, int ACCB = 0>
int run_block_sweeps(ltb_ctx* ctx, int64_t batch, const BlockGeom& g, T* W, int* rot, int* active, int* count,
                     const JacobiOut& o, int max_sweeps, unsigned* relmax, float early) {
  using R = typename scalar_traits<T>::real;
  const int nbp = g.nb + (g.nb & 1);
  constexpr bool ACC = ACCB > 0;
  T* vacc = ACC ? reinterpret_cast<T*>(o.v_acc) : nullptr;
  const size_t smem = ACC ? block_acc_offset<T>(g.b, g.mp) + (size_t)ACCB * ACCB * sizeof(T)
                           : 2 * (size_t)g.mp * sizeof(T) * g.b + 2 * g.b * sizeof(R) + 16;
  auto kern = jacobi_block_kernel<T, WANT_V, MPL, NTMAX, ACCB>;
  LTB_TRY(ensure_smem(ctx, kern, smem));
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(ctx->stream, &cap);
  // truncated sweeps (o.lead with o.small2 > 0): one CTA per leading block, at most kLeadMax per slice
  const bool compact = o.lead && o.small2 > 0.f;
  const dim3 bgrid((unsigned)(compact ? std::min(kLeadMax, nbp / 2) : nbp / 2), (unsigned)batch);
  const int threads = 32 * std::min(g.b, NTMAX / 32);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int r = 0; r < nbp - 1; ++r) {
      kern<<<bgrid, threads, smem, ctx->stream>>>(g, r, r == 0 ? 1 : 0, W, rot, active, o.skip, relmax, vacc,
                                                  o.lead, o.lead ? o.small2 : 0.f, compact ? 1 : 0);
      LTB_LAUNCH_CHECK(ctx);
    }
    block_sweep_update_kernel<<<1, 256, 0, ctx->stream>>>(batch, rot, active, count, o.stats, relmax, early);
    LTB_LAUNCH_CHECK(ctx);
    if (cap != cudaStreamCaptureStatusNone) continue;  // no host read-back inside a capture
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scratch, count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (*reinterpret_cast<int*>(ctx->h_scratch) == 0) break;
  }
  return LTB_OK;
}

// ---- truncated sweeps (JacobiOut::truncate)
// With the working columns in descending order of norm (the carried, sigma-sorted bases) the
// singular values above tau live in the first few blocks.  A sweep that rotates only the pairs
// involving one of these `lead` blocks still converges (every rotation lowers off(W^H W)), to
// W = [W_L | W_S] with the columns of W_L mutually orthogonal and orthogonal to every column of
// W_S: the singular values of the slice are then the norms of W_L's columns together with the
// singular values of W_S, whatever the angles inside W_S.  The SVT only needs to know that no
// singular value of W_S exceeds tau: with S = W_S^H W_S / tau^2, lambda_max(S)^64 <= tr(S^64),
// so tr(S^64) <= 0.9 certifies it, and so does tr(S^(2^k)) <= 0.9 at any earlier squaring (up to
// six squarings of the Gram matrix on the tensor cores, stopped once every slice has passed; the
// last bound is within n^(1/128) = 5.6% of sigma_max(W_S)).  A slice that fails is finished with full
// sweeps.  lead = the blocks holding the columns with norm above 0.7 tau, plus two blocks.
constexpr float kLeadTheta = 0.7f;
constexpr double kCertifyBound = 0.9;
constexpr int kCertifySquarings = 6;
constexpr int kTruncSweeps = 16;  // truncated sweeps before a slice is handed to the full ones

template <typename T>
__global__ void block_lead_kernel(BlockGeom g, const T* __restrict__ W, double tau, int* __restrict__ lead) {
  using R = typename scalar_traits<T>::real;
  const int64_t s = blockIdx.x;
  const T* Ws = W + s * (int64_t)g.n * g.mp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ int last;
  if (threadIdx.x == 0) last = -1;
  __syncthreads();
  const double thr = (double)kLeadTheta * tau * (double)kLeadTheta * tau;
  for (int j = warp; j < g.n; j += nwarps) {
    R s2 = 0;
    for (int i = lane; i < g.m; i += 32) s2 += abs2_v(Ws[(int64_t)j * g.mp + i]);
    s2 = warp_sum_r(s2);
    if (lane == 0 && (double)s2 > thr) atomicMax(&last, j);  // the last large column decides
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int kl = (last + 1 + g.b - 1) / g.b + 1;
    lead[s] = (kl > kLeadMax || kl >= g.nb) ? g.nb : kl;  // (g.nb: not truncated, left to the full sweeps)
  }
}

// S <- mask(S) / tau^2: rows / columns of the large columns (squared norm = diagonal entry > small2)
// are zeroed: what remains is the Gram matrix of the small columns W_S
__global__ void certify_diag_kernel(int n, const cplx<float>* __restrict__ S, float* __restrict__ diag) {
  const int64_t off = (int64_t)blockIdx.y * n * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    diag[(int64_t)blockIdx.y * n + i] = S[off + (int64_t)i * n + i].re;
}
__global__ void certify_mask_kernel(int n, double tau, float small2, const float* __restrict__ diag,
                                    cplx<float>* __restrict__ S, const int* skip) {
  if (skip && *skip) return;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  const float* dg = diag + (int64_t)blockIdx.y * n;
  const float sc = (float)(1.0 / (tau * tau));
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n, j = l - i * n;
    cplx<float> v = S[off + l];
    // (a band above the sweeps' threshold: a column whose norm sits within rounding of it may have
    // been treated as small by a round, so it must be covered by the certificate)
    const float lim = small2 * 1.001f;
    const bool keep = dg[i] <= lim && dg[j] <= lim;
    S[off + l] = cplx<float>{keep ? v.re * sc : 0.f, keep ? v.im * sc : 0.f};
  }
}

// after each squaring: slices whose trace bound already holds pass; once every slice has passed the
// remaining squarings are skipped (cflags[0], the skip slot of their GEMMs); cflags[1 + s] = passed
__global__ void certify_init_kernel(int64_t batch, int* __restrict__ cflags, const int* __restrict__ skip) {
  for (int64_t s = threadIdx.x; s < batch; s += blockDim.x) cflags[1 + s] = 0;
  if (threadIdx.x == 0) cflags[0] = (skip && *skip) ? 1 : 0;
}
__global__ void certify_level_kernel(int64_t batch, int n, int nb, const cplx<float>* __restrict__ S,
                                     const int* __restrict__ was_active, const int* __restrict__ lead,
                                     int* __restrict__ cflags) {
  if (cflags[0]) return;  // (done: S was not updated by the skipped squaring)
  __shared__ int open_cnt;
  if (threadIdx.x == 0) open_cnt = 0;
  __syncthreads();
  for (int64_t s = threadIdx.x; s < batch; s += blockDim.x) {
    if (!was_active[s] || lead[s] >= nb || cflags[1 + s]) continue;
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += (double)S[s * (int64_t)n * n + (int64_t)i * n + i].re;
    if (tr <= kCertifyBound) cflags[1 + s] = 1;
    else atomicAdd(&open_cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0 && open_cnt == 0) cflags[0] = 1;
}

// a slice without a certificate (or whose truncated sweeps did not converge) becomes active again
// with every block leading
__global__ void certify_decide_kernel(int64_t batch, int nb, const int* __restrict__ cflags,
                                      const int* __restrict__ was_active, int* __restrict__ active,
                                      int* __restrict__ lead, int* __restrict__ count, const int* __restrict__ skip) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const bool stop = skip && *skip;
  for (int64_t s = threadIdx.x; s < batch; s += blockDim.x) {
    int fail = 0;
    if (!stop && was_active[s]) fail = lead[s] >= nb ? 1 : (active[s] || !cflags[1 + s]);
    active[s] = fail;
    if (fail) {
      lead[s] = nb;
      atomicAdd(&cnt, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *count = cnt;
}

// after the truncated sweeps: certify the small columns; *h_failed = slices to finish with full sweeps
inline int block_certify(ltb_ctx* ctx, int64_t batch, const BlockGeom& g, const cplx<float>* W, double tau,
                         float small2, const int* was_active, int* active, int* lead, int* count, const int* skip,
                         int* h_failed) {
  using T = cplx<float>;
  const int64_t n = g.n, nn = n * n;
  WsScope ws(ctx);
  T *S1 = nullptr, *S2 = nullptr;
  float* diag = nullptr;
  int* cflags = nullptr;
  LTB_TRY(ws.alloc(sizeof(T) * batch * nn, &S1));
  LTB_TRY(ws.alloc(sizeof(T) * batch * nn, &S2));
  LTB_TRY(ws.alloc(sizeof(float) * batch * n, &diag));
  LTB_TRY(ws.alloc(sizeof(int) * (batch + 1), &cflags));
  certify_init_kernel<<<1, 256, 0, ctx->stream>>>(batch, cflags, skip);
  LTB_LAUNCH_CHECK(ctx);
  // Gram matrix of the working columns (row j of the n x mp array W is column j; padding rows are zero)
  LTB_TRY(ltb_gemm_impl(ctx, LTB_C64, batch, n, n, g.mp, LTB_OP_C, W, g.mp, n * g.mp, LTB_OP_T, W, g.mp, n * g.mp, S1,
                        n, nn, nullptr, nullptr, nullptr, nullptr, nullptr, cflags));
  const dim3 egrid((unsigned)std::min<int64_t>((nn + 1023) / 1024, 64), (unsigned)batch);
  certify_diag_kernel<<<dim3((unsigned)((n + 255) / 256), (unsigned)batch), 256, 0, ctx->stream>>>((int)n, S1, diag);
  LTB_LAUNCH_CHECK(ctx);
  certify_mask_kernel<<<egrid, 256, 0, ctx->stream>>>((int)n, tau, small2, diag, S1, cflags);
  LTB_LAUNCH_CHECK(ctx);
  for (int q = 0; q < kCertifySquarings; ++q) {
    LTB_TRY(ltb_gemm_impl(ctx, LTB_C64, batch, n, n, n, LTB_OP_N, S1, n, nn, LTB_OP_N, S1, n, nn, S2, n, nn, nullptr,
                          nullptr, nullptr, nullptr, nullptr, cflags));
    std::swap(S1, S2);
    certify_level_kernel<<<1, 256, 0, ctx->stream>>>(batch, (int)n, g.nb, S1, was_active, lead, cflags);
    LTB_LAUNCH_CHECK(ctx);
  }
  certify_decide_kernel<<<1, 256, 0, ctx->stream>>>(batch, g.nb, cflags, was_active, active, lead, count, skip);
  LTB_LAUNCH_CHECK(ctx);
  LTB_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_scratch, count, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  *h_failed = *reinterpret_cast<int*>(ctx->h_scratch);
  return LTB_OK;
}

template <typename T, bool WANT_V>
int launch_jacobi_blocked(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const T* A, const JacobiOut& o_in,
                          int max_sweeps) {
  JacobiOut o = o_in;
  using R = typename scalar_traits<T>::real;
  if (batch > 65535) return ltb_set_error(ctx, LTB_ESHAPE, "svd: batch too large for the blocked tier");
  BlockGeom g;
  g.m = (int)std::max(I1, I2);
  g.n = (int)std::min(I1, I2);
  const int rows = g.m + (WANT_V ? g.n : 0);
  // register-tile variants (fp32 / complex64 SVT): rows padded to 32 * MPL, block size capped
  // by the variant's thread count (registers per thread)
  constexpr bool f32 = std::is_same<T, float>::value, c32 = std::is_same<T, cplx<float>>::value;
  constexpr bool f64 = std::is_same<T, double>::value;
  int mpl = 0, ntmax = 1024;
  if constexpr (!WANT_V && f64) {  // fp64 register tiles only with rotation accumulation (t_svd)
    const int need = (rows + 31) / 32;
    if (o.v_acc && need <= 16) mpl = need <= 8 ? 8 : 16;
  }
  if constexpr (!WANT_V && (f32 || c32)) {
    const int need = (rows + 31) / 32;
    if (need <= 8) {
      mpl = 8;
    } else if (need <= 16) {
      mpl = 16;
      ntmax = f32 ? 1024 : 512;
    } else if (need <= 32) {
      mpl = 32;
      ntmax = f32 ? 512 : 384;
    }
  }
  const int per16 = 16 / (int)std::min<size_t>(sizeof(T), 16);
  g.mp = mpl > 0 ? 32 * mpl : (rows + 31) / 32 * 32;
  g.mp = (g.mp + per16 - 1) / per16 * per16;
  const size_t colb = (size_t)g.mp * sizeof(T);
  const size_t fit = (kBlockSmem - 256) / (2 * colb);
  if (fit < 1) return ltb_set_error(ctx, LTB_EUNSUPPORTED, "svd: slice columns too long for the blocked tier");
  g.b = (int)std::min<size_t>(std::min<size_t>((size_t)ntmax / 32, (size_t)std::max(1, (g.n + 1) / 2)), fit);
  if (!WANT_V && (c32 || f32 || f64) && o.v_acc) g.b = std::min(g.b, acc_dim<T>::value / 2);
  g.nb = (g.n + g.b - 1) / g.b;
  T* W = nullptr;
  int* flags = nullptr;
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * (size_t)batch * g.n * g.mp, (void**)&W));
  LTB_TRY(ltb_ws_alloc(ctx, sizeof(int) * (size_t)(3 * batch + 4), (void**)&flags));
  int* rot = flags;
  int* active = flags + batch;
  unsigned* relmax = nullptr;
  float early = 0.f;
  if ((f32 || c32) && !WANT_V && !o.v_out && g_qr_early > 0.f) {  // svt / values in single precision
    relmax = reinterpret_cast<unsigned*>(flags + 2 * batch);
    early = g_qr_early * sqrtf(FLT_EPSILON * sqrtf((float)std::max(g.m, 1)));
  } else if (o.early_stop > 0.f) {  // the caller's early stop (warm carried fp64 SVT: sqrt(tol))
    relmax = reinterpret_cast<unsigned*>(flags + 2 * batch);
    early = o.early_stop;
  }
  int* count = flags + 3 * batch;
  LTB_CUDA_TRY(ctx, cudaMemsetAsync(rot, 0, sizeof(int) * batch, ctx->stream));
  LTB_CUDA_TRY(ctx, cudaMemsetAsync(flags + 2 * batch, 0, sizeof(int) * batch, ctx->stream));
  if (o.pre_active) {
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(active, o.pre_active, sizeof(int) * batch, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    fill_int_kernel<<<grid_for(batch, 256, 1024), 256, 0, ctx->stream>>>(batch, active, 1);
    LTB_LAUNCH_CHECK(ctx);
  }
  {
    dim3 grid((unsigned)std::min<int64_t>(((int64_t)g.n * g.mp + 255) / 256, 256), (unsigned)batch);
    block_load_kernel<T, WANT_V><<<grid, 256, 0, ctx->stream>>>(I1, I2, A, W, g);
    LTB_LAUNCH_CHECK(ctx);
  }
  auto sweeps = [&](int max_sweeps) -> int {
    int st = LTB_OK;
    if constexpr (!WANT_V && (c32 || f32 || f64)) {
      if (o.v_acc) {  // rotation accumulation: blocks of at most ACCB / 2 columns, one warp per column
        constexpr int AB = acc_dim<T>::value, NT = 16 * AB;
        if (mpl == 8) st = run_block_sweeps<T, WANT_V, 8, NT, AB>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
        else if (mpl == 16) st = run_block_sweeps<T, WANT_V, 16, NT, AB>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
        else if (mpl == 32 && !f64) st = run_block_sweeps<T, WANT_V, f64 ? 0 : 32, NT, AB>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
        else st = run_block_sweeps<T, WANT_V, 0, NT, AB>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
        LTB_TRY(st);
        st = -1;
      }
    }
    if (st == -1) {
      st = LTB_OK;
    } else if constexpr (!WANT_V && (f32 || c32)) {
      if (mpl == 8) st = run_block_sweeps<T, WANT_V, 8, 1024>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
      else if (mpl == 16 && f32) st = run_block_sweeps<T, WANT_V, 16, 1024>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
      else if (mpl == 16) st = run_block_sweeps<T, WANT_V, 16, 512>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
      else if (mpl == 32 && f32) st = run_block_sweeps<T, WANT_V, 32, 512>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
      else if (mpl == 32) st = run_block_sweeps<T, WANT_V, 32, 384>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
      else st = run_block_sweeps<T, WANT_V, 0, 1024>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
    } else {
      st = run_block_sweeps<T, WANT_V, 0, 1024>(ctx, batch, g, W, rot, active, count, o, max_sweeps, relmax, early);
    }
    return st;
  };
  if (g.n > 1) {
    bool truncated = false;
    int* lead = nullptr;
    int* was_active = nullptr;
    if constexpr (c32 && !WANT_V) {
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      cudaStreamIsCapturing(ctx->stream, &cap);
      if (o.truncate && o.tau > 0.0 && o.v_acc && cap == cudaStreamCaptureStatusNone && g.nb > 3) {
        LTB_TRY(ltb_ws_alloc(ctx, sizeof(int) * (size_t)(2 * batch), (void**)&lead));
        was_active = lead + batch;
        block_lead_kernel<T><<<(unsigned)batch, 256, 0, ctx->stream>>>(g, W, o.tau, lead);
        LTB_LAUNCH_CHECK(ctx);
        LTB_CUDA_TRY(ctx, cudaMemcpyAsync(was_active, active, sizeof(int) * batch, cudaMemcpyDeviceToDevice, ctx->stream));
        o.lead = lead;
        o.small2 = (float)((double)kLeadTheta * o.tau * (double)kLeadTheta * o.tau);
        truncated = true;
      }
    }
    int st = sweeps(truncated ? std::min(max_sweeps, kTruncSweeps) : max_sweeps);
    if constexpr (c32 && !WANT_V) {
      if (truncated && st == LTB_OK) {
        int failed = 0;
        st = block_certify(ctx, batch, g, W, o.tau, o.small2, was_active, active, lead, count, o.skip, &failed);
        // full sweeps for the slices without a certificate (lead = every block: no pair is skipped)
        if (st == LTB_OK && failed > 0) {
          o.small2 = 0.f;
          st = sweeps(max_sweeps);
        }
      }
    }
    if (lead) ltb_ws_free(ctx, lead);
    LTB_TRY(st);
  }
  const size_t fsmem = (size_t)g.n * (sizeof(R) + sizeof(int)) + 16;
  auto fin = block_finalize_kernel<T, WANT_V>;
  LTB_TRY(ensure_smem(ctx, fin, fsmem));
  fin<<<(unsigned)batch, 512, fsmem, ctx->stream>>>(g, W, o);
  LTB_LAUNCH_CHECK(ctx);
  ltb_ws_free(ctx, W);
  ltb_ws_free(ctx, flags);
  return LTB_OK;
}

// t_svd on the blocked tier for fp32 / complex64: the V-free kernel variants (register tiles,
// working columns of m rows instead of m + n) with the rotations accumulated per block pair
// and applied to V^T (JacobiOut::v_acc), instead of V riding along as extra rows
template <typename T>
__global__ void set_identity_kernel(int n, T* __restrict__ VT) {
  using R = typename scalar_traits<T>::real;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    VT[off + l] = cvt<T>((R)((l - i * n == i) ? 1 : 0));
  }
}

template <typename T>
int launch_jacobi_blocked_acc(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const T* A, JacobiOut o,
                              int max_sweeps) {
  const int64_t n = std::min(I1, I2);
  WsScope ws(ctx);
  T* vt = nullptr;
  LTB_TRY(ws.alloc(sizeof(T) * batch * n * n, &vt));
  const dim3 grid((unsigned)std::min<int64_t>((n * n + 1023) / 1024, 64), (unsigned)batch);
  set_identity_kernel<T><<<grid, 256, 0, ctx->stream>>>((int)n, vt);
  LTB_LAUNCH_CHECK(ctx);
  o.v_acc = vt;
  return launch_jacobi_blocked<T, false>(ctx, batch, I1, I2, A, o, max_sweeps);
}

template <typename T, bool WANT_V>
int launch_jacobi_blocked_any(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const T* A, const JacobiOut& o,
                              int max_sweeps) {
  if constexpr (WANT_V && (std::is_same<T, float>::value || std::is_same<T, cplx<float>>::value ||
                           std::is_same<T, double>::value)) {
    // only when V riding along as n extra rows would not allow larger blocks than the accumulation
    // does (acc_dim / 2 columns): smaller blocks mean more rounds per sweep (fp64: n = 512 gains,
    // n = 128 / 256 would lose)
    const int64_t n = std::min(I1, I2), rows_v = (std::max(I1, I2) + n + 31) / 32 * 32;
    const int64_t fit_v = (int64_t)((kBlockSmem - 256) / (2 * rows_v * sizeof(T)));
    const int64_t b_v = std::min<int64_t>(std::min<int64_t>(32, (n + 1) / 2), fit_v);
    if (batch <= 65535 && n > 1 && b_v <= acc_dim<T>::value / 2)
      return launch_jacobi_blocked_acc<T>(ctx, batch, I1, I2, A, o, max_sweeps);
  }
  return launch_jacobi_blocked<T, WANT_V>(ctx, batch, I1, I2, A, o, max_sweeps);
}

template <typename T, bool WANT_V>
int launch_jacobi(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const T* A, JacobiOut o) {
  using R = typename scalar_traits<T>::real;
  const int m = (int)std::max(I1, I2), n = (int)std::min(I1, I2);
  const int max_sweeps = std::is_same<R, float>::value ? 40 : 60;
  if (batch > 0x7fffffff) return ltb_set_error(ctx, LTB_ESHAPE, "svd: batch too large");
  o.stats = ctx->d_stats;
  constexpr bool big = std::is_same<T, cplx<double>>::value;
  if (ctx->opt_force_blocked) return launch_jacobi_blocked_any<T, WANT_V>(ctx, batch, I1, I2, A, o, max_sweeps);
  auto fits = [&](int mp) { return jacobi_smem_bytes<T>(m, n, WANT_V, mp) <= kSmemLimit; };
  if (m <= 8 && fits(8)) return launch_smem<T, WANT_V, 4, 2>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  if (m <= 32 && fits(32)) return launch_smem<T, WANT_V, 8, 4>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  if (m <= 64 && fits(64)) return launch_smem<T, WANT_V, 16, 4>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  if constexpr (!big) {
    if (m <= 128 && fits(128)) return launch_smem<T, WANT_V, 16, 8>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
    if (m <= 192 && fits(192)) return launch_smem<T, WANT_V, 16, 12>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
    if (m <= 256 && fits(256)) return launch_smem<T, WANT_V, 32, 8>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  } else {
    if (m <= 128 && fits(128)) return launch_smem<T, WANT_V, 32, 4>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  }
  if (fits(m | 1)) return launch_smem<T, WANT_V, 32, 0>(ctx, batch, I1, I2, A, o, max_sweeps, m, n);
  return launch_jacobi_blocked_any<T, WANT_V>(ctx, batch, I1, I2, A, o, max_sweeps);
}

// ---------------------------------------------------------------- QR-preconditioned fp32 SVT
// For an fp32 SVT the oriented slice W (m x n, m >= n) is first reduced by a
// Householder QR in shared memory, W = Q R, and the one-sided Jacobi runs on
// the n columns of X = R^T (Drmac-Veselic preconditioning): X J = V Sigma, the
// Jacobi columns y_j = sigma_j v_j are W's right singular vectors scaled by
// sigma.  The slice shrinks from m to n rows and the sweep count drops (13 ->
// 9-10 on config-3 iterates, tools/ sweep study); Q is never formed:
//   svt(W) = W V diag((s - tau)_+ / s) V^T = W (Y~ Y~^T),  y~_j = y_j sqrt((s_j - tau)_+ / s_j) / s_j,
// so the kernel emits Y~ (sorted, scaled) and two tensor-core GEMMs finish:
// Z = Y~ Y~^T, then out = A Z (I1 >= I2) or Z A (I1 < I2).
// CHOL: A holds the Gram matrices G = W^T W (batch x n x n, symmetric) of slices whose
// columns are nearly orthogonal (the carried PGA bases); the triangular factor comes from
// an in-place Cholesky, G = L L^T with L = R^T, accurate here because the diagonally
// scaled Gram matrix is well conditioned, and much shorter than the Householder QR.
// SLOTS: most pairs per team per round (1 when the teams cover every pair: the slot
// arrays then stay in registers instead of spilling to local memory)
// rotation parameters of one Jacobi pair (fp32, MUFU): on return c, sn, sg and tt describe
// the rotation w_p' = c w_p - sn sg w_q, w_q' = sn w_p + c sg w_q and the analytic norm
// update alpha' = alpha - tt |g|, beta' = beta + tt |g|; a pair below the threshold (or with
// norms / inner product below FLT_MIN) gets the identity (c = 1, sn = tt = 0, sg = 1), which
// leaves both columns bit-identical.  Returns whether the pair rotates; rel = |g| / sqrt(ab).
__device__ __forceinline__ bool jacobi_pair_params(float g, float al, float be, float tol, float& c, float& sn,
                                                   float& sg, float& tt, float& gabs, float& rel) {
  gabs = fabsf(g);
  const float sab = sqrt_apx(al) * sqrt_apx(be);
  const bool doit = (gabs > tol * sab) && (fminf(fminf(al, be), gabs) >= FLT_MIN);
  const float zeta = (be - al) * (0.5f * rcp_apx(gabs));
  const float az = fabsf(zeta);
  const float den = az < 1e18f ? az + sqrt_apx(fmaf(az, az, 1.f)) : 2.f * az;
  tt = copysignf(rcp_apx(den), zeta);
  const float x1 = fmaf(tt, tt, 1.f);
  float cc = rsqrt_apx(x1);
  cc = cc * fmaf(-0.5f * x1 * cc, cc, 1.5f);
  rel = doit ? gabs * rcp_apx(sab) : 0.f;
  c = doit ? cc : 1.f;
  sn = doit ? cc * tt : 0.f;
  tt = doit ? tt : 0.f;
  sg = (doit && g < 0.f) ? -1.f : 1.f;
  gabs = doit ? gabs : 0.f;  // (a NaN inner product must not reach the norm updates)
  return doit;
}

// Block-pair one-sided Jacobi sweeps over the n columns of W (n rows each, n % 4 == 0,
// blockDim.x == 2 n): the columns form n / 2 blocks of two, the circle method pairs the
// blocks (n / 2 - 1 rounds of n / 4 block pairs), and one 8-lane team takes one block pair
// per round: it loads the four columns into registers (MPL rows per lane, two rows per
// 8-byte access), rotates the four cross pairs in two steps of two disjoint pairs (plus the
// two within-block pairs in the sweep's first round), and stores the four columns back.
// Against one pair per team per round this halves the rounds, the barriers and the
// shared-memory traffic per rotation (the one-pair kernel is bound by that traffic,
// ~1.4 us per round on a config-3 slice); the four columns need ~72 registers per thread,
// which the 288-thread CTAs (two per SM) allow.  Same rotations, thresholds, analytic norm
// updates and stopping rules as the one-pair path.  Returns the number of sweeps run.
template <int MPL>
__device__ int jacobi_block_sweeps(float* W, int pitch, int n, float* nrm, int* flags, int* smax, float tol,
                                   int max_sweeps, float early_stop) {
  constexpr int H = MPL / 2;  // float2 per lane per column
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int team = tid >> 3, tl = tid & 7;
  const int nbk = n >> 1, m1 = nbk - 1;
  float* const Wc = W + 2 * tl;
  int sweeps_done = 0;
  for (int sweep = 0; sweep < max_sweeps && n > 1; ++sweep) {
    int* rot = &flags[sweep & 1];
    for (int j = warp; j < n; j += nwarps) {
      const float* wj = W + (size_t)j * pitch;
      float s2 = 0.f;
      for (int i = lane; i < n; i += 32) s2 += wj[i] * wj[i];
      s2 = warp_sum(s2);
      if (lane == 0) nrm[j] = s2;
    }
    __syncthreads();
    int P = team == 0 ? m1 : team, Q = team == 0 ? 0 : m1 - team;
    for (int r = 0; r < m1; ++r) {
      const int col[4] = {2 * P, 2 * P + 1, 2 * Q, 2 * Q + 1};
      float2 X[4][H];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < H; ++h) X[k][h] = *reinterpret_cast<const float2*>(Wc + (size_t)col[k] * pitch + 16 * h);
      float nr[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) nr[k] = nrm[col[k]];
      bool any = false;
      float worst = 0.f;
      // steps: (0,1)(2,3) within the blocks on the first round; then (0,2)(1,3), (0,3)(1,2)
#pragma unroll
      for (int st = 0; st < 3; ++st) {
        if (st == 0 && r != 0) continue;
        const int a0 = 0, b0 = st == 0 ? 1 : (st == 1 ? 2 : 3);
        const int a1 = st == 0 ? 2 : 1, b1 = st == 0 ? 3 : (st == 1 ? 3 : 2);
        float2 u0 = make_float2(0.f, 0.f), u1 = u0, v0 = u0, v1 = u0;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          if (h & 1) {
            u1 = __ffma2_rn(X[a0][h], X[b0][h], u1);
            v1 = __ffma2_rn(X[a1][h], X[b1][h], v1);
          } else {
            u0 = __ffma2_rn(X[a0][h], X[b0][h], u0);
            v0 = __ffma2_rn(X[a1][h], X[b1][h], v0);
          }
        }
        float g0 = (u0.x + u1.x) + (u0.y + u1.y), g1 = (v0.x + v1.x) + (v0.y + v1.y);
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) {
          g0 += __shfl_xor_sync(0xffffffffu, g0, off);
          g1 += __shfl_xor_sync(0xffffffffu, g1, off);
        }
        float c0, s0, sg0, t0, ga0, r0, c1, s1, sg1, t1, ga1, r1;
        any |= jacobi_pair_params(g0, nr[a0], nr[b0], tol, c0, s0, sg0, t0, ga0, r0);
        any |= jacobi_pair_params(g1, nr[a1], nr[b1], tol, c1, s1, sg1, t1, ga1, r1);
        worst = fmaxf(worst, fmaxf(r0, r1));
        const float2 C0 = make_float2(c0, c0), S0 = make_float2(s0, s0), N0 = make_float2(-s0 * sg0, -s0 * sg0),
                     Q0 = make_float2(c0 * sg0, c0 * sg0);
        const float2 C1 = make_float2(c1, c1), S1 = make_float2(s1, s1), N1 = make_float2(-s1 * sg1, -s1 * sg1),
                     Q1 = make_float2(c1 * sg1, c1 * sg1);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float2 xa = X[a0][h], xb = X[b0][h], ya = X[a1][h], yb = X[b1][h];
          X[a0][h] = __ffma2_rn(C0, xa, __fmul2_rn(N0, xb));
          X[b0][h] = __ffma2_rn(S0, xa, __fmul2_rn(Q0, xb));
          X[a1][h] = __ffma2_rn(C1, ya, __fmul2_rn(N1, yb));
          X[b1][h] = __ffma2_rn(S1, ya, __fmul2_rn(Q1, yb));
        }
        nr[a0] = fmaxf(nr[a0] - t0 * ga0, 0.f);
        nr[b0] = nr[b0] + t0 * ga0;
        nr[a1] = fmaxf(nr[a1] - t1 * ga1, 0.f);
        nr[b1] = nr[b1] + t1 * ga1;
      }
      if (any) {  // team-uniform: the four columns changed
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int h = 0; h < H; ++h) *reinterpret_cast<float2*>(Wc + (size_t)col[k] * pitch + 16 * h) = X[k][h];
        if (tl == 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) nrm[col[k]] = nr[k];
          *rot = 1;
          atomicMax(&smax[sweep & 1], __float_as_int(worst));
        }
      }
      P = team == 0 ? m1 : (P + 1 == m1 ? 0 : P + 1);
      Q = Q + 1 == m1 ? 0 : Q + 1;
      __syncthreads();
    }
    const int anyr = *rot;
    const float worst = __int_as_float(smax[sweep & 1]);
    __syncthreads();
    if (tid == 0) flags[(sweep + 1) & 1] = smax[(sweep + 1) & 1] = 0;
    __syncthreads();
    sweeps_done = sweep + 1;
    if (!anyr || worst < early_stop) break;
  }
  return sweeps_done;
}

// One step of the 4-column-block Jacobi (jacobi_block4_sweeps): four disjoint pairs
// (A_j, B_j) of the team's eight register columns.  The four inner products are reduced over
// the team's 16 lanes in five shuffles (after the first two levels each lane keeps one of the
// four sums), lanes 4j..4j+3 compute pair j's rotation, and its (c sg, sn, tt |g|) reach the
// other lanes by shuffles; the rotations then run two pairs per FFMA2.
template <int R, int A0, int B0, int A1, int B1, int A2, int B2, int A3, int B3>
__device__ __forceinline__ void blk4_step(float (&X)[8][R], float* nrm, int p4, int q4, int tl, int lane, float tol,
                                          bool& any, float& worst) {
  float2 d01 = make_float2(0.f, 0.f), d23 = d01, e01 = d01, e23 = d01;
#pragma unroll
  for (int h = 0; h < R; ++h) {
    if (h & 1) {
      e01 = __ffma2_rn(make_float2(X[A0][h], X[A1][h]), make_float2(X[B0][h], X[B1][h]), e01);
      e23 = __ffma2_rn(make_float2(X[A2][h], X[A3][h]), make_float2(X[B2][h], X[B3][h]), e23);
    } else {
      d01 = __ffma2_rn(make_float2(X[A0][h], X[A1][h]), make_float2(X[B0][h], X[B1][h]), d01);
      d23 = __ffma2_rn(make_float2(X[A2][h], X[A3][h]), make_float2(X[B2][h], X[B3][h]), d23);
    }
  }
  d01 = make_float2(d01.x + e01.x, d01.y + e01.y);
  d23 = make_float2(d23.x + e23.x, d23.y + e23.y);
  const bool b3 = tl & 8, b2 = tl & 4;
  float k0 = b3 ? d23.x : d01.x, k1 = b3 ? d23.y : d01.y;
  const float s0 = b3 ? d01.x : d23.x, s1 = b3 ? d01.y : d23.y;
  k0 += __shfl_xor_sync(0xffffffffu, s0, 8);
  k1 += __shfl_xor_sync(0xffffffffu, s1, 8);
  float f = b2 ? k1 : k0;
  f += __shfl_xor_sync(0xffffffffu, b2 ? k0 : k1, 4);
  f += __shfl_xor_sync(0xffffffffu, f, 2);
  f += __shfl_xor_sync(0xffffffffu, f, 1);
  // this lane's pair j = 2 b3 + b2: its columns' norms (shared memory, kept by lane 4 j)
  constexpr int kA = A0 | (A1 << 3) | (A2 << 6) | (A3 << 9), kB = B0 | (B1 << 3) | (B2 << 6) | (B3 << 9);
  const int sh = 3 * ((b3 ? 2 : 0) + (b2 ? 1 : 0));
  const int ka = (kA >> sh) & 7, kb = (kB >> sh) & 7;
  const int ca = (ka < 4 ? p4 : q4) + (ka & 3), cb = (kb < 4 ? p4 : q4) + (kb & 3);
  const float al = nrm[ca], be = nrm[cb];
  float c, sn, sg, tt, gabs, rel;
  const bool doit = jacobi_pair_params(f, al, be, tol, c, sn, sg, tt, gabs, rel);
  any |= doit;
  worst = fmaxf(worst, rel);
  __syncwarp();
  if ((tl & 3) == 0 && doit) {
    nrm[ca] = fmaxf(al - tt * gabs, 0.f);
    nrm[cb] = be + tt * gabs;
  }
  __syncwarp();
  const float qv = c * sg;
  const int base = lane & 16;
  float Qj[4], Sj[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    Qj[j] = __shfl_sync(0xffffffffu, qv, base + 4 * j);
    Sj[j] = __shfl_sync(0xffffffffu, sn, base + 4 * j);
  }
  // w_a' = c w_a - sn sg w_b, w_b' = sn w_a + c sg w_b  (c = |c sg|, sg = sign(c sg))
  const float2 C01 = make_float2(fabsf(Qj[0]), fabsf(Qj[1])), C23 = make_float2(fabsf(Qj[2]), fabsf(Qj[3]));
  const float2 S01 = make_float2(Sj[0], Sj[1]), S23 = make_float2(Sj[2], Sj[3]);
  const float2 Q01 = make_float2(Qj[0], Qj[1]), Q23 = make_float2(Qj[2], Qj[3]);
  const float2 N01 = make_float2(Qj[0] < 0.f ? Sj[0] : -Sj[0], Qj[1] < 0.f ? Sj[1] : -Sj[1]);
  const float2 N23 = make_float2(Qj[2] < 0.f ? Sj[2] : -Sj[2], Qj[3] < 0.f ? Sj[3] : -Sj[3]);
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const float2 xa = make_float2(X[A0][h], X[A1][h]), xb = make_float2(X[B0][h], X[B1][h]);
    const float2 ya = make_float2(X[A2][h], X[A3][h]), yb = make_float2(X[B2][h], X[B3][h]);
    const float2 na = __ffma2_rn(C01, xa, __fmul2_rn(N01, xb)), nb = __ffma2_rn(S01, xa, __fmul2_rn(Q01, xb));
    const float2 ma = __ffma2_rn(C23, ya, __fmul2_rn(N23, yb)), mb = __ffma2_rn(S23, ya, __fmul2_rn(Q23, yb));
    X[A0][h] = na.x, X[A1][h] = na.y, X[B0][h] = nb.x, X[B1][h] = nb.y;
    X[A2][h] = ma.x, X[A3][h] = ma.y, X[B2][h] = mb.x, X[B3][h] = mb.y;
  }
}

// Block Jacobi with blocks of four columns (n = 16 R, blockDim.x == 2 n): 16-lane teams
// hold a block pair (eight columns, R rows per lane at stride 16) in registers, rotate its 16
// cross pairs in four steps of four disjoint pairs (and the within-block pairs in three more
// steps on the sweep's first round); n / 4 - 1 rounds per sweep.  Against the two-column
// blocks this halves the rounds and the shared-memory traffic per rotation again (that
// traffic bounds both), and the FFMA2s carry two pairs each.  pitch = 4 (mod 8): the two
// teams of a warp read columns 4P + i, 4(P + 1) + i, whose 64-byte rows then fall in
// complementary bank halves.  Same rotations, thresholds and stopping rules.
template <int R>
__device__ int jacobi_block4_sweeps(float* W, int pitch, int n, float* nrm, int* flags, int* smax, float tol,
                                    int max_sweeps, float early_stop) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int team = tid >> 4, tl = tid & 15;
  const int nbk = n >> 2, m1 = nbk - 1;
  float* const Wc = W + tl;
  int sweeps_done = 0;
  for (int sweep = 0; sweep < max_sweeps && n > 1; ++sweep) {
    int* rot = &flags[sweep & 1];
    for (int j = warp; j < n; j += nwarps) {
      const float* wj = W + (size_t)j * pitch;
      float s2 = 0.f;
      for (int i = lane; i < n; i += 32) s2 += wj[i] * wj[i];
      s2 = warp_sum(s2);
      if (lane == 0) nrm[j] = s2;
    }
    __syncthreads();
    int P = team == 0 ? m1 : team, Q = team == 0 ? 0 : m1 - team;
    for (int r = 0; r < m1; ++r) {
      float X[8][R];
      const int p4 = 4 * P, q4 = 4 * Q;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int col = (k < 4 ? p4 : q4) + (k & 3);
#pragma unroll
        for (int h = 0; h < R; ++h) X[k][h] = Wc[(size_t)col * pitch + 16 * h];
      }
      bool any = false;
      float worst = 0.f;
      if (r == 0) {  // the within-block pairs, once per sweep
        blk4_step<R, 0, 1, 2, 3, 4, 5, 6, 7>(X, nrm, p4, q4, tl, lane, tol, any, worst);
        blk4_step<R, 0, 2, 1, 3, 4, 6, 5, 7>(X, nrm, p4, q4, tl, lane, tol, any, worst);
        blk4_step<R, 0, 3, 1, 2, 4, 7, 5, 6>(X, nrm, p4, q4, tl, lane, tol, any, worst);
      }
      blk4_step<R, 0, 4, 1, 5, 2, 6, 3, 7>(X, nrm, p4, q4, tl, lane, tol, any, worst);
      blk4_step<R, 0, 5, 1, 6, 2, 7, 3, 4>(X, nrm, p4, q4, tl, lane, tol, any, worst);
      blk4_step<R, 0, 6, 1, 7, 2, 4, 3, 5>(X, nrm, p4, q4, tl, lane, tol, any, worst);
      blk4_step<R, 0, 7, 1, 4, 2, 5, 3, 6>(X, nrm, p4, q4, tl, lane, tol, any, worst);
      if (__any_sync(0xffffffffu, any)) {  // warp-uniform: store the (possibly) rotated columns
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int col = (k < 4 ? p4 : q4) + (k & 3);
#pragma unroll
          for (int h = 0; h < R; ++h) Wc[(size_t)col * pitch + 16 * h] = X[k][h];
        }
        const int wbits = __reduce_max_sync(0xffffffffu, __float_as_int(worst));
        if (lane == 0) {
          *rot = 1;
          atomicMax(&smax[sweep & 1], wbits);
        }
      }
      P = team == 0 ? m1 : (P + 1 == m1 ? 0 : P + 1);
      Q = Q + 1 == m1 ? 0 : Q + 1;
      __syncthreads();
    }
    const int anyr = *rot;
    const float worst = __int_as_float(smax[sweep & 1]);
    __syncthreads();
    if (tid == 0) flags[(sweep + 1) & 1] = smax[(sweep + 1) & 1] = 0;
    __syncthreads();
    sweeps_done = sweep + 1;
    if (!anyr || worst < early_stop) break;
  }
  return sweeps_done;
}

template <int TS, int MPL, int MINB, bool CHOL = false, int SLOTS = 4, int BLK = 0>
__global__ void __launch_bounds__(BLK ? 288 : (MINB == 2 ? 576 : kJacobiMaxThreads), MINB)
    jacobi_qr_kernel(int64_t I1, int64_t I2, const float* __restrict__ A, JacobiOut o, int max_sweeps, int pitch,
                     unsigned long long* dbg) {
  if (o.skip && *o.skip) return;
  auto stamp = [&](int slot) {  // optional stage timeline of CTA 0 (%globaltimer ns)
    if (dbg && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long tns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
      dbg[slot] = tns;
    }
  };
  stamp(0);
  // per-CTA span and sweeps (dbg[16 + 3 b ..]): start, end of the sweeps, sweep count
  auto cta_stamp = [&](int slot, unsigned long long v) {
    if (dbg && threadIdx.x == 0) {
      if (slot < 2) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      dbg[16 + 3 * (int64_t)blockIdx.x + slot] = v;
    }
  };
  cta_stamp(0, 0);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const bool trans = I1 < I2;
  const int n = (int)(trans ? I1 : I2);
  const int m = CHOL ? n : (int)(trans ? I2 : I1);
  const int64_t b = blockIdx.x;
  const float* Ab = A + b * (CHOL ? (int64_t)n * n : I1 * I2);
  float* W = reinterpret_cast<float*>(smem_raw);  // n columns, pitch >= max(m, TS * MPL), even
  float* vhead = W + (size_t)n * pitch;           // v_k[0] of the reflectors
  float* beta = vhead + n;
  float* nrm = beta + n;                          // n + 1
  int* flags = reinterpret_cast<int*>(nrm + n + 1);
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
  constexpr int TR = TS * MPL;  // register-tile rows of X (rows n..TR-1 are zero)

  if (CHOL) {  // G is symmetric: row i of G is column i of W (16-byte copies when rows allow)
    if ((n & 3) == 0) {
      const int n4 = n >> 2;
      for (int l = tid; l < n * n4; l += nth) {
        const int i = l / n4, j4 = l - i * n4;
        *reinterpret_cast<float4*>(W + (size_t)i * pitch + 4 * j4) = reinterpret_cast<const float4*>(Ab)[l];
      }
    } else {
      for (int l = tid; l < n * n; l += nth) {
        const int i = l / n, j = l - i * n;
        W[(size_t)i * pitch + j] = Ab[l];
      }
    }
  } else if (!trans) {
    for (int l = tid; l < m * n; l += nth) {
      const int i = l / n, j = l - i * n;
      W[(size_t)j * pitch + i] = Ab[l];
    }
  } else {
    for (int l = tid; l < m * n; l += nth) {
      const int j = l / m, i = l - j * m;
      W[(size_t)j * pitch + i] = Ab[l];
    }
  }
  if (tid < 4) flags[tid] = 0;
  __syncthreads();
  stamp(1);
  // ||A||_F <= tau: nothing survives the threshold (sigma_max <= ||A||_F; trace(G) = ||A||_F^2)
  if (warp == 0) {
    float s2 = 0.f;
    if (CHOL) {
      for (int j = lane; j < n; j += 32) s2 += W[(size_t)j * pitch + j];
    } else {
      for (int l = lane; l < m * n; l += 32) {
        const int j = l / m, i = l - j * m;
        const float v = W[(size_t)j * pitch + i];
        s2 += v * v;
      }
    }
    s2 = warp_sum(s2);
    if (lane == 0) flags[3] = (o.tau > 0.0 && (double)s2 <= o.tau * o.tau) ? 1 : 0;
  }
  __syncthreads();
  if (flags[3]) {
    if (tid == 0) {
      if (o.kept_out) o.kept_out[b] = 0;
      if (o.stats) atomicAdd(&o.stats[0], 1ull);
    }
    // carry mode: an identity basis with unit sigma keeps the carried V unchanged
    if (o.v_out) {
      float* vy = reinterpret_cast<float*>(o.v_out) + b * (int64_t)n * n;
      for (int l = tid; l < n * n; l += nth) vy[l] = (l / n == l % n) ? 1.f : 0.f;
    }
    if (o.sv_out)
      for (int j = tid; j < n; j += nth) reinterpret_cast<float*>(o.sv_out)[b * n + j] = 1.f;
    if (o.d_out)
      for (int j = tid; j < n; j += nth) reinterpret_cast<float*>(o.d_out)[b * n + j] = 0.f;
    return;
  }

  stamp(2);
  if constexpr (!CHOL) {
  // ---- Householder QR: R on and above the diagonal, v_k below it (v_k[0] in vhead)
  for (int k = 0; k < n; ++k) {
    float* wk = W + (size_t)k * pitch;
    if (warp == 0) {
      float s2 = 0.f;
      for (int i = k + 1 + lane; i < m; i += 32) s2 += wk[i] * wk[i];
      s2 = warp_sum(s2);
      if (lane == 0) {
        const float x0 = wk[k];
        const float nx = sqrtf(x0 * x0 + s2);
        const float alpha = x0 >= 0.f ? -nx : nx;
        const float v0 = x0 - alpha;
        const float vv = v0 * v0 + s2;
        // a numerically zero column (vv below FLT_MIN: 2 / vv would overflow) is left alone
        const bool refl = vv >= FLT_MIN;
        beta[k] = refl ? 2.f / vv : 0.f;
        vhead[k] = v0;
        if (refl) wk[k] = alpha;
      }
    }
    __syncthreads();
    const float bk = beta[k], v0 = vhead[k];
    if (bk != 0.f) {
      for (int j = k + 1 + warp; j < n; j += nwarps) {
        float* wj = W + (size_t)j * pitch;
        float dot = (lane == 0) ? v0 * wj[k] : 0.f;
        for (int i = k + 1 + lane; i < m; i += 32) dot += wk[i] * wj[i];
        dot = warp_sum(dot) * bk;
        if (lane == 0) wj[k] -= dot * v0;
        for (int i = k + 1 + lane; i < m; i += 32) wj[i] -= dot * wk[i];
      }
    }
    __syncthreads();
  }
  stamp(3);
  // ---- X = R^T in place: R[i][j] (row i < column j, upper triangle) moves to column i,
  // row j (below the diagonal, where the reflector lived); then clear the upper triangle
  // and the rows n .. TR-1
  for (int l = tid; l < n * n; l += nth) {
    const int i = l / n, j = l - i * n;
    if (j > i) W[(size_t)i * pitch + j] = W[(size_t)j * pitch + i];
  }
  __syncthreads();
  for (int l = tid; l < n * TR; l += nth) {
    const int i = l / TR, j = l - i * TR;
    if (j < i || j >= n) W[(size_t)i * pitch + j] = 0.f;
  }
  __syncthreads();

  stamp(4);
  } else {
    // ---- Cholesky G = L L^T in place (column j of L in column j, rows >= j); a non-positive
    // pivot (rank-deficient slice) zeroes its column.  Blocked right-looking with panels of
    // CB = 16 columns, three block barriers per panel:
    //   (1) the CB x CB diagonal block is factored by warp 0 in registers (lane r holds row r,
    //       pivots and multipliers by shuffles: no shared-memory round trips on the n-step
    //       critical path);
    //   (2) the panel rows below it are solved against it (L21 = A21 L11^-T), one thread per
    //       row with the row in registers and L11 broadcast from shared memory;
    //   (3) the trailing update A22 -= L21 L21^T in 4 x 4 register tiles (two 16-byte loads
    //       per 16 FMAs), lower-triangle tiles only.
    // (The previous warp-0 panel with per-column update passes took ~140 us of a ~640 us
    // config-3 slice, latency- and shared-memory-bound.)  pitch is a multiple of 4.
    constexpr int CB = 16;
    float* dinv = vhead;  // 1 / L[k][k] (0 for a zeroed column)
    for (int k0 = 0; k0 < n; k0 += CB) {
      const int nb = min(CB, n - k0);
      if (warp == 0) {
        float a[CB];
        const int r = lane;
#pragma unroll
        for (int c = 0; c < CB; ++c) a[c] = (r < nb && c <= r) ? W[(size_t)(k0 + c) * pitch + k0 + r] : 0.f;
        // (every loop fully unrolled with compile-time indices: a[] stays in registers)
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          const float pk = __shfl_sync(0xffffffffu, a[c], c);
          const float d = pk >= FLT_MIN ? sqrtf(pk) : 0.f;
          const float inv = d > 0.f ? 1.f / d : 0.f;
          a[c] = r == c ? d : (r > c ? a[c] * inv : a[c]);
          if (r == c && c < nb) dinv[k0 + c] = inv;
#pragma unroll
          for (int jj = 0; jj < CB; ++jj) {
            if (jj > c) {
              const float ljc = __shfl_sync(0xffffffffu, a[c], jj);
              a[jj] = r >= jj ? fmaf(-a[c], ljc, a[jj]) : a[jj];
            }
          }
        }
        if (r < nb) {
#pragma unroll
          for (int c = 0; c < CB; ++c)
            if (c <= r) W[(size_t)(k0 + c) * pitch + k0 + r] = a[c];
        }
      }
      __syncthreads();
      if (k0 == 0) stamp(8);
      const int s0 = k0 + nb;
      if (s0 >= n) break;
      for (int i = s0 + tid; i < n; i += nth) {  // (2) rows below the diagonal block
        float a[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) a[c] = c < nb ? W[(size_t)(k0 + c) * pitch + i] : 0.f;
        const float* l11 = W + (size_t)k0 * pitch + k0;
#pragma unroll
        for (int c = 0; c < CB; ++c) {
          a[c] *= c < nb ? dinv[k0 + c] : 0.f;
#pragma unroll
          for (int jj = 0; jj < CB; ++jj)
            if (jj > c) a[jj] = fmaf(-a[c], jj < nb ? l11[(size_t)c * pitch + jj] : 0.f, a[jj]);
        }
#pragma unroll
        for (int c = 0; c < CB; ++c)
          if (c < nb) W[(size_t)(k0 + c) * pitch + i] = a[c];
      }
      __syncthreads();
      if (k0 == 0) stamp(9);
      // (3) A22[j][i] -= sum_c L[i][c] L[j][c], s0 <= j <= i < n, 4 x 4 tiles (bi >= bj)
      const int T = (n - s0 + 3) >> 2;
      const float* lp = W + (size_t)k0 * pitch;
      for (int l = tid; l < T * (T + 1) / 2; l += nth) {
        int bi = (int)((sqrtf(8.f * (float)l + 1.f) - 1.f) * 0.5f);
        while (bi * (bi + 1) / 2 > l) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= l) ++bi;
        const int bj = l - bi * (bi + 1) / 2;
        const int i0 = s0 + 4 * bi, j0 = s0 + 4 * bj;
        float acc[4][4];
        const bool full = i0 + 3 < n;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const float* wj = W + (size_t)min(j0 + jj, n - 1) * pitch + i0;
          if (full) {
            const float4 v = *reinterpret_cast<const float4*>(wj);
            acc[jj][0] = v.x, acc[jj][1] = v.y, acc[jj][2] = v.z, acc[jj][3] = v.w;
          } else {
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) acc[jj][ii] = i0 + ii < n ? wj[ii] : 0.f;
          }
        }
#pragma unroll 4
        for (int c = 0; c < nb; ++c) {
          const float* lc = lp + (size_t)c * pitch;
          float li[4], lj[4];
          if (full) {
            const float4 v = *reinterpret_cast<const float4*>(lc + i0);
            li[0] = v.x, li[1] = v.y, li[2] = v.z, li[3] = v.w;
          } else {
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) li[ii] = i0 + ii < n ? lc[i0 + ii] : 0.f;
          }
          const float4 u = *reinterpret_cast<const float4*>(lc + j0);  // j0 + 3 <= i0 + 3 < pitch
          lj[0] = u.x, lj[1] = u.y, lj[2] = u.z, lj[3] = u.w;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) acc[jj][ii] = fmaf(-li[ii], lj[jj], acc[jj][ii]);
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          if (j0 + jj >= n) break;
          float* wj = W + (size_t)(j0 + jj) * pitch + i0;
          if (full) {
            *reinterpret_cast<float4*>(wj) = make_float4(acc[jj][0], acc[jj][1], acc[jj][2], acc[jj][3]);
          } else {
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
              if (i0 + ii < n) wj[ii] = acc[jj][ii];
          }
        }
      }
      __syncthreads();
      if (k0 == 0) stamp(10);
      if (k0 == 64) stamp(11);
    }
    // X = L: clear the upper triangle and the rows n .. TR-1
    stamp(3);
    for (int l = tid; l < n * TR; l += nth) {
      const int c = l / TR, r = l - c * TR;
      if (r < c || r >= n) W[(size_t)c * pitch + r] = 0.f;
    }
    __syncthreads();
    stamp(4);
  }

  // ---- one-sided Jacobi on the n columns of X (n rows), as jacobi_kernel's fp32 path
  const float tol = FLT_EPSILON * sqrtf((float)max(n, 1)) * o.tol_scale;
  const int npl = n + (n & 1);
  const int npairs = npl / 2;
  constexpr int TPW = 32 / TS;
  const int tl = lane % TS;
  const int team = lane / TS;
  int sweeps_done = 0;
  // circle-method slots of this thread's team: slot t handles pair k = base_t + team; the
  // pair of round r is p = (r + k) mod m1, q = (r - k) mod m1 (k = 0: p = m1, q = r), so
  // both advance by one per round and no index arithmetic is redone per pass
  const int m1 = npl - 1;
  const int stride = nwarps * TPW;
  const int nslot = (npairs + stride - 1) / stride;  // <= 4 for every launched shape
  const float* const Wc = W + 2 * tl;
  int* smax = flags + 4;  // per-sweep-parity largest relative rotated |gamma| (float bits; rank_sh later)
  if (tid == 0) smax[0] = smax[1] = 0;
  if constexpr (BLK == 4) {
    sweeps_done = jacobi_block4_sweeps<MPL>(W, pitch, n, nrm, flags, smax, tol, max_sweeps, o.early_stop);
  } else if constexpr (BLK == 2) {
    sweeps_done = jacobi_block_sweeps<MPL>(W, pitch, n, nrm, flags, smax, tol, max_sweeps, o.early_stop);
  } else {
  for (int sweep = 0; sweep < max_sweeps && n > 1; ++sweep) {
    int* rot = &flags[sweep & 1];
    for (int j = warp; j < n; j += nwarps) {
      const float* wj = W + (size_t)j * pitch;
      float s2 = 0.f;
      for (int i = lane; i < n; i += 32) s2 += wj[i] * wj[i];
      s2 = warp_sum(s2);
      if (lane == 0) nrm[j] = s2;
    }
    __syncthreads();
    int ps[SLOTS], qs[SLOTS];
#pragma unroll
    for (int t = 0; t < SLOTS; ++t) {
      const int k = warp * TPW + t * stride + team;
      ps[t] = (k == 0) ? m1 : k;
      qs[t] = (k == 0) ? 0 : m1 - k;
    }
    for (int r = 0; r < m1; ++r) {
#pragma unroll
      for (int t = 0; t < SLOTS; ++t) {
        if (t >= nslot) break;
        const int k = warp * TPW + t * stride + team;
        const int p = ps[t], q = qs[t];
        ps[t] = (k == 0) ? m1 : (p + 1 == m1 ? 0 : p + 1);
        qs[t] = (q + 1 == m1) ? 0 : q + 1;
        const bool active = k < npairs && p < n && q < n;
        float* wp = const_cast<float*>(Wc) + (size_t)(active ? p : 0) * pitch;
        float* wq = const_cast<float*>(Wc) + (size_t)(active ? q : 0) * pitch;
        float2 X2[MPL / 2], Y2[MPL / 2];
        float2 acc[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int h = 0; h < MPL / 2; ++h) {
          X2[h] = *reinterpret_cast<const float2*>(wp + 2 * TS * h);
          Y2[h] = *reinterpret_cast<const float2*>(wq + 2 * TS * h);
          acc[h % 3] = __ffma2_rn(X2[h], Y2[h], acc[h % 3]);  // three chains (FFMA2 latency)
        }
        float g = ((acc[0].x + acc[1].x) + acc[2].x) + ((acc[0].y + acc[1].y) + acc[2].y);
#pragma unroll
        for (int off = TS / 2; off > 0; off >>= 1) g += __shfl_xor_sync(0xffffffffu, g, off);
        const float al = active ? nrm[p] : 0.f;
        const float be = active ? nrm[q] : 0.f;
        const float gabs = fabsf(g);
        const float sab = sqrt_apx(al) * sqrt_apx(be);
        if (!active || !(gabs > tol * sab) || !(fminf(fminf(al, be), gabs) >= FLT_MIN)) continue;
        const float zeta = (be - al) * (0.5f * rcp_apx(gabs));
        const float az = fabsf(zeta);
        const float den = az < 1e18f ? az + sqrt_apx(fmaf(az, az, 1.f)) : 2.f * az;
        const float tt = copysignf(rcp_apx(den), zeta);
        const float x1 = fmaf(tt, tt, 1.f);
        float c = rsqrt_apx(x1);
        c = c * fmaf(-0.5f * x1 * c, c, 1.5f);
        const float sn = c * tt;
        const float sg = g >= 0.f ? 1.f : -1.f;
        const float2 C2 = make_float2(c, c), S2 = make_float2(sn, sn);
        const float2 NSQ = make_float2(-sn * sg, -sn * sg), CQ = make_float2(c * sg, c * sg);
#pragma unroll
        for (int h = 0; h < MPL / 2; ++h) {
          *reinterpret_cast<float2*>(wp + 2 * TS * h) = __ffma2_rn(C2, X2[h], __fmul2_rn(NSQ, Y2[h]));
          *reinterpret_cast<float2*>(wq + 2 * TS * h) = __ffma2_rn(S2, X2[h], __fmul2_rn(CQ, Y2[h]));
        }
        if (tl == 0) {
          nrm[p] = fmaxf(al - tt * gabs, 0.f);
          nrm[q] = be + tt * gabs;
          *rot = 1;
          atomicMax(&smax[sweep & 1], __float_as_int(gabs * rcp_apx(sab)));
        }
      }
      __syncthreads();
    }
    const int any = *rot;
    const float worst = __int_as_float(smax[sweep & 1]);
    __syncthreads();
    if (tid == 0) flags[(sweep + 1) & 1] = smax[(sweep + 1) & 1] = 0;
    __syncthreads();
    sweeps_done = sweep + 1;
    // without rotations the sweep changed nothing; when every rotation of the sweep had a
    // relative inner product below early_stop, the inner products the later rotations
    // disturbed are of order early_stop^2 between columns of distinct norms (quadratic
    // convergence); between columns of nearly equal norms a rotation can be wide, but
    // there the singular values, and so the SVT's shrink factors, nearly coincide
    if (!any || worst < o.early_stop) break;
  }
  }
  stamp(5);
  cta_stamp(1, 0);
  cta_stamp(2, (unsigned long long)sweeps_done);
  if (o.stats && tid == 0) {
    atomicAdd(&o.stats[0], 1ull);
    atomicAdd(&o.stats[1], (unsigned long long)sweeps_done);
    atomicMax(&o.stats[2], (unsigned long long)sweeps_done);  // the launch waits for its slowest slice
  }
  // ---- singular values, descending ranks, scaled columns y~_j
  float* sig = nrm;
  for (int j = warp; j < n; j += nwarps) {
    const float* wj = W + (size_t)j * pitch;
    float s2 = 0.f;
    for (int i = lane; i < n; i += 32) s2 += wj[i] * wj[i];
    s2 = warp_sum(s2);
    if (lane == 0) sig[j] = sqrtf(s2);
  }
  if (tid == 0) flags[2] = 0;
  __syncthreads();
  int* rank_sh = flags + 4;
  float* scale = beta;  // reuse: per-column output scale
  int kept_local = 0;
  for (int j = tid; j < n; j += nth) {
    const float sj = sig[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const float si = sig[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    rank_sh[j] = rank;
    if (o.sv_out) reinterpret_cast<float*>(o.sv_out)[b * n + rank] = sj;
    const bool keep = sj > (float)o.tau && sj > 0.f;
    kept_local += keep;
    scale[j] = keep ? sqrtf((sj - (float)o.tau) / sj) / sj : 0.f;
    // carry mode: sqrt((sigma - tau)_+ / sigma), the weight of v_j in svt = G V diag(.) V^T
    if (o.d_out) reinterpret_cast<float*>(o.d_out)[b * n + rank] = keep ? sqrtf((sj - (float)o.tau) / sj) : 0.f;
  }
  if (kept_local) atomicAdd(&flags[2], kept_local);
  __syncthreads();
  if (o.kept_out && tid == 0) o.kept_out[b] = flags[2];
  if (o.v_out) {  // carry mode: the unscaled Jacobi columns y_j = sigma_j v_j, sorted
    float* vy = reinterpret_cast<float*>(o.v_out) + b * (int64_t)n * n;
    for (int l = tid; l < n * n; l += nth) {
      const int j = l / n, i = l - j * n;
      vy[(int64_t)rank_sh[j] * n + i] = W[(size_t)j * pitch + i];
    }
  }
  if (!o.w_out) return;
  float* dst = reinterpret_cast<float*>(o.w_out) + b * (int64_t)n * n;
  for (int l = tid; l < n * n; l += nth) {
    const int j = l / n, i = l - j * n;
    dst[(int64_t)rank_sh[j] * n + i] = W[(size_t)j * pitch + i] * scale[j];
  }
}


size_t jacobi_qr_smem(int n, int pitch) { return ((size_t)n * pitch + 4 * (size_t)n + 1) * 4 + (n + 8) * 4 + 16; }

template <int TS, int MPL, int MINB, bool CHOL>
int launch_qr_variant(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* A, const JacobiOut& o,
                      int max_sweeps, int n, int pitch) {
  const size_t smem = jacobi_qr_smem(n, pitch);
  const int pairs = std::max(1, (n + 1) / 2);
  const int maxw = MINB == 2 ? 18 : 32;
  const int teams = std::max(1, (pairs * TS + 31) / 32);
  const int per_warp = (teams + maxw - 1) / maxw;
  const int nwarps = std::max(1, (teams + per_warp - 1) / per_warp);
  const int slots = (pairs + nwarps * (32 / TS) - 1) / (nwarps * (32 / TS));
  if (slots > 4) return LTB_EUNSUPPORTED;  // <= 4 slots per team
  auto kern = slots == 1 ? jacobi_qr_kernel<TS, MPL, MINB, CHOL, 1> : jacobi_qr_kernel<TS, MPL, MINB, CHOL, 4>;
  LTB_TRY(ensure_smem(ctx, kern, smem, true));
  kern<<<(unsigned)batch, 32 * nwarps, smem, ctx->stream>>>(I1, I2, A, o, max_sweeps, pitch, ctx->opt_qr_timeline);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

// the block-pair Jacobi variant (warm Cholesky path): 2 n threads, two CTAs per SM
template <int MPL, int BLK>
int launch_qr_blk(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* A, const JacobiOut& o,
                  int max_sweeps, int n, int pitch) {
  const size_t smem = jacobi_qr_smem(n, pitch);
  auto kern = jacobi_qr_kernel<BLK == 4 ? 16 : 8, MPL, 2, true, 1, BLK>;
  LTB_TRY(ensure_smem(ctx, kern, smem, true));
  kern<<<(unsigned)batch, 2 * n, smem, ctx->stream>>>(I1, I2, A, o, max_sweeps, pitch, ctx->opt_qr_timeline);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

// 1 when the QR-preconditioned resident kernel takes this fp32 SVT; 0 to use the others
constexpr int g_svt_qr = 1;
constexpr int g_qr_max_sweeps = 40;  // timing hook: 0 measures the QR and emission stages alone
// lanes per column pair in the fp32 QR/Cholesky Jacobi: 8 (one pair per team per round,
// fewer padding rows; 10-30% faster for 64 <= n <= 192, tools/qr_ts_ab.py) or 16
constexpr int g_qr_ts = 8;

// LTB_EUNSUPPORTED when the shape does not fit the QR-preconditioned kernel
// chol: A holds n x n Gram matrices (I1 == I2 == n), factored by Cholesky instead of Householder
int launch_jacobi_qr(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* A, const JacobiOut& o_in,
                     bool chol = false) {
  const int m = (int)std::max(I1, I2), n = (int)std::min(I1, I2);
  if (!g_svt_qr || ctx->opt_force_blocked || n < 32 || batch > 0x7fffffff) return LTB_EUNSUPPORTED;
  JacobiOut o = o_in;
  // cold calls too: stop after a sweep whose rotations all had relative inner products
  // below sqrt(tol) (see jacobi_qr_kernel; tol = the rotation threshold)
  if (o.early_stop == 0.f && g_qr_early > 0.f)
    o.early_stop = g_qr_early * sqrtf(FLT_EPSILON * sqrtf((float)n) * o.tol_scale);
  int TSv = 16, MPLv = 0;
  if (g_qr_ts == 8 && n > 48 && n <= 192) {  // 8-lane teams: one pair per team per round
    TSv = 8;
    MPLv = n <= 64 ? 8 : n <= 128 ? 16 : n <= 144 ? 18 : n <= 160 ? 20 : 24;
  } else if (n <= 64) MPLv = 4;
  else if (n <= 128) MPLv = 8;
  else if (n <= 160) MPLv = 10;
  else if (n <= 192) MPLv = 12;
  else if (n <= 256) { TSv = 32; MPLv = 8; }
  else return LTB_EUNSUPPORTED;
  int pitch = std::max(m, TSv * MPLv);
  pitch += pitch & 1;
  if (chol) pitch = (pitch + 3) & ~3;  // the Cholesky's 16-byte tile accesses
  // an 8-lane team reads 64 bytes of its column: with pitch = 16 (mod 32) floats the four
  // teams of a warp (consecutive columns) alternate bank halves instead of colliding
  if (TSv == 8) pitch += (16 - pitch % 32 + 32) % 32;
  const size_t smem = jacobi_qr_smem(n, pitch);
  if (smem > kSmemLimit) return LTB_EUNSUPPORTED;
  const bool two = 2 * (smem + 1024) <= 228 * 1024;
  const int ms = g_qr_max_sweeps;
  // warm Cholesky path: the block-pair Jacobi (n / 4 teams of 8 lanes, 2 n <= 288 threads)
  if (chol && TSv == 8 && n % 4 == 0 && 2 * n <= 288 && ctx->opt_jacobi_pairs != 1) {
    // pitch = 8 (mod 16) floats: the four teams of a warp read columns 2P (or 2P + 1) of
    // consecutive blocks P, whose 64-byte chunks then alternate bank halves (with pitch = 16
    // (mod 32) every even column starts in the same half: 4-way instead of 2-way wavefronts)
    const int base = std::max(m, TSv * MPLv);
    if (n % 16 == 0 && ctx->opt_jacobi_pairs == 3) {  // four-column blocks (measured slower: spills at 96 registers)
      const int bpitch4 = base + ((4 - base) % 8 + 8) % 8;  // 4 (mod 8)
      const size_t bsm4 = jacobi_qr_smem(n, bpitch4);
      if (2 * (bsm4 + 1024) <= 228 * 1024) {
        if (n == 128) return launch_qr_blk<8, 4>(ctx, batch, I1, I2, A, o, ms, n, bpitch4);
        if (n == 144) return launch_qr_blk<9, 4>(ctx, batch, I1, I2, A, o, ms, n, bpitch4);
      }
    }
    const int bpitch = base + ((8 - base) % 16 + 16) % 16;
    const size_t bsm = jacobi_qr_smem(n, bpitch);
    if (2 * (bsm + 1024) <= 228 * 1024) {
      if (MPLv == 16) return launch_qr_blk<16, 2>(ctx, batch, I1, I2, A, o, ms, n, bpitch);
      if (MPLv == 18) return launch_qr_blk<18, 2>(ctx, batch, I1, I2, A, o, ms, n, bpitch);
    }
  }
#define LTB_QR(TS_, MPL_)                                                                              \
  if (chol)                                                                                              \
    return two ? launch_qr_variant<TS_, MPL_, 2, true>(ctx, batch, I1, I2, A, o, ms, n, pitch)          \
               : launch_qr_variant<TS_, MPL_, 1, true>(ctx, batch, I1, I2, A, o, ms, n, pitch);         \
  return two ? launch_qr_variant<TS_, MPL_, 2, false>(ctx, batch, I1, I2, A, o, ms, n, pitch)           \
             : launch_qr_variant<TS_, MPL_, 1, false>(ctx, batch, I1, I2, A, o, ms, n, pitch)
  if (TSv == 32) { LTB_QR(32, 8); }
  if (TSv == 8) {
    switch (MPLv) {
      case 8: LTB_QR(8, 8);
      case 16: LTB_QR(8, 16);
      case 18: LTB_QR(8, 18);
      case 20: LTB_QR(8, 20);
      default: LTB_QR(8, 24);
    }
  }
  switch (MPLv) {
    case 4: LTB_QR(16, 4);
    case 8: LTB_QR(16, 8);
    case 10: LTB_QR(16, 10);
    default: LTB_QR(16, 12);
  }
#undef LTB_QR
}

// ---------------------------------------------------------------- SVT with a carried right basis
// Inside PGA the iterates change slowly, so the right singular vectors V of
// one iteration's slices precondition the next: the QR-preconditioned Jacobi
// runs on A0 = G V_prev (G^T V_prev oriented), whose columns are already
// nearly orthogonal, and converges in a few sweeps.  With V = V_prev V_A0
// (V_A0 from the normalised Jacobi columns, completed to an orthonormal basis)
//   svt(G) = G V diag((s - tau)_+ / s) V^T          (I1 >= I2)
//   svt(G) = V diag((s - tau)_+ / s) V^T G          (I1 <  I2, V of G^T)
// V is re-orthonormalised by one Newton-Schulz step, V <- V (3I - V^T V) / 2,
// every call, so rounding does not accumulate across iterations.
// one slice per blockIdx.y, 32-bit index math within the slice (the 64-bit divisions of a
// flat index made these HBM passes run at a third of the bandwidth)
__global__ void ns_combine_kernel(int n, const float* __restrict__ S, float* __restrict__ M, const int* skip) {
  if (skip && *skip) return;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    M[off + l] = (l - i * n == i ? 1.5f : 0.f) - 0.5f * S[off + l];
  }
}

__global__ void col_scale_kernel(int n, const float* __restrict__ V, const float* __restrict__ d, float* __restrict__ T,
                                 const int* skip) {
  if (skip && *skip) return;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  const float* db = d + (int64_t)blockIdx.y * n;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    T[off + l] = V[off + l] * db[l - i * n];
  }
}

}  // namespace

// fp32 SVT of `batch` I1 x I2 slices carrying the n x n right bases V (row-major,
// n = min(I1, I2)) between calls; warm == 0 starts from the identity.
// LTB_EUNSUPPORTED when the slice shape does not fit the QR-preconditioned kernel.
constexpr int g_carry_chol = 1;  // warm carried SVT: Cholesky of the Gram matrix (1) or Householder (0)
// carried SVT: multiplier of the Jacobi rotation threshold eps * sqrt(n)
constexpr float g_carry_tol_scale = 1.f;
// warm carried SVT: stop the Jacobi after a sweep whose rotated pairs all had a relative
// inner product below g_carry_early * sqrt(tol) (tol = the rotation threshold), i.e. the
// inner products left behind are ~tol; 0 runs to a sweep without rotations.  Config-3 PGA
// (tools/pga_early_ab.py): 2.77 -> 1.98 sweeps per slice, +13% it/s, the 200-iteration
// iterate's error against the fp64 run unchanged (3.2e-5)
constexpr float g_carry_early = 1.f;

namespace {
// One batch of the carried fp32 SVT in three phases, so that two batches can be interleaved
// on different streams (see ltb_svt_carry_impl): pre (A0 = G V, Gram matrix), the Jacobi, post
// (basis update, Newton-Schulz, recomposition).  Each phase launches on ctx->stream.
struct CarryPart {
  int64_t batch, I1, I2, m, n, nn;
  bool trans;
  const float* G;
  float *out, *V;
  int warm;
  const int* skip;
  double tau;
  void* ws[8] = {};
  int nws = 0;
  float *A0 = nullptr, *Y = nullptr, *sv = nullptr, *dd = nullptr, *VR = nullptr, *Vn = nullptr, *S = nullptr;
  int* kept = nullptr;
  CarryPart(int64_t b, int64_t i1, int64_t i2, const float* g, double t, float* o, float* v, int w, const int* sk)
      : batch(b), I1(i1), I2(i2), G(g), out(o), V(v), warm(w), skip(sk), tau(t) {
    trans = I1 < I2;
    m = trans ? I2 : I1;
    n = trans ? I1 : I2;
    nn = n * n;
  }
  template <typename T> int alloc(ltb_ctx* ctx, size_t bytes, T** p) {
    void* q = nullptr;
    LTB_TRY(ltb_ws_alloc(ctx, bytes, &q));
    ws[nws++] = q;
    *p = (T*)q;
    return LTB_OK;
  }
  void release(ltb_ctx* ctx) {  // stream-ordered on ctx->stream (the phase that used them last)
    while (nws > 0) ltb_ws_free(ctx, ws[--nws]);
  }
  int allocate(ltb_ctx* ctx) {
    LTB_TRY(alloc(ctx, sizeof(float) * batch * n * m, &A0));
    LTB_TRY(alloc(ctx, sizeof(float) * batch * nn, &Y));
    LTB_TRY(alloc(ctx, sizeof(float) * batch * n, &sv));
    LTB_TRY(alloc(ctx, sizeof(float) * batch * n, &dd));
    LTB_TRY(alloc(ctx, sizeof(float) * batch * nn, &VR));
    LTB_TRY(alloc(ctx, sizeof(float) * batch * nn, &Vn));
    LTB_TRY(alloc(ctx, sizeof(float) * batch * nn, &S));
    LTB_TRY(alloc(ctx, sizeof(int) * batch, &kept));
    return LTB_OK;
  }
  int pre(ltb_ctx* ctx) {
    const int F = LTB_F32;
    if (!warm) return LTB_OK;
    // A0 = V^T G (I1 < I2) or G V: the preconditioned slices, same shape as G
    if (trans)
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, m, n, LTB_OP_T, V, n, nn, LTB_OP_N, G, m, n * m, A0, m, n * m, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
    else
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, m, n, n, LTB_OP_N, G, n, m * n, LTB_OP_N, V, n, nn, A0, n, m * n, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
    if (g_carry_chol) {
      // A0's columns are nearly orthogonal: factor its Gram matrix (tensor-core GEMM) by
      // Cholesky instead of a Householder QR of A0
      if (trans)  // oriented W = A0^T: G = A0 A0^T
        LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, m, LTB_OP_N, A0, m, n * m, LTB_OP_T, A0, m, n * m, S, n, nn,
                              nullptr, nullptr, nullptr, nullptr, nullptr, skip));
      else  // W = A0: G = A0^T A0
        LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, m, LTB_OP_T, A0, n, m * n, LTB_OP_N, A0, n, m * n, S, n, nn,
                              nullptr, nullptr, nullptr, nullptr, nullptr, skip));
    }
    return LTB_OK;
  }
  int jacobi(ltb_ctx* ctx) {
    JacobiOut o{nullptr, sv, Y, kept, dd, tau, skip};
    o.stats = ctx->d_stats;
    o.tol_scale = g_carry_tol_scale;
    if (warm) o.early_stop = g_carry_early * sqrtf(FLT_EPSILON * sqrtf((float)n) * g_carry_tol_scale);
    if (warm && g_carry_chol) return launch_jacobi_qr(ctx, batch, n, n, S, o, true);
    return launch_jacobi_qr(ctx, batch, I1, I2, warm ? A0 : G, o);
  }
  int post(ltb_ctx* ctx) {
    const int F = LTB_F32;
    // V_A0: normalised Jacobi columns completed to an orthonormal basis (row-major, column j = v_j)
    LTB_TRY(ensure_smem(ctx, complete_u_kernel<float>, (size_t)n * sizeof(float)));
    complete_u_kernel<float><<<(unsigned)batch, 256, (size_t)n * sizeof(float), ctx->stream>>>((int)n, (int)n, Y, sv,
                                                                                                VR, 1);
    LTB_LAUNCH_CHECK(ctx);
    const float* Vc = VR;  // V_prev V_A0
    if (warm) {
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_N, V, n, nn, LTB_OP_N, VR, n, nn, Vn, n, nn, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
      Vc = Vn;
    }
    // Newton-Schulz: V = Vc (3I - Vc^T Vc) / 2, every call: without it the basis drifts from
    // orthonormality by about one fp32 rounding per call, and the 200-iteration config-3
    // iterate leaves the fp32 tolerance (measured error vs fp64: 3.2e-5 every call, 5.0e-5
    // every 2nd, 2.1e-4 every 4th)
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_T, Vc, n, nn, LTB_OP_N, Vc, n, nn, S, n, nn, nullptr, nullptr,
                          nullptr, nullptr, nullptr, skip));
    const dim3 grid((unsigned)std::min<int64_t>((nn + 1023) / 1024, 64), (unsigned)batch);
    ns_combine_kernel<<<grid, 256, 0, ctx->stream>>>((int)n, S, Y, skip);  // Y reused as M
    LTB_LAUNCH_CHECK(ctx);
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_N, Vc, n, nn, LTB_OP_N, Y, n, nn, V, n, nn, nullptr, nullptr,
                          nullptr, nullptr, nullptr, skip));
    // T = V diag(sqrt((s - tau)_+ / s)),  Z = T T^T (K limited to the kept count),  out
    col_scale_kernel<<<grid, 256, 0, ctx->stream>>>((int)n, V, dd, VR, skip);  // VR reused as T
    LTB_LAUNCH_CHECK(ctx);
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_N, VR, n, nn, LTB_OP_T, VR, n, nn, S, n, nn, nullptr, nullptr,
                          kept, nullptr, nullptr, skip));
    if (trans)
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, m, n, LTB_OP_N, S, n, nn, LTB_OP_N, G, m, n * m, out, m, n * m, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
    else
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, m, n, n, LTB_OP_N, G, n, m * n, LTB_OP_N, S, n, nn, out, n, m * n, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
    return LTB_OK;
  }
};

int carry_checks(int64_t batch, int64_t I1, int64_t I2) {
  const int64_t n = std::min(I1, I2);
  return (batch <= 0 || batch > 65535 || n < 32) ? LTB_EUNSUPPORTED : LTB_OK;  // grid.y carries the slice
}

// RAII: restores ctx->stream and releases the events on every return path
struct StreamSwap {
  ltb_ctx* ctx;
  cudaStream_t main;
  cudaEvent_t ev[6] = {};
  explicit StreamSwap(ltb_ctx* c) : ctx(c), main(c->stream) {}
  ~StreamSwap() {
    ctx->stream = main;
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  }
};
}  // namespace

// The warm Jacobi runs one slice per CTA, two CTAs per SM: a batch just above a multiple of the
// 2 x SMs slots (config 3: 300 slices on 296) leaves a few slices for a second wave, during
// which the rest of the GPU idles (the launch took about twice a slice's latency).  Every
// slice's chain (A0 / Gram GEMMs, Jacobi, basis update, recomposition) is independent, so the
// batch is split into the whole waves (big) and the remainder (small):
//   small pre   (low-priority stream)  -- runs beside big pre
//   big pre     (high priority)        -> event E
//   small Jacobi (low priority, waits E): pending beside the big Jacobi, so the block
//                scheduler dispatches the big one's CTAs first and the small one's into the
//                slots the first finished CTAs free
//   big Jacobi, big post (high priority): the post GEMMs run on the SMs the big Jacobi frees
//   small post  (a second high-priority stream, after the small Jacobi)
constexpr int g_carry_split = 1;

int ltb_svt_carry_impl(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const float* G, double tau, float* out,
                       float* V, int warm, const int* skip) {
  LTB_TRY(carry_checks(batch, I1, I2));
  const int64_t slots = 2 * (int64_t)ctx->num_sms;
  const int64_t whole = batch / slots * slots, rest = batch - whole;
  if (!(g_carry_split && warm && whole > 0 && rest > 0 && rest * 8 <= slots)) {
    CarryPart p(batch, I1, I2, G, tau, out, V, warm, skip);
    int st = p.allocate(ctx);
    if (st == LTB_OK) st = p.pre(ctx);
    if (st == LTB_OK) st = p.jacobi(ctx);
    if (st == LTB_OK) st = p.post(ctx);
    p.release(ctx);
    return st;
  }
  if (!ctx->split_hi) {
    int lo = 0, hi = 0;
    LTB_CUDA_TRY(ctx, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    LTB_CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->split_hi, cudaStreamNonBlocking, hi));
    LTB_CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->split_hi2, cudaStreamNonBlocking, hi));
    LTB_CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->split_lo, cudaStreamNonBlocking, lo));
  }
  const int64_t n = std::min(I1, I2), S = I1 * I2;
  StreamSwap sw(ctx);
  for (cudaEvent_t& e : sw.ev) LTB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t fork = sw.ev[0], e_pre = sw.ev[1], e_small_jac = sw.ev[2], j_big = sw.ev[3], j_small = sw.ev[4];
  // the workspace is allocated and (after the join) released on the caller's stream, so the
  // stream-ordered pool reuses it from call to call as in the unsplit case
  CarryPart big(whole, I1, I2, G, tau, out, V, warm, skip);
  CarryPart small(rest, I1, I2, G + whole * S, tau, out + whole * S, V + whole * n * n, warm, skip);
  struct Release {
    ltb_ctx* ctx;
    CarryPart *a, *b;
    cudaStream_t main;
    ~Release() {
      const cudaStream_t cur = ctx->stream;
      ctx->stream = main;
      a->release(ctx);
      b->release(ctx);
      ctx->stream = cur;
    }
  } rel{ctx, &big, &small, sw.main};
  LTB_TRY(big.allocate(ctx));
  LTB_TRY(small.allocate(ctx));
  LTB_CUDA_TRY(ctx, cudaEventRecord(fork, sw.main));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->split_hi, fork, 0));
  LTB_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->split_lo, fork, 0));
  int st = LTB_OK;
  ctx->stream = ctx->split_lo;
  if (st == LTB_OK) st = small.pre(ctx);
  ctx->stream = ctx->split_hi;
  if (st == LTB_OK) st = big.pre(ctx);
  if (st == LTB_OK) st = cudaEventRecord(e_pre, ctx->split_hi) == cudaSuccess ? LTB_OK : LTB_ECUDA;
  ctx->stream = ctx->split_lo;
  if (st == LTB_OK) st = cudaStreamWaitEvent(ctx->split_lo, e_pre, 0) == cudaSuccess ? LTB_OK : LTB_ECUDA;
  if (st == LTB_OK) st = small.jacobi(ctx);
  if (st == LTB_OK) st = cudaEventRecord(e_small_jac, ctx->split_lo) == cudaSuccess ? LTB_OK : LTB_ECUDA;
  ctx->stream = ctx->split_hi;
  if (st == LTB_OK) st = big.jacobi(ctx);
  if (st == LTB_OK) st = big.post(ctx);
  ctx->stream = ctx->split_hi2;
  if (st == LTB_OK) st = cudaStreamWaitEvent(ctx->split_hi2, e_small_jac, 0) == cudaSuccess ? LTB_OK : LTB_ECUDA;
  if (st == LTB_OK) st = small.post(ctx);
  // join every stream into the caller's (also on failure: nothing may outlive the call, and
  // the workspace is released behind all of it)
  cudaEventRecord(j_big, ctx->split_hi);
  cudaEventRecord(j_small, ctx->split_hi2);
  cudaEventRecord(sw.ev[5], ctx->split_lo);
  cudaStreamWaitEvent(sw.main, j_big, 0);
  cudaStreamWaitEvent(sw.main, j_small, 0);
  cudaStreamWaitEvent(sw.main, sw.ev[5], 0);
  if (st == LTB_ECUDA) return ltb_set_error(ctx, LTB_ECUDA, "carried SVT: stream ordering failed");
  return st;
}

// fp64 SVT carrying the slices' right bases V (n x n row-major, n = min(I1, I2)) between
// PGA iterations, as ltb_svt_carry_impl does in fp32 but without the QR / Cholesky stage:
// the resident Jacobi (accumulating its rotations J) runs on A0 = G V (V^T G when I1 < I2),
// whose columns are nearly orthogonal, so it needs a few sweeps instead of a dozen; its
// columns w_j = sigma_j u_j are those of G itself (V J is orthogonal), so the usual V-free
// recomposition with G applies unchanged, and V <- V J for the next call (rounding drift
// ~1e-16 per call in fp64: no re-orthonormalisation).  warm == 0: A0 = G, V <- J.
constexpr int g_carry64_early = 1;  // the sqrt(tol) early stop for warm fp64 carried SVTs

namespace {
__global__ void inv_sq64_kernel(int64_t total, const double* __restrict__ sv, double* __restrict__ r, const int* skip) {
  if (skip && *skip) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const double s = sv[i];
    r[i] = s > 0.0 ? (1.0 / s) / s : 0.0;
  }
}
// M = 1.5 I - 0.5 S; dev[s] = max |S - I| (float bits, NaN above everything)
__global__ void ns_combine64_kernel(int n, const double* __restrict__ S, double* __restrict__ M,
                                    unsigned* __restrict__ dev, const int* skip) {
  if (skip && *skip) return;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  float worst = 0.f;
  bool bad = false;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    const bool diag = (l - i * n == i);
    const double v = S[off + l];
    const double e = fabs(v - (diag ? 1.0 : 0.0));
    bad |= !(e == e);
    worst = fmaxf(worst, (float)e);
    M[off + l] = (diag ? 1.5 : 0.0) - 0.5 * v;
  }
  if (bad) worst = __int_as_float(0x7fc00000);
  atomicMax(&dev[blockIdx.y], __float_as_uint(worst));
}
__global__ void carry_commit64_kernel(int n, double* __restrict__ V, const double* __restrict__ Vn,
                                      const unsigned* __restrict__ dev, const int* skip) {
  if (skip && *skip) return;
  const bool ok = __uint_as_float(dev[blockIdx.y]) < 0.25f;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    V[off + l] = ok ? Vn[off + l] : ((l - i * n == i) ? 1.0 : 0.0);
  }
}
}  // namespace

// fp64 carried SVT for slices whose working columns fit in shared memory WITHOUT V but not with
// it (config 3 at the reference's precision: 176 x 144 doubles = 204 KB): instead of the blocked
// tier with V riding along as extra rows, the V-free resident Jacobi runs on A0 = G V_prev, and
// the new basis comes from its columns, v_j = G^H w_j / sigma_j^2 (one GEMM; the rounding error
// of w_j is amplified by (sigma_max / sigma_j)^2, harmless at fp64's eps for a preconditioner:
// 1e-16 x 1e8), followed by one Newton-Schulz step; a basis outside the step's convergence
// region (vanishing singular values) restarts from the identity.  The result itself never
// uses V (V-free recomposition with G), so the 1e-10 parity does not depend on it.
static int svt_carry64_vfree(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const double* G, double tau,
                             double* out, double* V, int warm, const int* skip) {
  const bool trans = I1 < I2;
  const int64_t m = trans ? I2 : I1, n = trans ? I1 : I2, nn = n * n, S = I1 * I2;
  const int F = LTB_F64;
  WsScope ws(ctx);
  double *A0 = nullptr, *w = nullptr, *z = nullptr, *d = nullptr, *sv = nullptr, *rs = nullptr, *Vn = nullptr,
         *Sg = nullptr, *M = nullptr;
  int* kept = nullptr;
  unsigned* dev = nullptr;
  if (warm) LTB_TRY(ws.alloc(sizeof(double) * batch * S, &A0));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n * m, &w));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n * m, &z));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n, &d));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n, &sv));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n, &rs));
  LTB_TRY(ws.alloc(sizeof(double) * batch * nn, &Vn));
  LTB_TRY(ws.alloc(sizeof(double) * batch * nn, &Sg));
  LTB_TRY(ws.alloc(sizeof(double) * batch * nn, &M));
  LTB_TRY(ws.alloc(sizeof(int) * batch, &kept));
  LTB_TRY(ws.alloc(sizeof(unsigned) * batch, &dev));
  const double* src = G;
  if (warm) {
    if (trans)  // A0 = V^T G
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_T, V, n, nn, LTB_OP_N, G, I2, S, A0, I2, S, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
    else  // A0 = G V
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_N, G, I2, S, LTB_OP_N, V, n, nn, A0, I2, S, nullptr,
                            nullptr, nullptr, nullptr, nullptr, skip));
    src = A0;
  }
  JacobiOut o{w, sv, nullptr, kept, d, tau, skip};
  if (warm) o.early_stop = (float)std::sqrt(DBL_EPSILON * std::sqrt((double)m));
  LTB_TRY((launch_jacobi<double, false>(ctx, batch, I1, I2, src, o)));
  if (!trans) {
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, I2, m, LTB_OP_C, w, m, n * m, LTB_OP_N, G, I2, S, z, I2, n * I2, kept,
                          nullptr, nullptr, d, nullptr, skip));
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_T, w, m, n * m, LTB_OP_N, z, I2, n * I2, out, I2, S,
                          nullptr, nullptr, kept, nullptr, nullptr, skip));
  } else {
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, n, m, LTB_OP_N, G, I2, S, LTB_OP_T, w, m, n * m, z, n, I1 * n, nullptr,
                          kept, nullptr, nullptr, d, skip));
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_N, z, n, I1 * n, LTB_OP_C, w, m, n * m, out, I2, S,
                          nullptr, nullptr, kept, nullptr, nullptr, skip));
  }
  // new basis from the columns: Vn[:, j] = G^T w_j / sigma_j^2 (I1 >= I2) or G w_j / sigma_j^2
  inv_sq64_kernel<<<grid_for(batch * n, 256, 1024), 256, 0, ctx->stream>>>(batch * n, sv, rs, skip);
  LTB_LAUNCH_CHECK(ctx);
  LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, m, trans ? LTB_OP_N : LTB_OP_T, G, I2, S, LTB_OP_T, w, m, n * m, Vn, n,
                        nn, nullptr, nullptr, nullptr, nullptr, rs, skip));
  // Newton-Schulz: V = Vn (1.5 I - 0.5 Vn^T Vn)
  LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_T, Vn, n, nn, LTB_OP_N, Vn, n, nn, Sg, n, nn, nullptr, nullptr,
                        nullptr, nullptr, nullptr, skip));
  LTB_CUDA_TRY(ctx, cudaMemsetAsync(dev, 0, sizeof(unsigned) * batch, ctx->stream));
  const dim3 egrid((unsigned)std::min<int64_t>((nn + 1023) / 1024, 64), (unsigned)batch);
  ns_combine64_kernel<<<egrid, 256, 0, ctx->stream>>>((int)n, Sg, M, dev, skip);
  LTB_LAUNCH_CHECK(ctx);
  LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_N, Vn, n, nn, LTB_OP_N, M, n, nn, Sg, n, nn, nullptr, nullptr,
                        nullptr, nullptr, nullptr, skip));
  carry_commit64_kernel<<<egrid, 256, 0, ctx->stream>>>((int)n, V, Sg, dev, skip);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

int ltb_svt_carry64_impl(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const double* G, double tau,
                         double* out, double* V, int warm, const int* skip) {
  const bool trans = I1 < I2;
  const int64_t m = trans ? I2 : I1, n = trans ? I1 : I2, nn = n * n;
  if (batch <= 0 || batch > 65535 || n < 2) return LTB_EUNSUPPORTED;
  if (!ctx->opt_force_blocked && n >= 32 &&
      jacobi_smem_bytes<double>((int)m, (int)n, true, (int)(m | 1)) > kSmemLimit &&
      jacobi_smem_bytes<double>((int)m, (int)n, false, (int)(m | 1)) <= kSmemLimit)
    return svt_carry64_vfree(ctx, batch, I1, I2, G, tau, out, V, warm, skip);
  const int F = LTB_F64;
  WsScope ws(ctx);
  double *A0 = nullptr, *w = nullptr, *vc = nullptr, *z = nullptr, *d = nullptr;
  int* kept = nullptr;
  LTB_TRY(ws.alloc(sizeof(double) * batch * I1 * I2, &A0));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n * m, &w));
  LTB_TRY(ws.alloc(sizeof(double) * batch * nn, &vc));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n * m, &z));
  LTB_TRY(ws.alloc(sizeof(double) * batch * n, &d));
  LTB_TRY(ws.alloc(sizeof(int) * batch, &kept));
  const double* src = G;
  if (warm) {
    if (trans)  // A0 = V^T G  (I1 x I2)
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_T, V, n, nn, LTB_OP_N, G, I2, I1 * I2, A0, I2, I1 * I2,
                            nullptr, nullptr, nullptr, nullptr, nullptr, skip));
    else  // A0 = G V
      LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_N, G, I2, I1 * I2, LTB_OP_N, V, n, nn, A0, I2, I1 * I2,
                            nullptr, nullptr, nullptr, nullptr, nullptr, skip));
    src = A0;
  }
  JacobiOut o{w, nullptr, vc, kept, d, tau, skip};
  // warm calls: stop after a sweep whose rotations all had relative inner products below
  // sqrt(tol), tol = eps sqrt(m) the rotation threshold (the inner products left are ~tol)
  if (warm && g_carry64_early) o.early_stop = (float)std::sqrt(DBL_EPSILON * std::sqrt((double)m));
  int st = launch_jacobi<double, true>(ctx, batch, I1, I2, src, o);
  if (st != LTB_OK) return st;
  if (!trans) {
    // Z = D W^T G (n x I2, rows limited to the kept count); out = W Z
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, I2, m, LTB_OP_C, w, m, n * m, LTB_OP_N, G, I2, I1 * I2, z, I2, n * I2,
                          kept, nullptr, nullptr, d, nullptr, skip));
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_T, w, m, n * m, LTB_OP_N, z, I2, n * I2, out, I2, I1 * I2,
                          nullptr, nullptr, kept, nullptr, nullptr, skip));
  } else {
    // Y = G W D (I1 x n, columns limited to the kept count); out = Y W^T
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, n, m, LTB_OP_N, G, I2, I1 * I2, LTB_OP_T, w, m, n * m, z, n, I1 * n,
                          nullptr, kept, nullptr, nullptr, d, skip));
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, I1, I2, n, LTB_OP_N, z, n, I1 * n, LTB_OP_C, w, m, n * m, out, I2, I1 * I2,
                          nullptr, nullptr, kept, nullptr, nullptr, skip));
  }
  // V <- V J (J's sorted columns are the rows of vc), or V <- J on the cold call
  if (warm) {
    LTB_TRY(ltb_gemm_impl(ctx, F, batch, n, n, n, LTB_OP_N, V, n, nn, LTB_OP_T, vc, n, nn, A0, n, nn, nullptr, nullptr,
                          nullptr, nullptr, nullptr, skip));
    LTB_CUDA_TRY(ctx, cudaMemcpyAsync(V, A0, sizeof(double) * batch * nn, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    cols_to_rowmajor_kernel<double><<<grid_for(batch * nn, 256, 4096), 256, 0, ctx->stream>>>(batch, (int)n, vc, V);
    LTB_LAUNCH_CHECK(ctx);
  }
  return LTB_OK;
}


// SVT of `batch` row-major I1 x I2 slices: out = U (S - tau)_+ V^H
int ltb_svt_impl(ltb_ctx* ctx, int dtype, int64_t batch, int64_t I1, int64_t I2, const void* d_a, double tau,
                 const double* /*d_tau*/, void* d_out, const int* d_skip) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "svt: bad dtype");
  if (batch < 0 || I1 < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "svt: negative dimension");
  if (batch == 0 || I1 == 0 || I2 == 0) return LTB_OK;
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    using R = typename scalar_traits<T>::real;
    const bool trans = I1 < I2;
    const int64_t m = trans ? I2 : I1, n = trans ? I1 : I2;
    if constexpr (std::is_same<T, float>::value) {
      // QR-preconditioned Jacobi: Y~ (n x n per slice), then Z = Y~ Y~^T and out = A Z | Z A
      float* y = nullptr;
      float* z = nullptr;
      int* kept = nullptr;
      LTB_TRY(ltb_ws_alloc(ctx, sizeof(float) * batch * n * n, (void**)&y));
      LTB_TRY(ltb_ws_alloc(ctx, sizeof(float) * batch * n * n, (void**)&z));
      LTB_TRY(ltb_ws_alloc(ctx, sizeof(int) * batch, (void**)&kept));
      JacobiOut o{y, nullptr, nullptr, kept, nullptr, tau, d_skip};
      o.stats = ctx->d_stats;
      const int st = launch_jacobi_qr(ctx, batch, I1, I2, (const float*)d_a, o);
      if (st == LTB_OK) {
        const float* A = (const float*)d_a;
        // Z = Y~ Y~^T: y stores the columns of Y~ as rows (K = rank index, limited to the kept count)
        LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, n, n, n, LTB_OP_T, y, n, n * n, LTB_OP_N, y, n, n * n, z, n, n * n,
                              nullptr, nullptr, kept, nullptr, nullptr, d_skip));
        if (!trans)  // out = A Z  (I1 x n)
          LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, I1, n, n, LTB_OP_N, A, I2, I1 * I2, LTB_OP_N, z, n, n * n,
                                (float*)d_out, I2, I1 * I2, nullptr, nullptr, nullptr, nullptr, nullptr, d_skip));
        else  // out = Z A  (n x I2)
          LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, n, I2, n, LTB_OP_N, z, n, n * n, LTB_OP_N, A, I2, I1 * I2,
                                (float*)d_out, I2, I1 * I2, nullptr, nullptr, nullptr, nullptr, nullptr, d_skip));
      }
      ltb_ws_free(ctx, y);
      ltb_ws_free(ctx, z);
      ltb_ws_free(ctx, kept);
      if (st != LTB_EUNSUPPORTED) return st;
    }
    T* w = nullptr;
    T* z = nullptr;
    R* d = nullptr;
    int* kept = nullptr;
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * batch * n * m, (void**)&w));
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * batch * n * (trans ? I1 : I2), (void**)&z));
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(R) * batch * n, (void**)&d));
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(int) * batch, (void**)&kept));
    JacobiOut o{w, nullptr, nullptr, kept, d, tau, d_skip};
    LTB_TRY((launch_jacobi<T, false>(ctx, batch, I1, I2, (const T*)d_a, o)));
    const T* A = (const T*)d_a;
    T* out = (T*)d_out;
    // fp32 runs the full-size first GEMM on the tensor cores (d = 0 past the kept
    // count zeroes those rows / columns); the CUDA-core path skips them instead
    const int* lim = std::is_same<T, float>::value ? nullptr : kept;
    if (!trans) {
      // Z = D W^H A   (n x I2, rows limited to the kept count)
      LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, n, I2, m, LTB_OP_C, w, m, n * m, LTB_OP_N, A, I2, I1 * I2, z, I2,
                            n * I2, lim, nullptr, nullptr, d, nullptr, d_skip));
      // out = W Z     (I1 x I2, inner dimension limited to the kept count)
      LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, I1, I2, n, LTB_OP_T, w, m, n * m, LTB_OP_N, z, I2, n * I2, out, I2,
                            I1 * I2, nullptr, nullptr, kept, nullptr, nullptr, d_skip));
    } else {
      // Y = A W D     (I1 x n, columns limited to the kept count)
      LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, I1, n, m, LTB_OP_N, A, I2, I1 * I2, LTB_OP_T, w, m, n * m, z, n,
                            I1 * n, nullptr, lim, nullptr, nullptr, d, d_skip));
      // out = Y W^H
      LTB_TRY(ltb_gemm_impl(ctx, dtype, batch, I1, I2, n, LTB_OP_N, z, n, I1 * n, LTB_OP_C, w, m, n * m, out, I2,
                            I1 * I2, nullptr, nullptr, kept, nullptr, nullptr, d_skip));
    }
    ltb_ws_free(ctx, w);
    ltb_ws_free(ctx, z);
    ltb_ws_free(ctx, d);
    ltb_ws_free(ctx, kept);
    return LTB_OK;
  });
}

namespace {
template <typename T>
__global__ void slice_gather_kernel(int64_t nu, int64_t S, const int* __restrict__ uniq, const T* __restrict__ src,
                                    T* __restrict__ dst, const int* skip) {
  if (skip && *skip) return;
  const int64_t total = nu * S;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = l / S;
    dst[l] = src[(int64_t)uniq[u] * S + (l - u * S)];
  }
}

template <typename T>
__global__ void slice_mirror_scatter_kernel(int64_t nu, int64_t S, const int* __restrict__ uniq,
                                            const int* __restrict__ partner, const T* __restrict__ src,
                                            T* __restrict__ dst, const int* skip) {
  if (skip && *skip) return;
  const int64_t total = nu * S;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < total; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = l / S, r = l - u * S;
    const int q = uniq[u], p = partner[q];
    const T v = src[l];
    dst[(int64_t)q * S + r] = v;
    if (p != q) dst[(int64_t)p * S + r] = conj_v(v);
  }
}
}  // namespace

// SVT of the transform-domain stack of a REAL tensor under `spec`: slices q
// and partner[q] are exact conjugates (SVT(conj A) = conj SVT(A), and the
// Jacobi kernel is conjugation-equivariant), so only one slice of every pair
// is solved and its conjugate mirrored -- P_u = 99 of 192 slices for config 4.
int ltb_svt_mirror_impl(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t batch, int64_t I1, int64_t I2,
                        const void* d_a, double tau, void* d_out, const int* d_skip) {
  if (!spec || !spec->d_uniq || spec->P != batch || !dtype_is_complex(dtype) || batch == 0 || I1 == 0 || I2 == 0)
    return ltb_svt_impl(ctx, dtype, batch, I1, I2, d_a, tau, nullptr, d_out, d_skip);
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    if constexpr (!scalar_traits<T>::is_complex) {
      return ltb_svt_impl(ctx, dtype, batch, I1, I2, d_a, tau, nullptr, d_out, d_skip);
    } else {
      const int64_t nu = spec->n_unique, S = I1 * I2;
      T* cin = nullptr;
      T* cout = nullptr;
      LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * nu * S, (void**)&cin));
      LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * nu * S, (void**)&cout));
      const unsigned grid = grid_for(nu * S, 256, ctx->num_sms * 8);
      slice_gather_kernel<T><<<grid, 256, 0, ctx->stream>>>(nu, S, spec->d_uniq, (const T*)d_a, cin, d_skip);
      LTB_LAUNCH_CHECK(ctx);
      LTB_TRY(ltb_svt_impl(ctx, dtype, nu, I1, I2, cin, tau, nullptr, cout, d_skip));
      slice_mirror_scatter_kernel<T><<<grid, 256, 0, ctx->stream>>>(nu, S, spec->d_uniq, spec->d_partner, cout,
                                                                    (T*)d_out, d_skip);
      LTB_LAUNCH_CHECK(ctx);
      ltb_ws_free(ctx, cin);
      ltb_ws_free(ctx, cout);
      return LTB_OK;
    }
  });
}

// ---------------------------------------------------------------- carried complex64 SVT (blocked tier)
// The PGA iterates of a complex transform domain whose slices do not fit in shared memory
// (config 4: 99 unique 1024 x 1024 complex slices) cost ~14 cold sweeps of the block-cyclic
// Jacobi per iteration.  As in the real carried paths the slices' right singular bases are
// kept between calls: the Jacobi runs on A0 = G V_prev (one tensor-core GEMM), whose columns
// are nearly orthogonal (a few sweeps with the sqrt(tol) early stop); its columns
// w_j = sigma_j u_j are G's own (V_prev J is unitary), so the V-free recomposition with G
// applies unchanged.  Every round of the blocked tier accumulates the rotations of its block
// pair in shared memory and multiplies the pair's rows of V^T by them (JacobiOut::v_acc), so
// V <- V_prev J without V riding along as extra rows of the working columns.  (The one-GEMM
// alternative v_j = G^H w_j / sigma_j^2 amplifies the rounding error of w_j by
// (sigma_max / sigma_j)^2: useless for the small singular values of a square noisy slice.)
// One Newton-Schulz step V <- V (3 I - V^H V) / 2 per call keeps the basis unitary to
// rounding; a slice whose basis leaves the step's convergence region (|V^H V - I| >= 1/4 or
// NaN) restarts from the identity.  The carried array is VT = V^T (row j = v_j, no
// conjugation): contiguous right vectors for the accumulation, and K contiguous on the left
// operand of every GEMM here.  Slices with ||G||_F <= tau have no singular value above tau:
// they are not solved at all (exact zero output), and when that holds for every slice the
// GEMMs are skipped too.
namespace {
constexpr int kFroChunks = 32;

__global__ void slice_fro_partial_kernel(int64_t S, const cplx<float>* __restrict__ G, double* __restrict__ partial) {
  const int64_t s = blockIdx.y;
  const float2* g = reinterpret_cast<const float2*>(G + s * S);
  double acc = 0.0;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < S; l += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = __ldg(g + l);
    acc += (double)v.x * v.x + (double)v.y * v.y;
  }
  __shared__ double sh[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    partial[s * kFroChunks + blockIdx.x] = t;
  }
}

// active[s] = ||G_s||_F > tau (NaN counts as active); skip2[0] = stop flag or no active slice
__global__ void carry_preactive_kernel(int64_t batch, const double* __restrict__ partial, double tau,
                                       int* __restrict__ active, const int* __restrict__ skip, int* __restrict__ skip2) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int local = 0;
  for (int64_t s = threadIdx.x; s < batch; s += blockDim.x) {
    double t = 0.0;
    for (int c = 0; c < kFroChunks; ++c) t += partial[s * kFroChunks + c];
    const int a = !(t <= tau * tau);
    active[s] = a;
    local += a;
  }
  if (local) atomicAdd(&cnt, local);
  __syncthreads();
  if (threadIdx.x == 0) skip2[0] = ((skip && *skip) || cnt == 0) ? 1 : 0;
}

__global__ void set_identity_c_kernel(int n, cplx<float>* __restrict__ VT) {
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    VT[off + l] = cplx<float>{(l - i * n == i) ? 1.f : 0.f, 0.f};
  }
}

// MT = 1.5 I - 0.5 conj(S)  (the transpose of the Newton-Schulz factor: S is Hermitian);
// dev[s] = max |S - I| (float bits: non-negative floats order like unsigned integers, NaN above)
__global__ void ns_combine_c_kernel(int n, const cplx<float>* __restrict__ S, cplx<float>* __restrict__ MT,
                                    unsigned* __restrict__ dev, const int* skip) {
  if (skip && *skip) return;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  float worst = 0.f;
  bool bad = false;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int i = l / n;
    const bool diag = (l - i * n == i);
    const cplx<float> v = S[off + l];
    const float dr = v.re - (diag ? 1.f : 0.f);
    const float e = fmaxf(fabsf(dr), fabsf(v.im));
    bad |= !(dr == dr) || !(v.im == v.im);
    worst = fmaxf(worst, e);
    MT[off + l] = cplx<float>{(diag ? 1.5f : 0.f) - 0.5f * v.re, 0.5f * v.im};
  }
  if (bad) worst = __int_as_float(0x7fc00000);
  atomicMax(&dev[blockIdx.y], __float_as_uint(worst));
}

// VT <- VTn with its rows (the right vectors) moved to their sigma-sorted places, so that the next
// call's working columns A0 = G V come in descending order of norm (de Rijk's ordering: the large
// columns share the first blocks and meet each other first), or the identity for a basis outside
// the Newton-Schulz convergence region
__global__ void carry_commit_kernel(int n, cplx<float>* __restrict__ VT, const cplx<float>* __restrict__ VTn,
                                    const unsigned* __restrict__ dev, const int* __restrict__ rank,
                                    const int* skip) {
  if (skip && *skip) return;
  const float d = __uint_as_float(dev[blockIdx.y]);
  const bool ok = d < 0.25f;
  const int nn = n * n;
  const int64_t off = (int64_t)blockIdx.y * nn;
  const int* rk = rank + (int64_t)blockIdx.y * n;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nn; l += gridDim.x * blockDim.x) {
    const int j = l / n, i = l - j * n;
    if (ok)
      VT[off + (int64_t)rk[j] * n + i] = VTn[off + l];
    else
      VT[off + l] = cplx<float>{(i == j) ? 1.f : 0.f, 0.f};
  }
}
}  // namespace

int ltb_svt_carry_c64_impl(ltb_ctx* ctx, int64_t batch, int64_t I1, int64_t I2, const void* d_g, double tau,
                           void* d_out, void* d_vt, int warm, const int* skip) {
  using T = cplx<float>;
  const int64_t m = I1, n = I2, nn = n * n, S = I1 * I2;
  if (batch <= 0 || batch > 65535 || I1 < I2 || n < 32 || (n & 1)) return LTB_EUNSUPPORTED;
  // slices that fit in shared memory keep the (much faster) resident kernel
  if (!ctx->opt_force_blocked && jacobi_smem_bytes<T>((int)m, (int)n, false, (int)(m | 1)) <= kSmemLimit)
    return LTB_EUNSUPPORTED;
  const int C = LTB_C64;
  const T* G = (const T*)d_g;
  T* out = (T*)d_out;
  T* VT = (T*)d_vt;
  WsScope ws(ctx);
  T *A0 = nullptr, *w = nullptr, *z = nullptr, *Sg = nullptr, *MT = nullptr, *VTn = nullptr;
  float* d = nullptr;
  double* partial = nullptr;
  int *kept = nullptr, *pre = nullptr, *skip2 = nullptr, *rank = nullptr;
  unsigned* dev = nullptr;
  LTB_TRY(ws.alloc(sizeof(int) * batch * n, &rank));
  if (warm) LTB_TRY(ws.alloc(sizeof(T) * batch * S, &A0));
  LTB_TRY(ws.alloc(sizeof(T) * batch * n * m, &w));
  LTB_TRY(ws.alloc(sizeof(T) * batch * nn, &z));
  LTB_TRY(ws.alloc(sizeof(T) * batch * nn, &Sg));
  LTB_TRY(ws.alloc(sizeof(T) * batch * nn, &MT));
  LTB_TRY(ws.alloc(sizeof(T) * batch * nn, &VTn));
  LTB_TRY(ws.alloc(sizeof(float) * batch * n, &d));
  LTB_TRY(ws.alloc(sizeof(double) * batch * kFroChunks, &partial));
  LTB_TRY(ws.alloc(sizeof(int) * batch, &kept));
  LTB_TRY(ws.alloc(sizeof(int) * batch, &pre));
  LTB_TRY(ws.alloc(sizeof(int) * 2, &skip2));
  LTB_TRY(ws.alloc(sizeof(unsigned) * batch, &dev));
  const dim3 egrid((unsigned)std::min<int64_t>((nn + 1023) / 1024, 64), (unsigned)batch);
  // slices without a singular value above tau
  slice_fro_partial_kernel<<<dim3(kFroChunks, (unsigned)batch), 256, 0, ctx->stream>>>(S, G, partial);
  LTB_LAUNCH_CHECK(ctx);
  carry_preactive_kernel<<<1, 256, 0, ctx->stream>>>(batch, partial, tau, pre, skip, skip2);
  LTB_LAUNCH_CHECK(ctx);
  if (warm) {  // A0 = G V  (B = V stored as VT: n x k)
    LTB_TRY(ltb_gemm_impl(ctx, C, batch, m, n, n, LTB_OP_N, G, n, S, LTB_OP_T, VT, n, nn, A0, n, S, nullptr, nullptr,
                          nullptr, nullptr, nullptr, skip2));
  } else {
    set_identity_c_kernel<<<egrid, 256, 0, ctx->stream>>>((int)n, VT);
    LTB_LAUNCH_CHECK(ctx);
  }
  JacobiOut o{w, nullptr, nullptr, kept, d, tau, skip2};
  o.stats = ctx->d_stats;
  o.pre_active = pre;
  o.v_acc = VT;
  o.rank_out = rank;
  o.truncate = warm != 0 && !ctx->opt_full_sweeps;  // (the carried bases are sigma-sorted: the large columns lead)
  LTB_TRY((launch_jacobi_blocked<T, false>(ctx, batch, I1, I2, warm ? A0 : G, o, 40)));
  // Z = D W^H G (rows limited to the kept count), out = W Z (zeros for a slice that keeps nothing)
  LTB_TRY(ltb_gemm_impl(ctx, C, batch, n, I2, m, LTB_OP_C, w, m, n * m, LTB_OP_N, G, I2, S, z, I2, nn, kept, nullptr,
                        nullptr, d, nullptr, skip));
  LTB_TRY(ltb_gemm_impl(ctx, C, batch, I1, I2, n, LTB_OP_T, w, m, n * m, LTB_OP_N, z, I2, nn, out, I2, S, nullptr,
                        nullptr, kept, nullptr, nullptr, skip));
  // Newton-Schulz: S = V^H V = conj(VT) VT^T, VT <- (1.5 I - 0.5 S)^T VT
  LTB_TRY(ltb_gemm_impl(ctx, C, batch, n, n, n, LTB_OP_C, VT, n, nn, LTB_OP_T, VT, n, nn, Sg, n, nn, nullptr, nullptr,
                        nullptr, nullptr, nullptr, skip2));
  LTB_CUDA_TRY(ctx, cudaMemsetAsync(dev, 0, sizeof(unsigned) * batch, ctx->stream));
  ns_combine_c_kernel<<<egrid, 256, 0, ctx->stream>>>((int)n, Sg, MT, dev, skip2);
  LTB_LAUNCH_CHECK(ctx);
  LTB_TRY(ltb_gemm_impl(ctx, C, batch, n, n, n, LTB_OP_N, MT, n, nn, LTB_OP_N, VT, n, nn, VTn, n, nn, nullptr, nullptr,
                        nullptr, nullptr, nullptr, skip2));
  carry_commit_kernel<<<egrid, 256, 0, ctx->stream>>>((int)n, VT, VTn, dev, rank, skip2);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

// the carried complex64 SVT on the transform-domain stack of a REAL tensor: one slice of
// every conjugate pair is solved (VT holds n_unique bases) and its conjugate mirrored
int ltb_svt_mirror_carry_c64_impl(ltb_ctx* ctx, const ltb_spec* spec, int64_t batch, int64_t I1, int64_t I2,
                                  const void* d_a, double tau, void* d_out, void* d_vt, int warm, const int* d_skip) {
  using T = cplx<float>;
  if (!spec || !spec->d_uniq || spec->P != batch)
    return ltb_svt_carry_c64_impl(ctx, batch, I1, I2, d_a, tau, d_out, d_vt, warm, d_skip);
  const int64_t nu = spec->n_unique, S = I1 * I2;
  WsScope ws(ctx);
  T *cin = nullptr, *cout = nullptr;
  LTB_TRY(ws.alloc(sizeof(T) * nu * S, &cin));
  LTB_TRY(ws.alloc(sizeof(T) * nu * S, &cout));
  const unsigned grid = grid_for(nu * S, 256, ctx->num_sms * 8);
  slice_gather_kernel<T><<<grid, 256, 0, ctx->stream>>>(nu, S, spec->d_uniq, (const T*)d_a, cin, d_skip);
  LTB_LAUNCH_CHECK(ctx);
  LTB_TRY(ltb_svt_carry_c64_impl(ctx, nu, I1, I2, cin, tau, cout, d_vt, warm, d_skip));
  slice_mirror_scatter_kernel<T><<<grid, 256, 0, ctx->stream>>>(nu, S, spec->d_uniq, spec->d_partner, cout, (T*)d_out,
                                                                d_skip);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

extern "C" int ltb_spec_slice_svt(ltb_ctx* ctx, const ltb_spec* spec, int dtype, int64_t batch, int64_t I1,
                                  int64_t I2, const void* d_a, double tau, void* d_out) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "svt: bad dtype");
  if (batch < 0 || I1 < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "svt: negative dimension");
  return ltb_svt_mirror_impl(ctx, spec, dtype, batch, I1, I2, d_a, tau, d_out, nullptr);
}

extern "C" int ltb_slice_singular_values(ltb_ctx* ctx, int dtype, int64_t batch, int64_t I1, int64_t I2,
                                         const void* d_a, void* d_s) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "svd: bad dtype");
  if (batch < 0 || I1 < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "svd: negative dimension");
  if (batch == 0 || I1 == 0 || I2 == 0) return LTB_OK;
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    JacobiOut o{nullptr, d_s, nullptr, nullptr, nullptr, 0.0, nullptr};
    if constexpr (std::is_same<T, float>::value) {  // sigma only: QR-preconditioned kernel when it fits
      o.stats = ctx->d_stats;
      const int st = launch_jacobi_qr(ctx, batch, I1, I2, (const float*)d_a, o);
      if (st != LTB_EUNSUPPORTED) return st;
    }
    return launch_jacobi<T, false>(ctx, batch, I1, I2, (const T*)d_a, o);
  });
}

extern "C" int ltb_slice_svd(ltb_ctx* ctx, int dtype, int64_t batch, int64_t I1, int64_t I2, const void* d_a,
                             void* d_u, void* d_s, void* d_v) {
  if (!dtype_valid(dtype)) return ltb_set_error(ctx, LTB_EPARAM, "svd: bad dtype");
  if (batch < 0 || I1 < 0 || I2 < 0) return ltb_set_error(ctx, LTB_ESHAPE, "svd: negative dimension");
  if (batch == 0 || I1 == 0 || I2 == 0) return LTB_OK;
  return dispatch_dtype(dtype, [&](auto tg) -> int {
    using T = typename decltype(tg)::type;
    using R = typename scalar_traits<T>::real;
    const bool trans = I1 < I2;
    const int m = (int)(trans ? I2 : I1), n = (int)(trans ? I1 : I2);
    T* w = nullptr;
    T* vcols = nullptr;
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * batch * n * m, (void**)&w));
    LTB_TRY(ltb_ws_alloc(ctx, sizeof(T) * batch * n * n, (void**)&vcols));
    JacobiOut o{w, d_s, vcols, nullptr, nullptr, 0.0, nullptr};
    LTB_TRY((launch_jacobi<T, true>(ctx, batch, I1, I2, (const T*)d_a, o)));
    // U of the oriented problem (m x m) and its V (n x n)
    T* u_dst = trans ? (T*)d_v : (T*)d_u;  // m x m
    T* v_dst = trans ? (T*)d_u : (T*)d_v;  // n x n
    LTB_TRY(ensure_smem(ctx, complete_u_kernel<T>, (size_t)m * sizeof(R)));
    complete_u_kernel<T><<<(unsigned)batch, 256, (size_t)m * sizeof(R), ctx->stream>>>(m, n, w, (const R*)d_s, u_dst);
    LTB_LAUNCH_CHECK(ctx);
    cols_to_rowmajor_kernel<T><<<grid_for(batch * n * n, 256, 4096), 256, 0, ctx->stream>>>(batch, n, vcols, v_dst);
    LTB_LAUNCH_CHECK(ctx);
    ltb_ws_free(ctx, w);
    ltb_ws_free(ctx, vcols);
    return LTB_OK;
  });
}
