// The shared-memory tube-tile transform engine (K1 / K1'), parameterised by a
// Loader (prologue: how tube values enter the tile) and a Storer (epilogue:
// how transformed values leave it, plus fused reductions).
//
// Reference: apply_l / apply_l_inv (transforms.py:176-226) = mode products
// (core.py:110-122) along the spec's modes, ascending forward, reversed
// inverse.  One CTA owns TT consecutive tubes (a tube = the P trailing
// elements of one (i1, i2)); the tile lives in shared memory q-major with the
// tube index fastest (pitch TT+1), so every mode product reads conflict-free.
// The per-mode matrices are staged once per CTA in shared memory, transposed
// and zero-padded to a multiple of the register block, so each inner step is
// one tile load + vector broadcast loads of RB matrix entries + RB FMAs.
#pragma once
#include "ltb_dispatch.cuh"

struct ModeStep {
  int n;
  int npad;  // n rounded up to the register block (smem matrix row length)
  int rb;    // register block (outputs per work item) for this mode
  float inv_nblk, inv_lo;
  int64_t hi, lo;
  int64_t mat_off;   // element offset of the row-major matrix in global memory
  int smem_off;      // element offset of the transposed padded matrix in shared memory
  int sym;           // ltb_spec::sym of the step's matrix (even/odd symmetry), 0 none
  int sym_on;        // the fp32 FFMA2 plan stages the half matrix and runs mode_step_f2_sym*
};

struct XformParams {
  int nsteps;
  ModeStep step[16];
  int P;
  int64_t NT;
  int TT;
  int ttshift;  // log2(TT)
  int pitch;
  float invP;   // 1/P for division-free index math
  int mats_in_smem;
  int mat_smem_elems;
};

constexpr int kXformThreads = 256;

template <typename Tc> constexpr int xform_rb() { return scalar_traits<Tc>::is_complex ? 4 : 8; }

inline void build_steps(const ltb_spec* spec, int inverse, XformParams& p) {
  p.nsteps = spec->nmodes;
  for (int k = 0; k < spec->nmodes; ++k) {
    const int m = inverse ? spec->nmodes - 1 - k : k;
    const int ax = spec->axes[m];
    int64_t hi = 1, lo = 1;
    for (int a = 0; a < ax; ++a) hi *= spec->trail_dims[a];
    for (int a = ax + 1; a < spec->ntrail; ++a) lo *= spec->trail_dims[a];
    p.step[k].n = spec->sizes[m];
    p.step[k].hi = hi;
    p.step[k].lo = lo;
    p.step[k].mat_off = spec->mat_off[m];
    p.step[k].sym = spec->is_complex ? 0 : spec->sym[inverse ? 1 : 0][m];
    p.step[k].sym_on = 0;
  }
  p.P = (int)spec->P;
  p.invP = 1.0f / (float)p.P;
}

// smem layout of the matrices for compute type Tc (register block RB)
template <typename Tc>
inline void plan_matrices(XformParams& p) {
  constexpr int RB = xform_rb<Tc>();
  int off = 0;
  for (int s = 0; s < p.nsteps; ++s) {
    ModeStep& ms = p.step[s];
    int rb = 1;
    while (rb < RB && rb < ms.n) rb <<= 1;  // smallest power of two >= n, capped at RB
    ms.rb = rb;
    ms.npad = (ms.n + rb - 1) / rb * rb;
    ms.inv_nblk = 1.0f / (float)(ms.npad / rb);
    ms.inv_lo = 1.0f / (float)ms.lo;
    ms.sym_on = 0;
    off = (off + RB - 1) / RB * RB;  // every matrix starts vector-aligned
    ms.smem_off = off;
    off += ms.n * ms.npad;
  }
  p.mat_smem_elems = off;
}

// l -> (t, q) with l = t * P + q, without an integer division (l < 2^24)
__device__ __forceinline__ void split_tube(int l, int P, float invP, int& t, int& q) {
  t = __float2int_rz((float)l * invP);
  q = l - t * P;
  if (q < 0) {
    --t;
    q += P;
  } else if (q >= P) {
    ++t;
    q -= P;
  }
}

// Walks the tube-major element indices l = l0, l0 + stride, ... of a tile, tracking
// q = l mod P and the q-major shared-memory index i = q * pitch + l / P incrementally
// (one division per walk instead of a split per element)
struct TubeWalk {
  int q, i, dq, di, wrap, P;
  __device__ __forceinline__ TubeWalk(int l0, int stride, const XformParams& p) : P(p.P) {
    int t;
    split_tube(l0, p.P, p.invP, t, q);
    i = q * p.pitch + t;
    const int dt = stride / p.P;
    dq = stride - dt * p.P;
    di = dq * p.pitch + dt;
    wrap = 1 - p.P * p.pitch;
  }
  __device__ __forceinline__ void next() {
    q += dq;
    i += di;
    if (q >= P) {
      q -= P;
      i += wrap;
    }
  }
};

// ---------------------------------------------------------------- async copies
// LDGSTS: global -> shared without a register round trip, so every thread keeps all of
// its tile loads in flight at once (a plain load + st.shared loop holds one per thread,
// which left the tile engine at a few hundred GB/s); completion via cp.async.wait_all
template <int B>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(B) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------- loaders
// load(p, S0, S1, extra, tube0, nt, tid): fill S0 (q-major, pitch) with the tile's tube
// values; S1 (same size) and `extra` (extra_bytes) are free scratch until the first mode
// step.  Outstanding cp.async copies are waited for by the kernel before its barrier.
template <typename Tin>
struct LoadPlain {
  static constexpr int kExtraBufs = 0;  // additional tile-sized buffers in shared memory
  static constexpr bool kMaskWords = false;
  const Tin* in;
  int layout;
  template <typename Tc>
  __device__ __forceinline__ void load(const XformParams& p, Tc* S, Tc* /*S1*/, unsigned char* /*extra*/,
                                       int64_t tube0, int nt, int tid) const {
    const int P = p.P, TT = p.TT, pitch = p.pitch;
    if constexpr (std::is_same<Tin, Tc>::value) {
      if (layout == LTB_TUBE_MAJOR) {
        const Tin* src = in + tube0 * P;
        const int cnt = nt * P;
        TubeWalk w(tid, kXformThreads, p);
        for (int l = tid; l < cnt; l += kXformThreads, w.next()) cp_async<sizeof(Tc)>(S + w.i, src + l);
      } else {
        const int cnt = P * TT;
        for (int l = tid; l < cnt; l += kXformThreads) {
          const int q = l >> p.ttshift;
          const int t = l & (TT - 1);
          if (t < nt) cp_async<sizeof(Tc)>(S + q * pitch + t, in + (int64_t)q * p.NT + tube0 + t);
        }
      }
      return;
    }
    if (layout == LTB_TUBE_MAJOR) {
      const Tin* src = in + tube0 * P;
      const int cnt = nt * P;
      TubeWalk w(tid, kXformThreads, p);
#pragma unroll 4
      for (int l = tid; l < cnt; l += kXformThreads, w.next()) S[w.i] = cvt<Tc>(src[l]);
    } else {
      const int cnt = P * TT;
#pragma unroll 4
      for (int l = tid; l < cnt; l += kXformThreads) {
        const int q = l >> p.ttshift;
        const int t = l & (TT - 1);
        if (t < nt) S[q * pitch + t] = cvt<Tc>(in[(int64_t)q * p.NT + tube0 + t]);
      }
    }
  }
  template <typename Tc>
  __device__ __forceinline__ void finish(const XformParams&, Tc*, Tc*, unsigned char*, int64_t, int, int) const {}
};

// ---------------------------------------------------------------- storers
// NACC fused per-CTA reductions; slot k is a max when (MAXMASK >> k) & 1.
template <typename Tout, bool RESIDUAL>
struct StorePlain {
  static constexpr int NACC = 2;
  static constexpr unsigned MAXMASK = 0;
  Tout* out;
  int layout;
  template <typename Tc>
  __device__ __forceinline__ void store(const XformParams& p, const Tc* S, int64_t tube0, int nt, int tid,
                                        double* acc) const {
    const int P = p.P, TT = p.TT, pitch = p.pitch;
    if (layout == LTB_TUBE_MAJOR) {
      Tout* o = out + tube0 * P;
      const int cnt = nt * P;
      TubeWalk w(tid, kXformThreads, p);
#pragma unroll 4
      for (int l = tid; l < cnt; l += kXformThreads, w.next()) {
        const Tc v = S[w.i];
        if (RESIDUAL) {
          acc[0] += (double)abs2_v(v);
          acc[1] += (double)im_v(v) * (double)im_v(v);
        }
        o[l] = cvt<Tout>(v);
      }
    } else {
      const int cnt = P * TT;
      for (int l = tid; l < cnt; l += kXformThreads) {
        const int q = l >> p.ttshift;
        const int t = l & (TT - 1);
        if (t < nt) {
          const Tc v = S[q * pitch + t];
          if (RESIDUAL) {
            acc[0] += (double)abs2_v(v);
            acc[1] += (double)im_v(v) * (double)im_v(v);
          }
          out[(int64_t)q * p.NT + tube0 + t] = cvt<Tout>(v);
        }
      }
    }
  }
};

// RB consecutive matrix entries in vector loads (alignment: the largest power of two
// dividing the row, at most 16 bytes, so row i0 = iblk * RB stays aligned for any RB)
constexpr int mrow_align(int bytes) { return bytes % 16 == 0 ? 16 : bytes % 8 == 0 ? 8 : bytes % 4 == 0 ? 4 : 2; }
template <typename Tm, int RB> struct alignas(mrow_align(sizeof(Tm) * RB)) mrow {
  Tm v[RB];
};

// floor(a / d) for 0 <= a < 2^24 via a float reciprocal (exact after one correction)
__device__ __forceinline__ int fdiv(int a, int d, float inv) {
  int q = __float2int_rz((float)a * inv);
  const int r = a - q * d;
  q += (r >= d) - (r < 0);
  return q;
}

// one mode product out of shared memory: every work item produces RBM outputs
// (rows i0 .. i0+RBM-1 of M times one fibre of the tile)
template <typename Tc, typename Tm, int RBM>
__device__ __forceinline__ void mode_step(const XformParams& p, const ModeStep& ms, const Tc* __restrict__ src,
                                          Tc* __restrict__ dst, const Tm* __restrict__ Msm,
                                          const Tm* __restrict__ Mg, int tid) {
  const int n = ms.n, npad = ms.npad, lo = (int)ms.lo, hi = (int)ms.hi;
  const int TT = p.TT, pitch = p.pitch;
  const int nblk = npad / RBM;
  const int work = hi * lo * nblk * TT;
  for (int w = tid; w < work; w += kXformThreads) {
    const int t = w & (TT - 1);
    const int r0 = w >> p.ttshift;
    const int r1 = fdiv(r0, nblk, ms.inv_nblk);
    const int iblk = r0 - r1 * nblk;
    const int hi_i = fdiv(r1, lo, ms.inv_lo);
    const int lo_i = r1 - hi_i * lo;
    const int i0 = iblk * RBM;
    const int base = hi_i * n * lo + lo_i;
    Tc acc[RBM];
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr) acc[rr] = zero_v<Tc>();
    const Tc* col = src + base * pitch + t;
    const int jstride = lo * pitch;
    if (p.mats_in_smem) {
      const Tm* mrowp = Msm + i0;
      for (int j = 0; j < n; ++j) {
        const Tc v = col[j * jstride];
        const mrow<Tm, RBM> mv = *reinterpret_cast<const mrow<Tm, RBM>*>(mrowp + j * npad);
#pragma unroll
        for (int rr = 0; rr < RBM; ++rr) fma_acc(acc[rr], mv.v[rr], v);
      }
    } else {
      for (int j = 0; j < n; ++j) {
        const Tc v = col[j * jstride];
#pragma unroll
        for (int rr = 0; rr < RBM; ++rr) {
          const int i = min(i0 + rr, n - 1);
          fma_acc(acc[rr], ldg_v(Mg + (size_t)i * n + j), v);
        }
      }
    }
    Tc* out = dst + base * pitch + t;
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr)
      if (i0 + rr < n) out[(i0 + rr) * jstride] = acc[rr];
  }
}

// fp32: each work item takes two tubes (t and t + TT/2) as one float2 and RBM
// outputs, so the FMAs issue as FFMA2 against the broadcast matrix entry
template <int RBM>
__device__ __forceinline__ void mode_step_f2(const XformParams& p, const ModeStep& ms, const float* __restrict__ src,
                                             float* __restrict__ dst, const float* __restrict__ Msm, int tid) {
  const int n = ms.n, npad = ms.npad, lo = (int)ms.lo, hi = (int)ms.hi;
  const int half = p.TT >> 1, pitch = p.pitch;
  const int hshift = p.ttshift - 1;
  const int nblk = npad / RBM;
  const int work = hi * lo * nblk * half;
  for (int w = tid; w < work; w += kXformThreads) {
    const int t = w & (half - 1);
    const int r0 = w >> hshift;
    const int r1 = fdiv(r0, nblk, ms.inv_nblk);
    const int iblk = r0 - r1 * nblk;
    const int hi_i = fdiv(r1, lo, ms.inv_lo);
    const int lo_i = r1 - hi_i * lo;
    const int i0 = iblk * RBM;
    const int base = hi_i * n * lo + lo_i;
    float2 acc[RBM];
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr) acc[rr] = make_float2(0.f, 0.f);
    const float* col = src + base * pitch + t;
    const int jstride = lo * pitch;
    const float* mrowp = Msm + i0;
#pragma unroll 4
    for (int j = 0; j < n; ++j, col += jstride, mrowp += npad) {
      const float2 v = make_float2(col[0], col[half]);
      const mrow<float, RBM> mv = *reinterpret_cast<const mrow<float, RBM>*>(mrowp);
#pragma unroll
      for (int rr = 0; rr < RBM; ++rr) acc[rr] = __ffma2_rn(make_float2(mv.v[rr], mv.v[rr]), v, acc[rr]);
    }
    float* out = dst + base * pitch + t;
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr)
      if (i0 + rr < n) {
        out[(i0 + rr) * jstride] = acc[rr].x;
        out[(i0 + rr) * jstride + half] = acc[rr].y;
      }
  }
}

// Even/odd symmetric modes (DCT-II and its inverse, ltb_spec::sym), fp32 FFMA2 as
// mode_step_f2, half the multiply-adds of the full product.  n even, h = n / 2.
// sym 1, A[i][n-1-j] = (-1)^i A[i][j] (forward DCT-II): out_i = sum_{j<h} A[i][j] (v_j +- v_{n-1-j}),
//   + for even i, - for odd i; a work item takes RBM rows of one parity.  Shared memory: two
//   parity planes, Msm[(par h + j) npad + e] = A[2 e + par][j] (j < h, e < h)
template <int RBM>
__device__ __forceinline__ void mode_step_f2_sym1(const XformParams& p, const ModeStep& ms,
                                                  const float* __restrict__ src, float* __restrict__ dst,
                                                  const float* __restrict__ Msm, int tid) {
  const int n = ms.n, h = n >> 1, npad = ms.npad, lo = (int)ms.lo, hi = (int)ms.hi;
  const int half = p.TT >> 1, pitch = p.pitch;
  const int hshift = p.ttshift - 1;
  const int nblk = npad / RBM;  // blocks per parity
  const int work = hi * lo * 2 * nblk * half;
  for (int w = tid; w < work; w += kXformThreads) {
    const int t = w & (half - 1);
    const int r0 = w >> hshift;
    const int r1 = fdiv(r0, 2 * nblk, ms.inv_nblk);  // inv_nblk = 1 / (2 nblk)
    const int rem = r0 - r1 * 2 * nblk;
    const int par = rem >= nblk ? 1 : 0;
    const int e0 = (rem - par * nblk) * RBM;
    const int hi_i = fdiv(r1, lo, ms.inv_lo);
    const int lo_i = r1 - hi_i * lo;
    const int base = hi_i * n * lo + lo_i;
    const int jstride = lo * pitch;
    const float sg = par ? -1.f : 1.f;
    const float2 SG = make_float2(sg, sg);
    float2 acc[RBM];
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr) acc[rr] = make_float2(0.f, 0.f);
    const float* c1 = src + base * pitch + t;
    const float* c2 = c1 + (n - 1) * jstride;
    const float* mrowp = Msm + par * h * npad + e0;
#pragma unroll 2
    for (int j = 0; j < h; ++j, c1 += jstride, c2 -= jstride, mrowp += npad) {
      const float2 x = __ffma2_rn(SG, make_float2(c2[0], c2[half]), make_float2(c1[0], c1[half]));
      const mrow<float, RBM> mv = *reinterpret_cast<const mrow<float, RBM>*>(mrowp);
#pragma unroll
      for (int rr = 0; rr < RBM; ++rr) acc[rr] = __ffma2_rn(make_float2(mv.v[rr], mv.v[rr]), x, acc[rr]);
    }
    float* out = dst + base * pitch + t;
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr)
      if (e0 + rr < h) {
        const int i = 2 * (e0 + rr) + par;
        out[i * jstride] = acc[rr].x;
        out[i * jstride + half] = acc[rr].y;
      }
  }
}

// sym 2, A[n-1-i][j] = (-1)^j A[i][j] (inverse DCT, the transpose): with E_i / O_i the sums over
//   even / odd j of A[i][j] v_j (i < h), out_i = E_i + O_i and out_{n-1-i} = E_i - O_i; a work
//   item takes RBM rows i < h and writes 2 RBM outputs.  Shared memory Msm[j npad + i] = A[i][j]
template <int RBM>
__device__ __forceinline__ void mode_step_f2_sym2(const XformParams& p, const ModeStep& ms,
                                                  const float* __restrict__ src, float* __restrict__ dst,
                                                  const float* __restrict__ Msm, int tid) {
  const int n = ms.n, h = n >> 1, npad = ms.npad, lo = (int)ms.lo, hi = (int)ms.hi;
  const int half = p.TT >> 1, pitch = p.pitch;
  const int hshift = p.ttshift - 1;
  const int nblk = npad / RBM;
  const int work = hi * lo * nblk * half;
  for (int w = tid; w < work; w += kXformThreads) {
    const int t = w & (half - 1);
    const int r0 = w >> hshift;
    const int r1 = fdiv(r0, nblk, ms.inv_nblk);
    const int i0 = (r0 - r1 * nblk) * RBM;
    const int hi_i = fdiv(r1, lo, ms.inv_lo);
    const int lo_i = r1 - hi_i * lo;
    const int base = hi_i * n * lo + lo_i;
    const int jstride = lo * pitch;
    float2 ae[RBM], ao[RBM];
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr) ae[rr] = ao[rr] = make_float2(0.f, 0.f);
    const float* col = src + base * pitch + t;
    const float* mrowp = Msm + i0;
#pragma unroll 2
    for (int j = 0; j < n; j += 2, col += 2 * jstride, mrowp += 2 * npad) {
      const float2 ve = make_float2(col[0], col[half]);
      const float2 vo = make_float2(col[jstride], col[jstride + half]);
      const mrow<float, RBM> me = *reinterpret_cast<const mrow<float, RBM>*>(mrowp);
      const mrow<float, RBM> mo = *reinterpret_cast<const mrow<float, RBM>*>(mrowp + npad);
#pragma unroll
      for (int rr = 0; rr < RBM; ++rr) {
        ae[rr] = __ffma2_rn(make_float2(me.v[rr], me.v[rr]), ve, ae[rr]);
        ao[rr] = __ffma2_rn(make_float2(mo.v[rr], mo.v[rr]), vo, ao[rr]);
      }
    }
    float* out = dst + base * pitch + t;
#pragma unroll
    for (int rr = 0; rr < RBM; ++rr)
      if (i0 + rr < h) {
        const int i = i0 + rr;
        out[i * jstride] = ae[rr].x + ao[rr].x;
        out[i * jstride + half] = ae[rr].y + ao[rr].y;
        out[(n - 1 - i) * jstride] = ae[rr].x - ao[rr].x;
        out[(n - 1 - i) * jstride + half] = ae[rr].y - ao[rr].y;
      }
  }
}

// ---------------------------------------------------------------- kernel
template <typename Tc, typename Tm, class Loader, class Storer>
__global__ void __launch_bounds__(kXformThreads)
    xform_tile_kernel(XformParams p, Loader ld, Storer st, const Tm* __restrict__ mats, double* __restrict__ partials,
                      const int* __restrict__ skip) {
  if (skip && *skip) return;
  constexpr int RB = xform_rb<Tc>();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Tm* Ms = reinterpret_cast<Tm*>(smem_raw);
  const int mat_bytes = p.mats_in_smem ? (p.mat_smem_elems * (int)sizeof(Tm) + 127) / 128 * 128 : 0;
  Tc* S0 = reinterpret_cast<Tc*>(smem_raw + mat_bytes);
  Tc* S1 = S0 + (size_t)p.P * p.pitch;
  unsigned char* extra = reinterpret_cast<unsigned char*>(S1 + (size_t)p.P * p.pitch);
  const int tid = threadIdx.x;
  const int TT = p.TT;

  // stage the transposed, zero-padded mode matrices once per (persistent) CTA:
  // Ms[off + j * npad + i] = M[i][j]
  if (p.mats_in_smem) {
    for (int s = 0; s < p.nsteps; ++s) {
      const int n = p.step[s].n, npad = p.step[s].npad;
      const Tm* M = mats + p.step[s].mat_off;
      Tm* dst = Ms + p.step[s].smem_off;
      if (p.step[s].sym_on == 1) {  // parity planes of the first h columns
        const int h = n >> 1;
        for (int l = tid; l < 2 * h * npad; l += kXformThreads) {
          const int r = l / npad, e = l - r * npad;  // r = par h + j
          const int par = r >= h ? 1 : 0, j = r - par * h;
          dst[l] = (e < h) ? M[(size_t)(2 * e + par) * n + j] : zero_v<Tm>();
        }
        continue;
      }
      if (p.step[s].sym_on == 2) {  // the first h rows, transposed
        const int h = n >> 1;
        for (int l = tid; l < n * npad; l += kXformThreads) {
          const int j = l / npad, i = l - j * npad;
          dst[l] = (i < h) ? M[(size_t)i * n + j] : zero_v<Tm>();
        }
        continue;
      }
      for (int l = tid; l < n * npad; l += kXformThreads) {
        const int j = l / npad, i = l - j * npad;
        dst[l] = (i < n) ? M[(size_t)i * n + j] : zero_v<Tm>();
      }
    }
  }
  double acc[Storer::NACC];
#pragma unroll
  for (int k = 0; k < Storer::NACC; ++k) acc[k] = ((Storer::MAXMASK >> k) & 1) ? -1.0e308 : 0.0;
  const int64_t ntiles = (p.NT + TT - 1) / TT;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
  const int64_t tube0 = tile * TT;
  const int nt = (int)min((int64_t)TT, p.NT - tube0);
  __syncthreads();  // previous tile's store has drained S0/S1
  ld.load(p, S0, S1, extra, tube0, nt, tid);
  cp_async_wait_all();
  __syncthreads();
  if constexpr (Loader::kExtraBufs > 0 || Loader::kMaskWords) {
    ld.finish(p, S0, S1, extra, tube0, nt, tid);
    __syncthreads();
  }

  Tc* src = S0;
  Tc* dst = S1;
  for (int s = 0; s < p.nsteps; ++s) {
    const ModeStep& ms = p.step[s];
    const Tm* Mg = mats + ms.mat_off;
    const Tm* Msm = Ms + ms.smem_off;
    bool done = false;
    if constexpr (std::is_same<Tc, float>::value && std::is_same<Tm, float>::value) {
      if (p.mats_in_smem && TT >= 2 && ms.sym_on) {
        if (ms.sym_on == 1) {
          switch (ms.rb) {
            case 4: mode_step_f2_sym1<4>(p, ms, src, dst, Msm, tid); break;
            case 6: mode_step_f2_sym1<6>(p, ms, src, dst, Msm, tid); break;
            case 10: mode_step_f2_sym1<10>(p, ms, src, dst, Msm, tid); break;
            default: mode_step_f2_sym1<8>(p, ms, src, dst, Msm, tid); break;
          }
        } else {
          switch (ms.rb) {
            case 4: mode_step_f2_sym2<4>(p, ms, src, dst, Msm, tid); break;
            case 6: mode_step_f2_sym2<6>(p, ms, src, dst, Msm, tid); break;
            default: mode_step_f2_sym2<8>(p, ms, src, dst, Msm, tid); break;
          }
        }
        done = true;
      } else if (p.mats_in_smem && TT >= 2) {
        switch (ms.rb) {  // kF2Blocks
          case 1: mode_step_f2<1>(p, ms, src, dst, Msm, tid); break;
          case 2: mode_step_f2<2>(p, ms, src, dst, Msm, tid); break;
          case 4: mode_step_f2<4>(p, ms, src, dst, Msm, tid); break;
          case 6: mode_step_f2<6>(p, ms, src, dst, Msm, tid); break;
          case 10: mode_step_f2<10>(p, ms, src, dst, Msm, tid); break;
          case 12: mode_step_f2<12>(p, ms, src, dst, Msm, tid); break;
          case 16: mode_step_f2<16>(p, ms, src, dst, Msm, tid); break;
          default: mode_step_f2<8>(p, ms, src, dst, Msm, tid); break;
        }
        done = true;
      }
    }
    if (!done) {
      switch (ms.rb) {
        case 1: mode_step<Tc, Tm, 1>(p, ms, src, dst, Msm, Mg, tid); break;
        case 2: mode_step<Tc, Tm, 2>(p, ms, src, dst, Msm, Mg, tid); break;
        case 4: mode_step<Tc, Tm, 4>(p, ms, src, dst, Msm, Mg, tid); break;
        default: mode_step<Tc, Tm, RB>(p, ms, src, dst, Msm, Mg, tid); break;
      }
    }
    __syncthreads();
    Tc* tmp = src;
    src = dst;
    dst = tmp;
  }

  st.store(p, src, tube0, nt, tid, acc);
  }  // tiles
  if (partials) {
    __shared__ double red[Storer::NACC][kXformThreads / 32];
    const int wid = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int k = 0; k < Storer::NACC; ++k) {
      double v = acc[k];
      const bool mx = (Storer::MAXMASK >> k) & 1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = mx ? fmax(v, w) : v + w;
      }
      if (lane == 0) red[k][wid] = v;
    }
    __syncthreads();
    if (tid < Storer::NACC) {
      const bool mx = (Storer::MAXMASK >> tid) & 1;
      double v = mx ? -1.0e308 : 0.0;
      for (int w = 0; w < kXformThreads / 32; ++w) v = mx ? fmax(v, red[tid][w]) : v + red[tid][w];
      partials[(int64_t)blockIdx.x * Storer::NACC + tid] = v;
    }
  }
}

// Pick tubes-per-tile (power of two) and the matrix staging; returns 0 when
// the tile does not fit in shared memory.  Fills p.TT / ttshift / pitch /
// mats_in_smem and the total dynamic shared memory.
// fp32 FFMA2 mode steps: the register block (matrix rows per work item) of each mode is
// picked from kF2Blocks so that the step's work items (rows / rb x fibres x tube pairs)
// fill whole rounds of the CTA's threads; e.g. n = 100 under a 3 x 100 spec with 16-tube
// tiles: rb = 8 gives 312 items (two rounds, the second 22% busy), rb = 10 gives 240 (one)
constexpr int kF2Blocks[] = {1, 2, 4, 6, 8, 10, 12, 16};
constexpr int g_xform_sym = 1;  // even/odd symmetric modes at half the multiply-adds

inline void plan_matrices_f2(XformParams& p) {
  const int half = p.TT >> 1;
  int off = 0;
  for (int s = 0; s < p.nsteps; ++s) {
    ModeStep& ms = p.step[s];
    if (ms.sym && g_xform_sym) {  // even/odd modes: rows of one parity (1) or the first half (2)
      const int h = ms.n >> 1;
      int64_t best = -1;
      for (int rb : {4, 6, 8, 10}) {
        if (ms.sym == 2 && rb > 8) continue;  // 2 rb accumulators
        const int64_t nblk = (h + rb - 1) / rb;
        const int64_t items = ms.hi * ms.lo * nblk * (ms.sym == 1 ? 2 : 1) * half;
        const int64_t per = ms.sym == 1 ? (int64_t)h * (rb + 4) : (int64_t)ms.n * (rb + 2);
        const int64_t cost = (items + kXformThreads - 1) / kXformThreads * per;
        if (best < 0 || cost < best) {
          best = cost;
          ms.rb = rb;
        }
      }
      ms.npad = (h + ms.rb - 1) / ms.rb * ms.rb;
      const int nblk = ms.npad / ms.rb;
      ms.inv_nblk = 1.0f / (float)(ms.sym == 1 ? 2 * nblk : nblk);
      ms.inv_lo = 1.0f / (float)ms.lo;
      ms.sym_on = ms.sym;
      off = (off + 3) / 4 * 4;
      ms.smem_off = off;
      off += (ms.sym == 1 ? 2 * h : ms.n) * ms.npad;
      continue;
    }
    ms.sym_on = 0;
    int64_t best = -1;
    for (int rb : kF2Blocks) {
      const int64_t nblk = (ms.n + rb - 1) / rb;
      const int64_t items = ms.hi * ms.lo * nblk * half;
      const int64_t cost = (items + kXformThreads - 1) / kXformThreads * (rb + 3);  // rb FFMA2 + loads per j
      if (best < 0 || cost < best) {
        best = cost;
        ms.rb = rb;
      }
    }
    ms.npad = (ms.n + ms.rb - 1) / ms.rb * ms.rb;
    ms.inv_nblk = 1.0f / (float)(ms.npad / ms.rb);
    ms.inv_lo = 1.0f / (float)ms.lo;
    off = (off + 3) / 4 * 4;  // 16-byte aligned matrix starts
    ms.smem_off = off;
    off += ms.n * ms.npad;
  }
  p.mat_smem_elems = off;
}

// extra_bufs: loader scratch tiles beyond S0 / S1; mask_words: room for the tile's
// packed observation-mask words (PGA prologue)
template <typename Tc, typename Tm>
inline int plan_tile(XformParams& p, size_t* smem_out, int extra_bufs = 0, bool mask_words = false) {
  plan_matrices<Tc>(p);
  const size_t mat_bytes = ((size_t)p.mat_smem_elems * sizeof(Tm) + 127) / 128 * 128;
  p.mats_in_smem = mat_bytes <= 48 * 1024 ? 1 : 0;
  const size_t mb = p.mats_in_smem ? mat_bytes : 0;
  auto smem_for = [&](int tt) {
    return mb + (size_t)(2 + extra_bufs) * p.P * (tt + 1) * sizeof(Tc) +
           (mask_words ? ((size_t)tt * p.P / 32 + 2) * 4 : 0);
  };
  int TT = 0;
  for (int tt = 32; tt >= 8 && !TT; tt >>= 1)  // two CTAs per SM
    if (smem_for(tt) <= 112 * 1024) TT = tt;
  for (int tt = 32; tt >= 1 && !TT; tt >>= 1)
    if (smem_for(tt) <= 200 * 1024) TT = tt;
  if (!TT) return 0;
  p.TT = TT;
  p.ttshift = 0;
  while ((1 << p.ttshift) < TT) ++p.ttshift;
  p.pitch = TT + 1;
  *smem_out = smem_for(TT);
  if constexpr (std::is_same<Tc, float>::value && std::is_same<Tm, float>::value) {
    if (p.mats_in_smem && TT >= 2) {  // the FFMA2 steps: rebalance the register blocks
      const XformParams keep = p;
      plan_matrices_f2(p);
      const size_t mb2 = ((size_t)p.mat_smem_elems * sizeof(Tm) + 127) / 128 * 128;
      const size_t total = *smem_out - mb + mb2;
      if (mb2 <= 48 * 1024 && (total <= *smem_out || total <= 112 * 1024)) *smem_out = total;
      else p = keep;
    }
  }
  return TT;
}

// persistent grid: enough CTAs to fill every SM at the kernel's occupancy, capped by the tile count
template <typename K>
int64_t xform_grid(ltb_ctx* ctx, const XformParams& p, K kern, size_t smem) {
  const int64_t ntiles = (p.NT + p.TT - 1) / p.TT;
  const int per_sm = ltb_occupancy(reinterpret_cast<const void*>(kern), kXformThreads, smem);
  return std::min<int64_t>(ntiles, (int64_t)per_sm * ctx->num_sms);
}

template <typename Tc, typename Tm, class Loader, class Storer>
int launch_xform_tile(ltb_ctx* ctx, XformParams p, const Loader& ld, const Storer& st, const Tm* mats,
                      double* partials, const int* skip, size_t smem, int64_t* grid_out = nullptr) {
  auto kern = xform_tile_kernel<Tc, Tm, Loader, Storer>;
  LTB_TRY(ensure_smem(ctx, kern, smem));
  const int64_t nblocks = xform_grid(ctx, p, kern, smem);
  if (grid_out) *grid_out = nblocks;  // number of per-CTA partials written
  if (nblocks == 0) return LTB_OK;
  kern<<<(unsigned)nblocks, kXformThreads, smem, ctx->stream>>>(p, ld, st, mats, partials, skip);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

// deterministic fixed-order reduction of per-block partials (NACC slots each)
__global__ void finalize_partials_kernel(const double* __restrict__ partials, int64_t nblocks, int nacc,
                                         unsigned maxmask, double* __restrict__ out);
