// The shared-memory tube-tile transform engine (K1 / K1'), parameterised by a
// Loader (prologue: how tube values enter the tile) and a Storer (epilogue:
// how transformed values leave it, plus fused reductions).
//
// Reference: apply_l / apply_l_inv (transforms.py:176-226) = mode products
// (core.py:110-122) along the spec's modes, ascending forward, reversed
// inverse.  One CTA owns TT consecutive tubes (a tube = the P trailing
// elements of one (i1, i2)); the tile lives in shared memory q-major with the
// tube index fastest (pitch TT+1), so every mode product reads conflict-free
// and the small per-mode matrices are warp-uniform broadcast loads.
#pragma once
#include "ltb_dispatch.cuh"

struct ModeStep {
  int n;
  int64_t hi, lo;
  int64_t mat_off;
};

struct XformParams {
  int nsteps;
  ModeStep step[16];
  int P;
  int64_t NT;
  int TT;
  int pitch;
};

constexpr int kXformThreads = 256;

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
  }
  p.P = (int)spec->P;
}

// ---------------------------------------------------------------- loaders
template <typename Tin>
struct LoadPlain {
  const Tin* in;
  int layout;
  template <typename Tc>
  __device__ __forceinline__ void load(const XformParams& p, Tc* S, int64_t tube0, int nt, int tid) const {
    const int P = p.P, TT = p.TT, pitch = p.pitch;
    if (layout == LTB_TUBE_MAJOR) {
      const Tin* src = in + tube0 * P;
      const int cnt = nt * P;
      for (int l = tid; l < cnt; l += kXformThreads) {
        const int t = l / P;
        const int q = l - t * P;
        S[q * pitch + t] = cvt<Tc>(src[l]);
      }
    } else {
      const int cnt = P * TT;
      for (int l = tid; l < cnt; l += kXformThreads) {
        const int q = l / TT;
        const int t = l - q * TT;
        if (t < nt) S[q * pitch + t] = cvt<Tc>(in[(int64_t)q * p.NT + tube0 + t]);
      }
    }
  }
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
      for (int l = tid; l < cnt; l += kXformThreads) {
        const int t = l / P;
        const int q = l - t * P;
        const Tc v = S[q * pitch + t];
        if (RESIDUAL) {
          acc[0] += (double)abs2_v(v);
          acc[1] += (double)im_v(v) * (double)im_v(v);
        }
        o[l] = cvt<Tout>(v);
      }
    } else {
      const int cnt = P * TT;
      for (int l = tid; l < cnt; l += kXformThreads) {
        const int q = l / TT;
        const int t = l - q * TT;
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

// ---------------------------------------------------------------- kernel
template <typename Tc, typename Tm, class Loader, class Storer>
__global__ void __launch_bounds__(kXformThreads)
    xform_tile_kernel(XformParams p, Loader ld, Storer st, const Tm* __restrict__ mats, double* __restrict__ partials,
                      const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tc* S0 = reinterpret_cast<Tc*>(smem_raw);
  Tc* S1 = S0 + (size_t)p.P * p.pitch;
  const int tid = threadIdx.x;
  const int TT = p.TT;
  const int pitch = p.pitch;
  const int64_t tube0 = (int64_t)blockIdx.x * TT;
  const int nt = (int)min((int64_t)TT, p.NT - tube0);

  ld.load(p, S0, tube0, nt, tid);
  __syncthreads();

  constexpr int RB = scalar_traits<Tc>::is_complex ? 4 : 8;
  Tc* src = S0;
  Tc* dst = S1;
  for (int s = 0; s < p.nsteps; ++s) {
    const int n = p.step[s].n;
    const int lo = (int)p.step[s].lo;
    const int hi = (int)p.step[s].hi;
    const Tm* M = mats + p.step[s].mat_off;
    const int nblk = (n + RB - 1) / RB;
    const int work = hi * lo * nblk * TT;
    for (int w = tid; w < work; w += kXformThreads) {
      const int t = w % TT;
      int r = w / TT;
      const int iblk = r % nblk;
      r /= nblk;
      const int lo_i = r % lo;
      const int hi_i = r / lo;
      const int i0 = iblk * RB;
      const int base = hi_i * n * lo + lo_i;
      Tc acc[RB];
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) acc[rr] = zero_v<Tc>();
      for (int j = 0; j < n; ++j) {
        const Tc v = src[(base + j * lo) * pitch + t];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
          const int i = min(i0 + rr, n - 1);
          const Tm mv = ldg_v(M + (size_t)i * n + j);
          fma_acc(acc[rr], mv, v);
        }
      }
#pragma unroll
      for (int rr = 0; rr < RB; ++rr) {
        const int i = i0 + rr;
        if (i < n) dst[(base + i * lo) * pitch + t] = acc[rr];
      }
    }
    __syncthreads();
    Tc* tmp = src;
    src = dst;
    dst = tmp;
  }

  double acc[Storer::NACC];
#pragma unroll
  for (int k = 0; k < Storer::NACC; ++k) acc[k] = ((Storer::MAXMASK >> k) & 1) ? -1.0e308 : 0.0;
  st.store(p, src, tube0, nt, tid, acc);
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

// pick tubes-per-tile; 0 => the tile does not fit in shared memory
template <typename Tc>
inline int choose_tt(int P, size_t* smem_out) {
  auto smem_for = [&](int tt) { return (size_t)2 * P * (tt + 1) * sizeof(Tc); };
  for (int tt = 32; tt >= 8; tt >>= 1)
    if (smem_for(tt) <= 100 * 1024) {
      *smem_out = smem_for(tt);
      return tt;
    }
  for (int tt = 32; tt >= 1; tt >>= 1)
    if (smem_for(tt) <= 200 * 1024) {
      *smem_out = smem_for(tt);
      return tt;
    }
  return 0;
}

template <typename Tc, typename Tm, class Loader, class Storer>
int launch_xform_tile(ltb_ctx* ctx, XformParams p, const Loader& ld, const Storer& st, const Tm* mats,
                      double* partials, const int* skip, size_t smem) {
  auto kern = xform_tile_kernel<Tc, Tm, Loader, Storer>;
  if (smem > 48 * 1024)
    LTB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t nblocks = (p.NT + p.TT - 1) / p.TT;
  if (nblocks > 0x7fffffff) return ltb_set_error(ctx, LTB_ESHAPE, "transform: too many tubes");
  if (nblocks == 0) return LTB_OK;
  kern<<<(unsigned)nblocks, kXformThreads, smem, ctx->stream>>>(p, ld, st, mats, partials, skip);
  LTB_LAUNCH_CHECK(ctx);
  return LTB_OK;
}

// deterministic fixed-order reduction of per-block partials (NACC slots each)
__global__ void finalize_partials_kernel(const double* __restrict__ partials, int64_t nblocks, int nacc,
                                         unsigned maxmask, double* __restrict__ out);
