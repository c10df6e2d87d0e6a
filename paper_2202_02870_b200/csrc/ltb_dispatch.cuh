// Runtime dtype -> template type dispatch helpers.
#pragma once
#include "ltb_common.cuh"

template <typename T> struct type_tag { using type = T; };

template <typename F> int dispatch_dtype(int dt, F&& f) {
  switch (dt) {
    case LTB_F32: return f(type_tag<float>{});
    case LTB_F64: return f(type_tag<double>{});
    case LTB_C64: return f(type_tag<cplx<float>>{});
    case LTB_C128: return f(type_tag<cplx<double>>{});
  }
  return LTB_EPARAM;
}

template <typename T> constexpr int dtype_of();
template <> constexpr int dtype_of<float>() { return LTB_F32; }
template <> constexpr int dtype_of<double>() { return LTB_F64; }
template <> constexpr int dtype_of<cplx<float>>() { return LTB_C64; }
template <> constexpr int dtype_of<cplx<double>>() { return LTB_C128; }

template <typename R, bool C> struct pick_t { using type = R; };
template <typename R> struct pick_t<R, true> { using type = cplx<R>; };
template <typename R, bool C> using pick = typename pick_t<R, C>::type;

inline int grid_for(int64_t n, int threads, int max_blocks) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}
