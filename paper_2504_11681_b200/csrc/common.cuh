// Shared device helpers for the TurboFNO B200 kernels (sm_100a).
//
// Element type everywhere is complex64 = float2 (re, im), matching the
// reference's COMPLEX_DTYPE (fnofuse/core.py:17-19).  Twiddles come from one
// table of omega_{TW_MAX}^k built in double precision on the host and rounded
// to fp32 (the reference builds its per-stage twiddles the same way,
// fnofuse/fft.py:114-124).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define TFNO_TW_LOG2 13
#define TFNO_TW_MAX (1 << TFNO_TW_LOG2)   // largest supported transform length

namespace tfno {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
// multiply by -i (forward, DIR = -1) or +i (inverse, DIR = +1)
template <int DIR>
__device__ __forceinline__ float2 mul_dir_i(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}
// acc += a * b (4 FFMA)
__device__ __forceinline__ void cmac(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}

// twiddle omega_n^k for direction DIR from the forward table of length n
// (tw[k] = exp(-2 pi i k / n)); the inverse is the conjugate.
template <int DIR>
__device__ __forceinline__ float2 tw_dir(float2 t) { return DIR < 0 ? t : conjf2(t); }

// ---- in-register DFTs, natural-order output, y_m = sum_k x_k w_R^{DIR*m*k} ----
template <int DIR>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int DIR>
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
  float2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  float2 t2 = cadd(x1, x3), t3 = mul_dir_i<DIR>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <int DIR>
__device__ __forceinline__ void dft8(float2* v) {
  const float r = 0.70710678118654752440f;
  float2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  float2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<DIR>(e0, e1, e2, e3);
  dft4<DIR>(o0, o1, o2, o3);
  // o1 *= w8^1, o2 *= w8^2, o3 *= w8^3   (w8 = exp(DIR*2*pi*i/8))
  float2 t1, t3;
  if (DIR < 0) {
    t1 = make_float2((o1.x + o1.y) * r, (o1.y - o1.x) * r);
    t3 = make_float2((o3.y - o3.x) * r, -(o3.x + o3.y) * r);
  } else {
    t1 = make_float2((o1.x - o1.y) * r, (o1.x + o1.y) * r);
    t3 = make_float2(-(o3.x + o3.y) * r, (o3.x - o3.y) * r);
  }
  float2 t2 = mul_dir_i<DIR>(o2);
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, t1);
  v[5] = csub(e1, t1);
  v[2] = cadd(e2, t2);
  v[6] = csub(e2, t2);
  v[3] = cadd(e3, t3);
  v[7] = csub(e3, t3);
}

template <int R, int DIR>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 2) {
    dft2<DIR>(v[0], v[1]);
  } else if constexpr (R == 4) {
    dft4<DIR>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 8) {
    dft8<DIR>(v);
  } else if constexpr (R == 1) {
  }
}

__host__ __device__ __forceinline__ int ilog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

}  // namespace tfno
