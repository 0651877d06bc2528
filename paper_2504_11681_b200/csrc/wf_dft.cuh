// In-register DFTs of length L = 16 / 32 used by the warp-synchronous row
// FFTs (warpfft.cu) and the fused 1D layer kernel (fused1d.cu).
#pragma once
#include "common.cuh"

namespace tfno {
namespace wf {

// natural-order in-register DFT of length L (16 or 32): L = P*8,
// x[n1 + P n2] -> DFT8 over n2 -> twiddle w_L^{n1 k2} -> DFT_P over n1,
// output k = k2 + 8 k1.  v is overwritten with the natural-order output.
template <int L, int DIR>
__device__ __forceinline__ void dftL(float2* v, const float2* __restrict__ twL /* w_L^k, k < L (forward sign) */) {
  constexpr int P = L / 8;
  float2 a[P][8];
#pragma unroll
  for (int n1 = 0; n1 < P; ++n1) {
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) a[n1][n2] = v[n1 + P * n2];
    dft8<DIR>(a[n1]);
  }
#pragma unroll
  for (int n1 = 1; n1 < P; ++n1)
#pragma unroll
    for (int k2 = 1; k2 < 8; ++k2) a[n1][k2] = cmul(a[n1][k2], tw_dir<DIR>(twL[n1 * k2]));
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    float2 b[P];
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) b[n1] = a[n1][k2];
    dft<P, DIR>(b);
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) v[k2 + 8 * k1] = b[k1];
  }
}

// first KP outputs of a forward DFT_L (KP <= 8): sum over n1 of the twiddled
// DFT8 outputs (k1 = 0 of the second factor)
template <int L, int KP>
__device__ __forceinline__ void dftL_first(const float2* v, float2* out, const float2* __restrict__ twL) {
  constexpr int P = L / 8;
  float2 a[P][8];
#pragma unroll
  for (int n1 = 0; n1 < P; ++n1) {
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) a[n1][n2] = v[n1 + P * n2];
    dft8<-1>(a[n1]);
  }
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    float2 s = a[0][k];
#pragma unroll
    for (int n1 = 1; n1 < P; ++n1) s = cadd(s, k ? cmul(a[n1][k], twL[n1 * k]) : a[n1][k]);
    out[k] = s;
  }
}

// inverse DFT_L with only the first KP inputs nonzero (KP <= 8):
// z[t_lo + 8 t_hi] = sum_k (x[k] w_L^{+k t_lo}) w_P^{+k t_hi}, P = L/8: per t_lo
// twiddle the KP inputs, fold k -> k mod P, inverse DFT_P over k mod P -> t_hi.
template <int L, int KP>
__device__ __forceinline__ void idftL_padded(const float2* x, float2* out, const float2* __restrict__ twL) {
  constexpr int P = L / 8;
  static_assert(KP <= 8, "padded inputs");
#pragma unroll
  for (int tl = 0; tl < 8; ++tl) {
    float2 f[P];
#pragma unroll
    for (int r = 0; r < P; ++r) f[r] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int e = (k * tl) % L;
      const float2 xk = e ? cmul(x[k], conjf2(twL[e])) : x[k];
      f[k % P] = cadd(f[k % P], xk);
    }
    dft<P, 1>(f);
#pragma unroll
    for (int th = 0; th < P; ++th) out[tl + 8 * th] = f[th];
  }
}

}  // namespace wf

}  // namespace tfno
